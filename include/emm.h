/* emm.h — C ABI of the B200-native unified multimodal prefix cache feeding
 * encode and prefill (ElasticMM hot path, arXiv 2507.10069).
 *
 * Plain pointers and sizes only.  Every entry point returns an int status
 * (0 = EMM_OK); emm_last_error() gives the thread-local message.  Device
 * entry points are asynchronous on the caller's cudaStream_t (passed as
 * void*) and never synchronise unless stated.
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/pkg/src/mmsim/<file>:<line>).  The Python binding that a
 * reference maintainer would add is shown in INTEGRATION.md; the in-tree
 * binding is paper_2507_10069_b200/_lib.py (ctypes).
 */
#ifndef EMM_H_
#define EMM_H_
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EMM_OK 0
#define EMM_E_INVALID 1
#define EMM_E_RELEASE_WITHOUT_MATCH 2 /* mmsim.cache.ReleaseWithoutMatch, cache.py:18-19 */
#define EMM_E_CUDA 3
#define EMM_E_OOM 4
#define EMM_E_INTERNAL 5

const char* emm_last_error(void);
int emm_version(void);

/* ------------------------------------------------------------------------
 * Host control plane: bit-exact decisions (cache.py:31-406)
 * ---------------------------------------------------------------------- */
typedef struct emm_pool emm_pool;   /* ImagePool   cache.py:31-74   */
typedef struct emm_tree emm_tree;   /* PrefixTree  cache.py:105-336 */
typedef struct emm_cache emm_cache; /* UnifiedCache cache.py:363-406 */

/* ImagePool(capacity_tokens)                          cache.py:34-38 */
int emm_pool_create(int64_t capacity_tokens, emm_pool** out);
int emm_pool_destroy(emm_pool* p);
/* ImagePool.lookup -> token count or -1 (None)       cache.py:40-46 */
int emm_pool_lookup(emm_pool* p, const char* content_hash, double now, int64_t* tokens_or_m1);
/* ImagePool.insert -> *ok = True/False               cache.py:48-61 */
int emm_pool_insert(emm_pool* p, const char* content_hash, int64_t token_count, double now,
                    int64_t bytes_estimate, int32_t* ok);
/* total_tokens, evictions, capacity, len()          cache.py:35-38,73-74 */
int emm_pool_info(emm_pool* p, int64_t out4[4]);
/* hashes evicted since the previous call, '\n'-joined into buf; *needed =
 * bytes required (call again with a larger buffer if needed > cap).      */
int emm_pool_take_evicted(emm_pool* p, char* buf, int64_t cap, int64_t* needed);

/* PrefixTree(capacity_tokens)                         cache.py:108-117 */
int emm_tree_create(int64_t capacity_tokens, emm_tree** out);
int emm_tree_destroy(emm_tree* t);
/* PrefixTree.match_prefix -> (matched_kv, handle)    cache.py:121-156 */
int emm_tree_match(emm_tree* t, const uint64_t* keys, const int64_t* weights, int64_t n,
                   double now, int64_t* matched_kv, uint64_t* handle);
/* PrefixTree.release; EMM_E_RELEASE_WITHOUT_MATCH    cache.py:158-167 */
int emm_tree_release(emm_tree* t, uint64_t handle);
/* PrefixTree.insert_prefix -> KV tokens added        cache.py:171-217 */
int emm_tree_insert(emm_tree* t, const uint64_t* keys, const int64_t* weights, int64_t n,
                    double now, int64_t* added);
/* PrefixTree.evict -> tokens freed                   cache.py:267-284 */
int emm_tree_evict(emm_tree* t, int64_t needed, double now, int64_t* freed);
/* capacity, total_tokens, evictions, increments, decrements, live handles,
 * eviction_log length, node count                   cache.py:108-117,326-336 */
int emm_tree_info(emm_tree* t, int64_t out8[8]);
/* eviction_log rows [i0, i0+n): (node_id, kv, last_used)   cache.py:114,283 */
int emm_tree_eviction_log(emm_tree* t, int64_t i0, int64_t n, int64_t* node_ids,
                          int64_t* kvs, double* last_used);
/* reachable nodes in pre-order (iter_nodes, cache.py:305-310): per node its
 * id, parent id, kv, user_count, last_used and span (keys/weights, CSR). */
int emm_tree_nodes(emm_tree* t, int64_t max_nodes, int64_t max_syms, int64_t* n_nodes,
                   int64_t* n_syms, int64_t* ids, int64_t* parents, int64_t* kvs,
                   int64_t* user_counts, double* last_used, int64_t* span_off,
                   uint64_t* span_keys, int64_t* span_w);
/* len(handle.entries) or -1 when not live            cache.py:93-103 */
int emm_tree_handle_entries(emm_tree* t, uint64_t handle, int64_t* n_entries);

/* UnifiedCache(budget_tokens, image_fraction)         cache.py:366-370 */
int emm_cache_create(int64_t budget_tokens, double image_fraction, emm_cache** out);
int emm_cache_destroy(emm_cache* c);
/* sub-objects for introspection (c.images / c.prefixes) */
int emm_cache_parts(emm_cache* c, emm_pool** images, emm_tree** prefixes);
int emm_cache_image_lookup(emm_cache* c, const char* content_hash, double now,
                           int64_t* tokens_or_m1);                       /* cache.py:372-379 */
int emm_cache_image_insert(emm_cache* c, const char* content_hash, int64_t token_count,
                           double now, int64_t bytes_estimate, int32_t* ok); /* :381-383 */
int emm_cache_match_prefix(emm_cache* c, const uint64_t* keys, const int64_t* weights,
                           int64_t n, double now, int64_t* matched_kv,
                           uint64_t* handle);                             /* :385-392 */
/* Same call with only the first n_avail of n_total keys encoded so far
 * (cache.py:121-156 stops at the first mismatch, so the caller encodes lazily):
 * when the walk would read past n_avail, nothing is changed and *need_more = 1;
 * the caller encodes more keys and calls again.  weights may be NULL (the
 * matched weight comes from the stored spans, cache.py:145). */
int emm_cache_match_prefix_lazy(emm_cache* c, const uint64_t* keys, int64_t n_avail,
                                int64_t n_total, double now, int64_t* matched_kv,
                                uint64_t* handle, int32_t* need_more);    /* :385-392 */
int emm_cache_insert_prefix(emm_cache* c, const uint64_t* keys, const int64_t* weights,
                            int64_t n, double now, int64_t* added);       /* :394-396 */
int emm_cache_release(emm_cache* c, uint64_t handle);                     /* :398-399 */
/* snapshot_stats(): image_hits, image_misses, image_tokens_saved,
 * prefix_lookups, prefix_hits, prefix_tokens_saved, evictions,
 * image_pool_tokens, prefix_pool_tokens               cache.py:341-360,401-406 */
int emm_cache_stats(emm_cache* c, int64_t out9[9]);

/* host restatement of the block hash (emm_hash.h) for the control plane */
int emm_prefix_hashes_host(const uint64_t* keys, const int64_t* weights, int64_t n,
                           uint64_t* h0, uint64_t* h1);

/* ------------------------------------------------------------------------
 * Device data plane (sm_100a).  All pointers are device pointers unless
 * named *_host.  Launches count toward emm_launch_count().
 * ---------------------------------------------------------------------- */
uint64_t emm_launch_count(void);
/* let `dev` load/store `peer` memory (K6 migration over NVLink P2P)         */
int emm_enable_peer_access(int dev, int peer);
int emm_device_sm_count(int device, int* sms);

/* K1 — block hashes of a batch of unified sequences (CSR by request):
 * h0/h1[j] = prefix hash at symbol j of its request, cumw[j] = inclusive
 * prefix sum of weights within the request.  Replaces the tuple identity of
 * Engine.unified_sequence (engine.py:448-461) for device matching.        */
int emm_block_hash(const uint64_t* keys, const int64_t* weights, const int64_t* seq_off,
                   int64_t n_seqs, uint64_t* h0, uint64_t* h1, int64_t* cumw, void* stream);

/* K1 — 122-bit content digest of n_imgs images; image i is the byte range
 * [img_start[i], img_start[i] + img_len[i]) of `bytes` (starts 8-byte
 * aligned; given on device and on host).  out[2*i], out[2*i+1] = lanes.
 * scratch_dev holds emm_pixel_digest_scratch_bytes() bytes.  Replaces the
 * identity hash of workload.generate (workload.py:191-192) with a hash of
 * the pixels.                                                              */
int64_t emm_pixel_digest_scratch_bytes(const int64_t* img_len_host, int64_t n_imgs);
int emm_pixel_digest(const uint8_t* bytes, const int64_t* img_start_dev,
                     const int64_t* img_len_dev, const int64_t* img_start_host,
                     const int64_t* img_len_host, int64_t n_imgs, void* scratch_dev,
                     uint64_t* out, void* stream);

/* Device mirror of one PrefixTree (GPU hash table + virtual token map).   */
typedef struct emm_index emm_index;
/* attach a device index to cache c: table for max_syms symbols, virtual
 * token space of v_tokens records, physical slots [0, n_slots).          */
int emm_index_attach(emm_cache* c, int device, int64_t max_syms, int64_t v_tokens,
                     int64_t n_slots, emm_index** out);
/* KV source for the next insert_prefix of each sequence: the sequence whose
 * prefix hash at its last symbol is (h0,h1) has its KV-token t at rows
 * src_row0 + t of the registered request KV buffer.                       */
int emm_index_set_kv_source(emm_index* ix, uint64_t h0, uint64_t h1, int64_t src_row0);
int emm_index_clear_kv_sources(emm_index* ix);
/* KV pool and request-buffer geometry for scatter-on-insert:
 * pool rows  : pool  + (layer*2 + kv)*pool_kv_stride  + slot*row_bytes
 * req  rows  : req   + (layer*2 + kv)*req_kv_stride   + row*row_bytes      */
int emm_index_set_kv_geometry(emm_index* ix, void* pool, int64_t pool_kv_stride, void* req,
                              int64_t req_kv_stride, int64_t row_bytes, int64_t n_layers);
/* Prefill batches split across GPUs: register another request KV buffer
 * (same row geometry; may live on a peer GPU, read over NVLink by the
 * scatter) -> *buffer; emm_index_set_kv_geometry resets the list to its
 * own buffer 0.  Sources then name the buffer their rows live in.         */
int emm_index_add_request_buffer(emm_index* ix, void* req, int64_t req_kv_stride, int* buffer);
int emm_index_set_kv_source_buf(emm_index* ix, uint64_t h0, uint64_t h1, int buffer,
                                int64_t src_row0);
/* apply pending device updates (publish / erase / scatter) on `stream`    */
int emm_index_flush(emm_index* ix, void* stream);
/* K2 — batched GPU prefix match.  Inputs: per-request prefix hashes (from
 * emm_block_hash), want_kv[r] (= cached_prefix, engine.py:546).  Outputs:
 * matched_sym[r], matched_kv[r] (device-computed, must equal the host tree,
 * cache.py:121-156), sym_v[j] (scratch: virtual token start of each matched
 * symbol) and the token-granular block table bt[bt_off[r] + t] = pool slot
 * of KV token t < min(want_kv[r], matched_kv[r]).                         */
int emm_index_match(emm_index* ix, const uint64_t* h0, const uint64_t* h1,
                    const int64_t* cumw, const int64_t* seq_off, int64_t n_seqs,
                    const int64_t* want_kv, const int64_t* bt_off, int64_t* matched_sym,
                    int64_t* matched_kv, int64_t* sym_v, int32_t* bt, void* stream);
/* stream used by the automatic flush after emm_cache_insert_prefix        */
int emm_index_set_stream(emm_index* ix, void* stream);
/* live symbols, tombstones, table capacity, free slots, device error flag
 * (synchronous read), free virtual tokens                                 */
int emm_index_info(emm_index* ix, int64_t out6[6]);
/* host mirror of tok_slot[v0, v0+n) (introspection)                       */
int emm_index_tok_slots_host(emm_index* ix, int64_t v0, int64_t n, int32_t* out);

/* K3/K6 — row copy between paged pools and request buffers (TMA bulk
 * staged).  For each layer l < n_layers and K/V half h, row i:
 *   dst + (l*2+h)*dst_stride + dst_rows[i]*row_bytes
 *     <- src + (l*2+h)*src_stride + src_rows[i]*row_bytes
 * dst may live on a peer GPU (NVLink P2P).                                */
int emm_kv_copy_rows(const void* src, int64_t src_stride, const int32_t* src_rows, void* dst,
                     int64_t dst_stride, const int32_t* dst_rows, int64_t n_rows,
                     int64_t row_bytes, int64_t n_layers, void* stream);
/* K6 on the copy engines: rows [0, n_rows) of every (layer, K/V) plane as ONE
 * strided DMA (cudaMemcpy2DAsync, cudaMemcpyDefault: peer-to-peer over NVLink
 * when src and dst live on different GPUs with peer access enabled), no SMs
 * used.  Same plane layout as emm_kv_copy_rows with identity row maps.
 * Replaces migration_cost (costmodel.py:138-142) for execute_migration
 * (engine.py:753-788).                                                     */
int emm_kv_copy_planes_ce(const void* src, int64_t src_stride, void* dst, int64_t dst_stride,
                          int64_t n_rows, int64_t row_bytes, int64_t n_layers, void* stream);
/* K6 verification ("exact copying ... checksums"; the
 * reference only books the move, engine.py:797-823): *out_device (a device
 * uint64) = sum mod 2^64 over planes p < 2*n_layers and rows i < n_rows of
 * XXH64(row bytes, seed = p << 32 | i), the row at planes + p*plane_stride +
 * (rows ? rows[i] : i)*row_bytes.  Equal on both sides of an exact copy.
 * row_bytes and plane_stride multiples of 16, planes 16-byte aligned.     */
int emm_kv_checksum(const void* planes, int64_t plane_stride, const int32_t* rows,
                    int64_t n_rows, int64_t row_bytes, int64_t n_layers, uint64_t* out_device,
                    void* stream);

/* tcgen05 GEMM: C[M,N] = epilogue(A[M,K] . B[N,K]^T), bf16 in, fp32 TMEM
 * accumulate.  Replaces the analytic encode_time/prefill_time arithmetic
 * (costmodel.py:102-119) with real work.  epi: see EMM_EPI_*.             */
#define EMM_EPI_NONE 0
#define EMM_EPI_GELU_TANH 1
#define EMM_EPI_QUICK_GELU 2
#define EMM_EPI_GELU_ERF 3
#define EMM_EPI_GLU_SILU 4 /* B rows interleaved per 128: C[:, n/2] = silu(g)*u */
#define EMM_EPI_QKV_ROPE 5 /* split fused QKV, rotate-half RoPE, write q and the KV cache */

/* Epilogue description for emm_gemm_bf16_ex.  The folded-RMSNorm fields let
 * a GEMM consume the un-normalised residual stream x (norm weight folded
 * into B): acc[m][:] *= rsqrt(row_ss_in[m] * (1/rms_dim) + rms_eps); a
 * residual GEMM can emit row_ss_out[m] += sum(out[m][:]^2) for the next.  */
typedef struct emm_gemm_epilogue {
  int kind;
  const void* bias;          /* bf16 [N] or NULL */
  const void* residual;      /* bf16 [M, ldr] or NULL */
  int64_t ldr;
  const float* row_ss_in;    /* fp32 [M] or NULL */
  float rms_eps;
  int64_t rms_dim;
  float* row_ss_out;         /* fp32 [M] (zeroed by the caller) or NULL */
  void* q_out;               /* EMM_EPI_QKV_ROPE: bf16 [M, ld_q] */
  int64_t ld_q;
  void* k_out;               /* bf16 rows kv_row[m] of [*, ld_kv] */
  void* v_out;
  int64_t ld_kv;
  const int32_t* kv_row;
  const int32_t* pos;        /* RoPE position of row m (NULL: no rotation) */
  const float* rope_cs;      /* fp32 (cos, sin) pairs [max_pos][hd/2] */
  int hq, hkv, hd;
  /* multimodal RoPE (Qwen2-VL M-RoPE): when pos_h != NULL, rotary pair i
   * rotates by pos[m] (i < mrope_t), pos_h[m] (i < mrope_t + mrope_h) or
   * pos_w[m] (the rest).  NULL = 1-D RoPE by pos.                          */
  const int32_t* pos_h;
  const int32_t* pos_w;
  int mrope_t, mrope_h;
  /* optional: zero row_ss_zero[m] for every output row (the buffer the NEXT
   * residual GEMM accumulates its row sum of squares into; saves a memset
   * launch per layer)                                                     */
  float* row_ss_zero;
  /* optional 2-D vision RoPE on output columns [0, rope2_cols) (the q and k
   * sections of a fused QKV whose weight rows put each rotary pair (i, i +
   * hd/2) of a head in adjacent columns): pair i of a head rotates by
   * pos_h[m] (i < hd/4) or pos_w[m] with (cos, sin) = rope2_cs[pos][i mod
   * hd/4] — Qwen2.5-VL's vision rotary embedding, applied in the epilogue  */
  const float* rope2_cs;
  int rope2_cols, rope2_hd;
} emm_gemm_epilogue;
int emm_gemm_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                  int64_t M, int64_t N, int64_t K, const void* bias, const void* residual,
                  int64_t ldr, int epi, void* stream);
int emm_gemm_bf16_ex(const void* A, int64_t lda, const void* B, int64_t ldb, void* C,
                     int64_t ldc, int64_t M, int64_t N, int64_t K, const emm_gemm_epilogue* epi,
                     void* stream);


/* K4/K5 — varlen GQA flash attention on tcgen05 (S, P, O in TMEM).  Sequence
 * s: q rows [q_start, q_start+q_len) of q, keys/values rows [kv_start,
 * kv_start+kv_len) of k/v; causal => queries are the LAST q_len positions of
 * the KV sequence (uncached suffix after the cached prefix, engine.py:546).
 * row_bounds (optional, int32 pairs per q row of the q buffer): the row sees
 * KV positions [lo, hi) of its sequence only (the Qwen2.5-VL vision
 * windows; overrides causal).  tiles: n_tiles x (seq, q_head, first q tile,
 * first KV block, end KV block) — the KV blocks of 128 keys any row of the
 * item can see; an item is tile_rows = 256 queries (two 128-row tiles
 * sharing each K/V block) or 128 (one tile, S double-buffered in TMEM).
 * head_dim 64, 80 or 128.                                                  */
int emm_attention_bf16(const void* q, int64_t q_tok_stride, const void* k, const void* v,
                       int64_t kv_tok_stride, void* out, int64_t out_tok_stride,
                       int64_t n_q_tokens, int64_t n_kv_tokens, int n_q_heads, int n_kv_heads,
                       int head_dim, const int32_t* tiles, int n_tiles, const int32_t* q_start,
                       const int32_t* q_len, const int32_t* kv_start, const int32_t* kv_len,
                       const int32_t* row_bounds, float scale, int causal, int tile_rows,
                       void* stream);

/* out[i] = table[ids[i]] (row_bytes each; pitches in bytes)              */
int emm_embed_rows(const void* table, int64_t ld_bytes, const int32_t* ids, void* out,
                   int64_t ldo_bytes, int64_t T, int64_t row_bytes, void* stream);
/* decode: per request r < n, slot[r] = bt[bt_off[r] + kv_len[r]];
 * kv_len[r] += 1; pos[r] = next_pos[r]++  (device-side step advance)      */
int emm_decode_advance(const int32_t* bt, const int64_t* bt_off, int32_t* kv_len,
                       int32_t* next_pos, int32_t* slot, int32_t* pos, int64_t n, void* stream);
/* Decode: one query token per request against its KV
 * history in a token-granular paged arena: key t of request r is row
 * bt[bt_off[r] + t] of k_plane / v_plane (row stride row_stride elements,
 * kv head h at column h*hd), t < kv_len[r] <= max_kv_len.  q / out:
 * [n_req, hq*hd].  GQA with hq/hkv <= 16, head_dim 64 or 128.  The key
 * range is split across CTAs when requests x kv heads is below two waves;
 * the splits need emm_decode_attention_workspace() bytes of scratch.       */
int64_t emm_decode_attention_workspace(int64_t n_req, int hq, int hkv, int hd,
                                       int64_t max_kv_len);
int emm_decode_attention_bf16(const void* q, int64_t q_stride, const void* k_plane,
                              const void* v_plane, int64_t row_stride, const int32_t* bt,
                              const int64_t* bt_off, const int32_t* kv_len, int64_t n_req,
                              int hq, int hkv, int hd, int64_t max_kv_len, void* out,
                              int64_t out_stride, void* workspace, int64_t workspace_bytes,
                              float scale, void* stream);

/* RMSNorm (b == NULL) or LayerNorm of T rows of width D (optionally the rows
 * listed in `rows`), bf16 in/out, fp32 statistics.                        */
int emm_norm_bf16(const void* x, int64_t ldx, const int32_t* rows, const void* w,
                  const void* b, void* out, int64_t ldo, int64_t T, int64_t D, float eps,
                  int layernorm, void* stream);
/* split fused QKV rows, rotate-half RoPE at pos[t] (rope != 0), write q to
 * q_out[t] and k/v into the request KV buffer rows kv_row[t]               */
int emm_rope_split_bf16(const void* qkv, int64_t ld_qkv, int64_t T, int hq, int hkv, int hd,
                        const int32_t* pos, float theta, int rope, void* q_out, int64_t ld_q,
                        void* k_out, void* v_out, const int32_t* kv_row, int64_t ld_kv,
                        void* stream);
/* fp32 per-row sum of squares (input of the folded RMSNorm of layer 0)      */
int emm_row_sumsq_bf16(const void* x, int64_t ldx, int64_t T, int64_t D, float* out,
                       void* stream);
/* out[i] = row_bytes at device address src_ptr[i] (decoder input assembly
 * from text-embedding rows and image slabs)                                */
int emm_gather_rows(const int64_t* src_ptr, void* out, int64_t ldo_bytes, int64_t T,
                    int64_t row_bytes, void* stream);
/* uint8 HWC pixels -> normalised bf16 patch rows (c, ky, kx), K padded     */
int emm_patchify(const uint8_t* pix, const int64_t* pix_off, const int32_t* gh,
                 const int32_t* gw, const int64_t* patch_off, int n_img, int max_patches,
                 int patch, int k_pad, const float* mean3, const float* std3, void* out,
                 void* stream);
/* Qwen2.5-VL patchify: output row r = image row_img[r], raster patch
 * row_patch[r] (window order is the caller's permutation); columns
 * (c, t, ky, kx) over `temporal` copies of the frame, zero-padded to k_pad. */
int emm_patchify_rows(const uint8_t* pix, const int64_t* pix_off, const int32_t* gw,
                      const int32_t* row_img, const int32_t* row_patch, int64_t n_rows,
                      int patch, int temporal, int k_pad, const float* mean3,
                      const float* std3, void* out, void* stream);
/* in-place 2-D rotary embedding (Qwen2.5-VL vision) of the first n_heads
 * heads of each row of x (q then k of a fused QKV buffer): pair i < hd/4
 * rotates by pos_h[t] * theta^(-4i/hd), the next hd/4 pairs by pos_w[t].    */
int emm_rope2d_bf16(void* x, int64_t ldx, int64_t T, int n_heads, int hd,
                    const int32_t* pos_h, const int32_t* pos_w, float theta, void* stream);
/* ViT token rows: [CLS] + patch embeddings + learned position embeddings   */
int emm_vit_embed(const void* patch, const void* cls, const void* pos, void* out,
                  const int64_t* tok_off, const int64_t* patch_off, int n_img, int64_t n_rows,
                  int has_cls, int D, void* stream);
/* row-wise argmax (first token of every request)                           */
int emm_argmax_rows(const void* x, int64_t ldx, int64_t T, int64_t V, int32_t* out,
                    void* stream);
/* the same with the vocabulary split over CTAs: ws = caller-owned scratch of
 * emm_argmax_workspace_keys(T, V) 64-bit keys (no state kept between calls,
 * so safe under CUDA-graph capture and on any stream)                        */
#define EMM_ARGMAX_CHUNK 8192
int64_t emm_argmax_workspace_keys(int64_t T, int64_t V);
int emm_argmax_rows_ws(const void* x, int64_t ldx, int64_t T, int64_t V, int32_t* out,
                       uint64_t* ws, void* stream);

/* ------------------------------------------------------------------------
 * Scheduler host loop (csrc/host_sched.cpp): bit-exact
 * with the reference's Python.  `cost` = 8 doubles of the CostProfile
 * (costmodel.py:33-66), in this order:
 * ---------------------------------------------------------------------- */
#define EMM_COST_PREFILL_RATE 0
#define EMM_COST_PARALLEL_ALPHA 1
#define EMM_COST_MIGRATION_BANDWIDTH 2
#define EMM_COST_DECODE_BASE 3
#define EMM_COST_DECODE_BATCH_COEFF 4
#define EMM_COST_DECODE_KV_COEFF 5
#define EMM_COST_ENCODE_RATE 6
#define EMM_COST_DECODE_BATCH_THRESHOLD 7
typedef struct emm_estimator emm_estimator; /* LoadEstimator balancer.py:115-164 */
/* How the reference's sum(...) over floats adds (process-wide): 1 = CPython
 * >= 3.12 (Neumaier-compensated), 0 = CPython 3.10 / 3.11 (plain left to
 * right).  The binding sets it from sys.version_info at load.             */
int emm_sched_set_float_sum(int compensated);
int emm_estimator_create(const double* cost, double window_seconds, double bucket_seconds,
                         emm_estimator** out);                         /* balancer.py:123-128 */
int emm_estimator_destroy(emm_estimator* e);
int emm_estimator_service_seconds(emm_estimator* e, int64_t input_tokens, int64_t image_tokens,
                                  int64_t output_tokens, double* out); /* balancer.py:130-138 */
int emm_estimator_observe(emm_estimator* e, double now, int64_t input_tokens,
                          int64_t image_tokens, int64_t output_tokens); /* balancer.py:140-143 */
int emm_estimator_avg_required(emm_estimator* e, double now, int64_t* out); /* :150-153 */
int emm_estimator_peak_required(emm_estimator* e, double now, int64_t* out); /* :155-164 */
/* both, in that order (what engine.py:968-969 reads on every pass)        */
int emm_estimator_required(emm_estimator* e, double now, int64_t* avg, int64_t* peak);
int emm_estimator_len(emm_estimator* e, int64_t* out);
/* assign_idle_instances(avg_required, busy_counts, idle ids)  balancer.py:67-84;
 * groups in the caller's dict order, grants[i] for group_ids[i]           */
int emm_assign_idle(const int64_t* group_ids, const int64_t* avg_required,
                    const int64_t* busy_counts, int64_t n_groups, int64_t n_idle,
                    int64_t* grants);
/* place_reservations(requests, headroom)  partition.py:169-184.
 * reqs: n_req x (request id, kv_need); headroom: n_slots x (instance, free);
 * *ok = 0 where the reference returns None                                */
int emm_place_reservations(const int64_t* reqs, int64_t n_req, const int64_t* headroom,
                           int64_t n_slots, int64_t* placed_instance, int32_t* ok);
/* allocate_prefill(...)  partition.py:187-290.
 * reqs: n_req x (id, kv_need, input_len, prefill_tokens); idle / extra_homes:
 * n x (instance, kv_headroom); victims: n_vic x (instance, kv_unused,
 * kv_used, capacity, migratable); decode batch view = output_lens[n_out],
 * remaining_output, resident_kv, pool_instances; max_instances < 0 = None.
 * counts[6] = (instance ids, placements (-1 = None), preempted, forced,
 * dropped, decisions); placements as (request, instance) pairs in request
 * order; decision gain NaN = None (forced).  Output arrays sized n_idle +
 * n_vic (ids), n_req (placements, dropped), n_vic (the rest).              */
int emm_allocate_prefill(const double* cost, double penalty_w, int64_t max_instances,
                         const int64_t* reqs, int64_t n_req, const int64_t* idle, int64_t n_idle,
                         const int64_t* victims, int64_t n_vic, const int64_t* output_lens,
                         int64_t n_out, int64_t remaining_output, int64_t resident_kv,
                         int64_t pool_instances, const int64_t* extra_homes, int64_t n_extra,
                         int64_t* counts, int64_t* instance_ids, int64_t* placements,
                         int64_t* preempted, int64_t* forced, int64_t* dropped,
                         int64_t* dec_instance, int32_t* dec_forced, double* dec_gain,
                         double* dec_cost);

#ifdef __cplusplus
}
#endif
#endif /* EMM_H_ */
