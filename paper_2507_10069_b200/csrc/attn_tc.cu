// attn_tc.cu — prefill / encoder attention on tcgen05 for sm_100a (K4 / K5).
//
// Varlen flash attention over a batch of sequences: the uncached suffix's
// queries attend over [cached prefix KV | suffix KV] (causal, queries aligned
// to the end of the KV sequence), or bidirectionally inside an image (ViT).
// GQA by head grouping.  This is the compute the reference models as
// prefill_time / encode_time (pkg/src/mmsim/costmodel.py:102-119).
//
// Persistent: one CTA per SM loops over work items (sequence, q-head, PAIR
// of 128-query tiles; longest first) — the two tiles of an item share every
// K/V block loaded into shared memory, and the next item's Q/K/V loads and
// S MMAs overlap the current item's epilogue:
//   warp 0       TMA: Q0, Q1 once; K/V 128-row blocks into a 2-stage ring
//   warp 1       MMA: S_i = Q_i K_j^T (SS) and O_i += P_i V_j with P_i read
//                straight from TMEM (TS); issue order S0 S1 | PV0 S0' | PV1 S1'
//                so the tensor core works on one tile while the other tile's
//                softmax runs
//   warps 4..7   softmax of tile 0, warps 8..11 softmax of tile 1: one thread
//                per query row, row max over S in TMEM, p = exp2(s - m) packed
//                to bf16 and stored back over S (P aliases S), lazy O rescale
//                (only when the running max grows by > 2^8), 1/l at the end.
// TMEM: S0/P0 [0,128) S1/P1 [128,256) O0 [256,256+HD) O1 [384, 384+HD).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../../include/emm.h"
#include "ptx.cuh"
#include "runtime.h"

namespace emm {

constexpr int ATT_THREADS = 384;
constexpr int ATT_BM = 128;  // query rows per tile (2 tiles per CTA)
constexpr int ATT_BN = 128;  // kv rows per block
constexpr float ATT_RESCALE_THRESH = 8.0f;  // log2 units: p <= 256 between rescales
#ifndef ATT_EXP_X
#define ATT_EXP_X 0  // profiling knobs: 1 = no exp2, 2 = skip pass 1, 3 = softmax no-op
#endif

struct AttnArgs {
  const int32_t* tiles;  // [n_tiles][3] = seq, q head, first q tile (of a pair)
  int n_tiles;
  const int32_t* q_start;
  const int32_t* q_len;
  const int32_t* kv_start;
  const int32_t* kv_len;
  __nv_bfloat16* out;
  int64_t out_tok_stride;  // elements
  int n_q_heads, group;    // group = n_q_heads / n_kv_heads
  float scale_log2;        // softmax scale * log2(e)
  int causal;
};

// head_dim = CH x 64 (SW128 chunks, 16 KiB per 128 rows) + REM (0 or 16: one
// SW32 chunk of 4 KiB; head_dim 80 of the Qwen2.5-VL vision tower).
template <int HD>
struct AttnCfg {
  static constexpr int CH = HD / 64;               // 64-element SW128 chunks per row
  static constexpr int REM = HD % 64;              // SW32 tail (0 or 16 elements)
  static_assert(REM == 0 || REM == 16, "head_dim must be 64k or 64k + 16");
  static constexpr int TILE_BYTES = 128 * HD * 2;  // one 128-row bf16 tile
  static constexpr int Q_OFF = 0;                  // Q0, Q1
  static constexpr int K_OFF = 2 * TILE_BYTES;     // 2 stages
  static constexpr int V_OFF = K_OFF + 2 * TILE_BYTES;
  static constexpr int BAR_OFF = V_OFF + 2 * TILE_BYTES;
  // q_full, k_full[2], v_full[2], kv_empty[2], s_full[2], p_full[2], o_done[2],
  // q_empty, o_free[2]
  static constexpr int N_BARS = 16;
  static constexpr int SMEM = BAR_OFF + N_BARS * 8 + 16 + 1024;
};

__device__ __forceinline__ float fast_exp2(float x) {
#if ATT_EXP_X == 1
  return x;
#else
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
#endif
}

__device__ __forceinline__ int attn_nblk(const AttnArgs& a, int seq, int qt_last) {
  const int ql = a.q_len[seq], kl = a.kv_len[seq];
  if (!a.causal) return (kl + ATT_BN - 1) / ATT_BN;
  const int last_q = min(ql, (qt_last + 1) * ATT_BM) - 1;  // last query row of the pair
  const int last_pos = kl - ql + last_q;                   // its absolute KV position
  return min(last_pos / ATT_BN + 1, (kl + ATT_BN - 1) / ATT_BN);
}

template <int HD>
__global__ void __launch_bounds__(ATT_THREADS, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmQ,
                       const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV,
                       const __grid_constant__ CUtensorMap tmQr,
                       const __grid_constant__ CUtensorMap tmKr,
                       const __grid_constant__ CUtensorMap tmVr, const AttnArgs a) {
  using Cfg = AttnCfg<HD>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::BAR_OFF);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* v_full = bars + 3;
  uint64_t* kv_empty = bars + 5;
  uint64_t* s_full = bars + 7;
  uint64_t* p_full = bars + 9;
  uint64_t* o_done = bars + 11;
  uint64_t* q_empty = bars + 13;
  uint64_t* o_free = bars + 14;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + Cfg::N_BARS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    if (Cfg::REM) {
      tma_prefetch(&tmQr);
      tma_prefetch(&tmKr);
      tma_prefetch(&tmVr);
    }
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&o_done[i], 1);
      mbar_init(&o_free[i], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  // every role walks the same item sequence; g counts KV blocks across items
  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------- TMA
      int g = 0, it = 0;
      for (int item = blockIdx.x; item < a.n_tiles; item += gridDim.x, ++it) {
        const int seq = a.tiles[3 * item], head = a.tiles[3 * item + 1],
                  qt0 = a.tiles[3 * item + 2];
        const int kvh = head / a.group;
        const int q0 = a.q_start[seq] + qt0 * ATT_BM, kv0 = a.kv_start[seq];
        const int nblk = attn_nblk(a, seq, qt0 + 1);
        mbar_wait(q_empty, (it & 1) ^ 1);
        mbar_arrive_expect_tx(q_full, 2 * Cfg::TILE_BYTES);
        for (int t = 0; t < 2; ++t) {
          for (int c = 0; c < Cfg::CH; ++c)
            tma_load_3d(smem + Cfg::Q_OFF + t * Cfg::TILE_BYTES + c * 16384, &tmQ, q_full,
                        c * 64, head, q0 + t * ATT_BM);
          if (Cfg::REM)
            tma_load_3d(smem + Cfg::Q_OFF + t * Cfg::TILE_BYTES + Cfg::CH * 16384, &tmQr,
                        q_full, Cfg::CH * 64, head, q0 + t * ATT_BM);
        }
        for (int j = 0; j < nblk; ++j, ++g) {
          const int st = g & 1;
          mbar_wait(&kv_empty[st], ((g >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&k_full[st], Cfg::TILE_BYTES);
          for (int c = 0; c < Cfg::CH; ++c)
            tma_load_3d(smem + Cfg::K_OFF + st * Cfg::TILE_BYTES + c * 16384, &tmK, &k_full[st],
                        c * 64, kvh, kv0 + j * ATT_BN);
          if (Cfg::REM)
            tma_load_3d(smem + Cfg::K_OFF + st * Cfg::TILE_BYTES + Cfg::CH * 16384, &tmKr,
                        &k_full[st], Cfg::CH * 64, kvh, kv0 + j * ATT_BN);
          mbar_arrive_expect_tx(&v_full[st], Cfg::TILE_BYTES);
          for (int c = 0; c < Cfg::CH; ++c)
            tma_load_3d(smem + Cfg::V_OFF + st * Cfg::TILE_BYTES + c * 16384, &tmV, &v_full[st],
                        c * 64, kvh, kv0 + j * ATT_BN);
          if (Cfg::REM)
            tma_load_3d(smem + Cfg::V_OFF + st * Cfg::TILE_BYTES + Cfg::CH * 16384, &tmVr,
                        &v_full[st], Cfg::CH * 64, kvh, kv0 + j * ATT_BN);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------- MMA
      constexpr uint32_t idesc_s = idesc_bf16_f32(128, ATT_BN, false, false);
      constexpr uint32_t idesc_o = idesc_bf16_f32(128, Cfg::CH * 64, false, true);
      constexpr uint32_t idesc_or = idesc_bf16_f32(128, 16, false, true);
      const uint32_t q_addr = smem_u32(smem + Cfg::Q_OFF);
      auto issue_s = [&](int t, int g) {  // S_t = Q_t K_g^T into TMEM [t*128, +128)
        const uint32_t k_addr = smem_u32(smem + Cfg::K_OFF + (g & 1) * Cfg::TILE_BYTES);
        const uint32_t qa = q_addr + t * Cfg::TILE_BYTES;
#pragma unroll
        for (int kk = 0; kk < Cfg::CH * 4; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          mma_ss(tbase + t * 128, desc_sw128_kmajor(qa + off), desc_sw128_kmajor(k_addr + off),
                 idesc_s, kk != 0);
        }
        if (Cfg::REM) {  // the 16-wide SW32 tail is one more K = 16 step
          const uint32_t off = Cfg::CH * 16384;
          mma_ss(tbase + t * 128, desc_sw32_kmajor(qa + off), desc_sw32_kmajor(k_addr + off),
                 idesc_s, true);
        }
        mma_commit(&s_full[t]);
      };
      auto issue_pv = [&](int t, int g, bool first) {  // O_t += P_t V_g, P_t from TMEM
        const uint32_t v_addr = smem_u32(smem + Cfg::V_OFF + (g & 1) * Cfg::TILE_BYTES);
        const uint32_t o_addr = tbase + 256 + t * 128;
#pragma unroll
        for (int kk = 0; kk < ATT_BN / 16; ++kk) {
          const uint64_t bdesc = desc_sw128_mnmajor(v_addr + kk * 2048, 16384);
          mma_ts(o_addr, tbase + t * 128 + kk * 8, bdesc, idesc_o, (!first) || kk != 0);
          if (Cfg::REM)  // O columns [CH*64, HD) from the SW32 tail of V
            mma_ts(o_addr + Cfg::CH * 64, tbase + t * 128 + kk * 8,
                   desc_sw32_mnmajor(v_addr + Cfg::CH * 16384 + kk * 512), idesc_or,
                   (!first) || kk != 0);
        }
        mma_commit(&o_done[t]);
      };
      int g = 0, it = 0;
      for (int item = blockIdx.x; item < a.n_tiles; item += gridDim.x, ++it) {
        const int seq = a.tiles[3 * item], qt0 = a.tiles[3 * item + 2];
        const int nblk = attn_nblk(a, seq, qt0 + 1);
        mbar_wait(q_full, it & 1);
        mbar_wait(&k_full[g & 1], (g >> 1) & 1);
        tc_fence_after();
        issue_s(0, g);
        issue_s(1, g);
        if (nblk == 1) mma_commit(q_empty);
        for (int j = 0; j < nblk; ++j, ++g) {
          const int st = g & 1;
          const bool more = j + 1 < nblk;
          mbar_wait(&v_full[st], (g >> 1) & 1);
          if (more) mbar_wait(&k_full[st ^ 1], ((g + 1) >> 1) & 1);
          for (int t = 0; t < 2; ++t) {
            mbar_wait(&p_full[t], g & 1);
            if (j == 0) mbar_wait(&o_free[t], (it & 1) ^ 1);  // epilogue of the last item read O
            tc_fence_after();
            issue_pv(t, g, j == 0);
            if (more) issue_s(t, g + 1);  // in-order: reads P_t before S_t is overwritten
          }
          if (more && j + 2 == nblk) mma_commit(q_empty);  // last S of the item issued
          mma_commit(&kv_empty[st]);
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------- softmax
    const int t = (warp - 4) >> 2;               // tile of this warpgroup
    const int ew = warp & 3;                     // TMEM lane quarter
    const int r = ew * 32 + lane;                // query row in the tile
    const uint32_t lane_off = (uint32_t)(ew * 32) << 16;
    const uint32_t t_s = tbase + lane_off + t * 128;
    const uint32_t t_o = tbase + lane_off + 256 + t * 128;
    int g = 0, it = 0;
    for (int item = blockIdx.x; item < a.n_tiles; item += gridDim.x, ++it) {
      const int seq = a.tiles[3 * item], head = a.tiles[3 * item + 1],
                qt0 = a.tiles[3 * item + 2];
      const int q_len = a.q_len[seq], kv_len = a.kv_len[seq];
      const int nblk = attn_nblk(a, seq, qt0 + 1);
      const int qrow = (qt0 + t) * ATT_BM + r;   // query index within the sequence
      const int qpos = kv_len - q_len + qrow;    // absolute KV position of the query
      const int lim = a.causal ? min(qpos + 1, kv_len) : kv_len;  // visible keys: pos < lim
      float m_used = -INFINITY, l_run = 0.f;
      for (int j = 0; j < nblk; ++j, ++g) {
        mbar_wait(&s_full[t], g & 1);
        tc_fence_after();
        const int kbase = j * ATT_BN;
        // interior blocks (every key visible to every row of this warp) skip masking
        const bool full = __all_sync(0xffffffffu, kbase + ATT_BN <= lim);
        // pass 1: row max of the raw scores (scale > 0 commutes with max)
        float mx = -INFINITY;
#if ATT_EXP_X >= 2
        mx = 0.f;
#pragma unroll 1
        for (int c = 0; c < 0; ++c) {
#else
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
#endif
          uint32_t v[32];
          tmem_ld32(t_s + c * 32, v);
          tmem_wait_ld();
          if (full) {
#pragma unroll
            for (int i = 0; i < 32; ++i) mx = fmaxf(mx, __uint_as_float(v[i]));
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              mx = fmaxf(mx, kbase + c * 32 + i < lim ? __uint_as_float(v[i]) : -INFINITY);
          }
        }
        mx *= a.scale_log2;
        // lazy rescale: O and l only when the running max grew by > 2^8
        const bool grow = mx > m_used + ATT_RESCALE_THRESH;
        if (j == 0) {
          m_used = mx;
        } else if (__any_sync(0xffffffffu, grow)) {
          // S_t's commit covers PV_{j-1}: O_t is complete here
          const float m_new = grow ? mx : m_used;
          const float alpha = fast_exp2(m_used - m_new);
#pragma unroll 1
          for (int c = 0; c < HD / 32; ++c) {
            uint32_t o[32];
            tmem_ld32(t_o + c * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(t_o + c * 32, o);
          }
          if (HD % 32) {
            uint32_t o[16];
            tmem_ld16(t_o + (HD / 32) * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st16(t_o + (HD / 32) * 32, o);
          }
          l_run *= alpha;
          m_used = m_new;
        }
        const float nbase = m_used == -INFINITY ? 0.f : -m_used;
        const float sc = a.scale_log2;
        // pass 2: p = exp2(s*scale - m) -> bf16 pairs over the first 64 columns (P aliases S)
        float rsum0 = 0.f, rsum1 = 0.f;
#pragma unroll 1
        for (int c = 0; c < (ATT_EXP_X == 3 ? 0 : 4); ++c) {
          uint32_t v[32];
          tmem_ld32(t_s + c * 32, v);
          tmem_wait_ld();
          uint32_t pk[16];
          if (full) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float p0 = fast_exp2(fmaf(__uint_as_float(v[2 * i]), sc, nbase));
              const float p1 = fast_exp2(fmaf(__uint_as_float(v[2 * i + 1]), sc, nbase));
              rsum0 += p0;
              rsum1 += p1;
              pk[i] = pack_bf16(p0, p1);
            }
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int kp = kbase + c * 32 + 2 * i;
              const float p0 =
                  kp < lim ? fast_exp2(fmaf(__uint_as_float(v[2 * i]), sc, nbase)) : 0.f;
              const float p1 =
                  kp + 1 < lim ? fast_exp2(fmaf(__uint_as_float(v[2 * i + 1]), sc, nbase)) : 0.f;
              rsum0 += p0;
              rsum1 += p1;
              pk[i] = pack_bf16(p0, p1);
            }
          }
          tmem_st16(t_s + c * 16, pk);
        }
        const float rsum = rsum0 + rsum1;
        l_run += rsum;
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[t]);
      }
      // epilogue: O / l -> bf16, then hand O back to the MMA warp
      mbar_wait(&o_done[t], (g - 1) & 1);
      tc_fence_after();
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      const bool ok = qrow < q_len;
      __nv_bfloat16* orow = a.out +
                            (int64_t)(a.q_start[seq] + qrow) * a.out_tok_stride +
                            (int64_t)head * HD;
#pragma unroll 1
      for (int c = 0; c < HD / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(t_o + c * 32, o);
        tmem_wait_ld();
        if (ok) {
          uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 u;
            u.x = pack_bf16(__uint_as_float(o[8 * q + 0]) * inv, __uint_as_float(o[8 * q + 1]) * inv);
            u.y = pack_bf16(__uint_as_float(o[8 * q + 2]) * inv, __uint_as_float(o[8 * q + 3]) * inv);
            u.z = pack_bf16(__uint_as_float(o[8 * q + 4]) * inv, __uint_as_float(o[8 * q + 5]) * inv);
            u.w = pack_bf16(__uint_as_float(o[8 * q + 6]) * inv, __uint_as_float(o[8 * q + 7]) * inv);
            dst[q] = u;
          }
        }
      }
      if (HD % 32) {
        uint32_t o[16];
        tmem_ld16(t_o + (HD / 32) * 32, o);
        tmem_wait_ld();
        if (ok) {
          uint4* dst = reinterpret_cast<uint4*>(orow + (HD / 32) * 32);
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            uint4 u;
            u.x = pack_bf16(__uint_as_float(o[8 * q + 0]) * inv, __uint_as_float(o[8 * q + 1]) * inv);
            u.y = pack_bf16(__uint_as_float(o[8 * q + 2]) * inv, __uint_as_float(o[8 * q + 3]) * inv);
            u.z = pack_bf16(__uint_as_float(o[8 * q + 4]) * inv, __uint_as_float(o[8 * q + 5]) * inv);
            u.w = pack_bf16(__uint_as_float(o[8 * q + 6]) * inv, __uint_as_float(o[8 * q + 7]) * inv);
            dst[q] = u;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_free[t]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

template <int HD>
static int launch_attn(const void* q, int64_t q_tok_stride, const void* k, const void* v,
                       int64_t kv_tok_stride, int64_t n_q_tokens, int64_t n_kv_tokens,
                       int n_q_heads, int n_kv_heads, const AttnArgs& args, int n_tiles,
                       cudaStream_t stream) {
  using Cfg = AttnCfg<HD>;
  CUtensorMap tq, tk, tv, tqr, tkr, tvr;
  const CUtensorMapDataType bf = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  if (!make_tmap_3d(&tq, q, bf, 2, HD, n_q_heads, n_q_tokens, HD * 2, q_tok_stride * 2, 64, 1,
                    ATT_BM, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_tmap_3d(&tk, k, bf, 2, HD, n_kv_heads, n_kv_tokens, HD * 2, kv_tok_stride * 2, 64,
                    1, ATT_BN, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_tmap_3d(&tv, v, bf, 2, HD, n_kv_heads, n_kv_tokens, HD * 2, kv_tok_stride * 2, 64,
                    1, ATT_BN, CU_TENSOR_MAP_SWIZZLE_128B))
    return EMM_E_INVALID;
  if (Cfg::REM) {
    if (!make_tmap_3d(&tqr, q, bf, 2, HD, n_q_heads, n_q_tokens, HD * 2, q_tok_stride * 2, 16,
                      1, ATT_BM, CU_TENSOR_MAP_SWIZZLE_32B) ||
        !make_tmap_3d(&tkr, k, bf, 2, HD, n_kv_heads, n_kv_tokens, HD * 2, kv_tok_stride * 2,
                      16, 1, ATT_BN, CU_TENSOR_MAP_SWIZZLE_32B) ||
        !make_tmap_3d(&tvr, v, bf, 2, HD, n_kv_heads, n_kv_tokens, HD * 2, kv_tok_stride * 2,
                      16, 1, ATT_BN, CU_TENSOR_MAP_SWIZZLE_32B))
      return EMM_E_INVALID;
  } else {
    tqr = tq;
    tkr = tk;
    tvr = tv;
  }
  static bool attr_done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_done[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_tc_kernel<HD>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return cuda_status(e, "attn smem attribute");
    attr_done[dev & 63] = true;
  }
  const int grid = n_tiles < sm_count() ? n_tiles : sm_count();
  attn_fwd_tc_kernel<HD><<<grid, ATT_THREADS, Cfg::SMEM, stream>>>(tq, tk, tv, tqr, tkr, tvr,
                                                                     args);
  count_launch();
  EMM_CUDA_CHECK_LAUNCH("attn_fwd_tc_kernel");
  return EMM_OK;
}

}  // namespace emm

extern "C" int emm_attention_bf16(const void* q, int64_t q_tok_stride, const void* k,
                                  const void* v, int64_t kv_tok_stride, void* out,
                                  int64_t out_tok_stride, int64_t n_q_tokens,
                                  int64_t n_kv_tokens, int n_q_heads, int n_kv_heads,
                                  int head_dim, const int32_t* tiles, int n_tiles,
                                  const int32_t* q_start, const int32_t* q_len,
                                  const int32_t* kv_start, const int32_t* kv_len, float scale,
                                  int causal, void* stream) {
  using namespace emm;
  if (n_tiles <= 0) return EMM_OK;
  if (!q || !k || !v || !out || n_kv_heads <= 0 || n_q_heads % n_kv_heads != 0 ||
      (head_dim != 64 && head_dim != 80 && head_dim != 128) || (q_tok_stride % 8) || (kv_tok_stride % 8) ||
      (out_tok_stride % 8)) {
    emm_abi::set_error("emm_attention_bf16: head_dim 64/80/128, GQA divisibility, 16B pitches");
    return EMM_E_INVALID;
  }
  AttnArgs a;
  a.tiles = tiles;
  a.n_tiles = n_tiles;
  a.q_start = q_start;
  a.q_len = q_len;
  a.kv_start = kv_start;
  a.kv_len = kv_len;
  a.out = reinterpret_cast<__nv_bfloat16*>(out);
  a.out_tok_stride = out_tok_stride;
  a.n_q_heads = n_q_heads;
  a.group = n_q_heads / n_kv_heads;
  a.scale_log2 = scale * 1.4426950408889634f;
  a.causal = causal;
  cudaStream_t st = (cudaStream_t)stream;
  if (head_dim == 128)
    return launch_attn<128>(q, q_tok_stride, k, v, kv_tok_stride, n_q_tokens, n_kv_tokens,
                            n_q_heads, n_kv_heads, a, n_tiles, st);
  if (head_dim == 80)
    return launch_attn<80>(q, q_tok_stride, k, v, kv_tok_stride, n_q_tokens, n_kv_tokens,
                           n_q_heads, n_kv_heads, a, n_tiles, st);
  return launch_attn<64>(q, q_tok_stride, k, v, kv_tok_stride, n_q_tokens, n_kv_tokens,
                         n_q_heads, n_kv_heads, a, n_tiles, st);
}
