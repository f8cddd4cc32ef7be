// decode_attn.cu — paged GQA decode attention (the
// decode stage after prefill, costmodel.py:121-136 / engine.py:670-693 in
// the reference, which models it analytically).
//
// One new query token per request attends to its whole KV history, whose
// rows live in a token-granular paged arena [layer][K|V][slot][kv_heads*hd]
// (the same layout as the prefix pool, "PagedAttention at the
// granularity of a single token"), addressed through a per-request block
// table bt[bt_off[r] + t] = slot.  The work is HBM-bound (every K/V byte is
// read once per step), so the kernel is built to stream bytes:
//
//  * grid (split, kv_head, request): all G = hq/hkv query heads of a KV head
//    share one pass over its rows (GQA: K/V read once, not G times); the key
//    range is split so that requests x kv_heads x splits fills the SMs;
//  * 4 warps per CTA, each streaming its own 16-key tiles through a 2-stage
//    cp.async ring in shared memory (16-byte chunks, XOR-swizzled rows: the
//    block-table indirection rules out TMA tensor maps; rows are 256 B
//    contiguous so every 16 lanes read one row coalesced; 64 KB of smem per
//    CTA at head_dim 128 -> 3 CTAs per SM: 32-key tiles, deeper rings or 8
//    warps all measured slower — occupancy beats ring depth here);
//  * S = Q K^T and O += P V on the tensor cores with mma.sync m16n8k16 (bf16
//    in, fp32 accumulate; the G query heads padded to 16 rows): a decode
//    step is far below the tcgen05 break-even size, and the MMA keeps the
//    FP32 pipes free — the kernel stays bandwidth-bound;
//  * online softmax in registers (exp2, per-row max over quad shuffles), P
//    re-used from the S accumulators as the A operand of PV (no smem trip);
//  * warps merge in shared memory; splits merge in a second small kernel.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>

#include "../../include/emm.h"
#include "ptx.cuh"
#include "runtime.h"

namespace emm {

#ifndef DA_TILE_KEYS
#define DA_TILE_KEYS 16
#endif
#ifndef DA_STAGES
#define DA_STAGES 2  // cp.async ring depth per warp
#endif
#ifndef DA_WAVES
#define DA_WAVES 4  // target CTA waves per launch (measured best of 2, 4, 8, 16)
#endif
#ifndef DA_NWARPS
#define DA_NWARPS 4
#endif
constexpr int DA_WARPS = DA_NWARPS;
constexpr int DA_TILE = DA_TILE_KEYS;  // keys per warp tile (16 or 32)
constexpr int DA_NT = DA_TILE / 8;     // n-tiles of S per tile
constexpr int DA_KS = DA_TILE / 16;    // k-steps of PV per tile

struct DecodeArgs {
  const __nv_bfloat16* q;  // [n_req, hq*hd] (row stride q_stride elements)
  int64_t q_stride;
  const __nv_bfloat16* k;  // this layer's K plane: row `slot` at k + slot*row_stride
  const __nv_bfloat16* v;
  int64_t row_stride;      // elements (= kv_heads*hd for the arena)
  const int32_t* bt;
  const int64_t* bt_off;
  const int32_t* kv_len;
  __nv_bfloat16* out;      // [n_req, hq*hd]
  int64_t out_stride;
  float* ws;               // split partials: O [..][G][hd] then (m, l) pairs
  int n_req, hq, hkv, G, n_split, tiles_per_split;
  float scale_log2;
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1,
                                          uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4],
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// byte offset of 16-byte chunk `ch` of row `row` in a [DA_TILE][HD] bf16 tile
template <int HD>
__device__ __forceinline__ uint32_t da_off(int row, int ch) {
  constexpr int CH = HD / 8;  // chunks per row
  return (uint32_t)(row * CH + (ch ^ (row & 7))) * 16u;
}

template <int HD>
__global__ void __launch_bounds__(DA_WARPS * 32)
    decode_attn_kernel(const DecodeArgs a) {
  constexpr int CH = HD / 8;                       // 16-byte chunks per row
  constexpr int TILE_BYTES = DA_TILE * HD * 2;     // one K (or V) tile
  constexpr int KSTEPS = HD / 16;
  constexpr int NT_O = HD / 8;                     // n-tiles of the output
  extern __shared__ __align__(128) uint8_t smem[];
  pdl_wait();  // launched with programmatic serialization: inputs are ready after this
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int split = blockIdx.x, kvh = blockIdx.y, req = blockIdx.z;
  const int G = a.G;
  const int len = a.kv_len[req];
  const int64_t bt0 = a.bt_off[req];
  const int t_begin = split * a.tiles_per_split;
  int t_end = t_begin + a.tiles_per_split;
  const int n_tiles_all = (len + DA_TILE - 1) / DA_TILE;
  if (t_end > n_tiles_all) t_end = n_tiles_all;

  // Q fragments (A operand, rows = the G query heads of this KV head)
  uint32_t qa[KSTEPS][4];
  {
    const int r0 = lane >> 2, r1 = r0 + 8, c = (lane & 3) * 2;
    const __nv_bfloat16* qb = a.q + (int64_t)req * a.q_stride + (int64_t)kvh * G * HD;
#pragma unroll
    for (int kk = 0; kk < KSTEPS; ++kk) {
      const int col = kk * 16 + c;
      auto ld = [&](int r, int cc) -> uint32_t {
        return r < G ? *reinterpret_cast<const uint32_t*>(qb + (int64_t)r * HD + cc) : 0u;
      };
      qa[kk][0] = ld(r0, col);
      qa[kk][1] = ld(r1, col);
      qa[kk][2] = ld(r0, col + 8);
      qa[kk][3] = ld(r1, col + 8);
    }
  }

  uint8_t* wsm = smem + warp * (DA_STAGES * 2 * TILE_BYTES);  // [stage][K|V] tiles of this warp
  const uint32_t wsm_u = smem_u32(wsm);
  const int64_t kv_head_off = (int64_t)kvh * HD;

  auto issue = [&](int tile, int stage) {
    const int key0 = tile * DA_TILE;
    int slot = 0;
    if (lane < DA_TILE) {
      int idx = key0 + lane;
      if (idx >= len) idx = len - 1;  // masked below; load a real row (no NaN)
      slot = a.bt[bt0 + idx];
    }
    const uint32_t kdst = wsm_u + stage * 2 * TILE_BYTES;
    const uint32_t vdst = kdst + TILE_BYTES;
#pragma unroll
    for (int it = 0; it < DA_TILE * CH / 32; ++it) {
      const int id = it * 32 + lane;
      const int row = id / CH, ch = id % CH;
      const int s = __shfl_sync(0xffffffffu, slot, row);
      const int64_t off = (int64_t)s * a.row_stride + kv_head_off + ch * 8;
      cp_async16(kdst + da_off<HD>(row, ch), a.k + off);
      cp_async16(vdst + da_off<HD>(row, ch), a.v + off);
    }
  };

  float o[NT_O][4];
#pragma unroll
  for (int j = 0; j < NT_O; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  int tile = t_begin + warp;
#pragma unroll
  for (int i = 0; i < DA_STAGES - 1; ++i) {
    if (tile + i * DA_WARPS < t_end) issue(tile + i * DA_WARPS, i);
    cp_async_commit();
  }
  int stage = 0;
  for (; tile < t_end; tile += DA_WARPS) {
    const int next = tile + (DA_STAGES - 1) * DA_WARPS;
    int nst = stage + DA_STAGES - 1;
    if (nst >= DA_STAGES) nst -= DA_STAGES;
    if (next < t_end) issue(next, nst);
    cp_async_commit();
    cp_async_wait<DA_STAGES - 1>();
    __syncwarp();
    const uint32_t kt = wsm_u + stage * 2 * TILE_BYTES;
    const uint32_t vt = kt + TILE_BYTES;
    // ---- S = Q K^T  (16 x 32)
    float s[DA_NT][4];
#pragma unroll
    for (int j = 0; j < DA_NT; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int j = 0; j < DA_NT; ++j) {    // 8 keys per n-tile
#pragma unroll
      for (int kk = 0; kk < KSTEPS; kk += 2) {
        // matrices: (keys j*8.., dims kk*16), (+8 dims), ((kk+1)*16), (+8)
        const int mat = lane >> 3, r = lane & 7;
        const int ch = kk * 2 + mat;
        uint32_t b0, b1, b2, b3;
        ldsm_x4(kt + da_off<HD>(j * 8 + r, ch), b0, b1, b2, b3);
        mma_bf16_16816(s[j], qa[kk], b0, b1);
        mma_bf16_16816(s[j], qa[kk + 1], b2, b3);
      }
    }
    // ---- mask + online softmax (rows r0 = lane>>2, r1 = r0 + 8)
    const int key0 = tile * DA_TILE;
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int j = 0; j < DA_NT; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int key = key0 + j * 8 + (lane & 3) * 2 + e;
        const bool ok = key < len;
        s[j][e] = ok ? s[j][e] * a.scale_log2 : -INFINITY;
        s[j][2 + e] = ok ? s[j][2 + e] * a.scale_log2 : -INFINITY;
        mx0 = fmaxf(mx0, s[j][e]);
        mx1 = fmaxf(mx1, s[j][2 + e]);
      }
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
    const float al0 = mn0 == -INFINITY ? 1.f : exp2f(m0 - mn0);
    const float al1 = mn1 == -INFINITY ? 1.f : exp2f(m1 - mn1);
    const float nb0 = mn0 == -INFINITY ? 0.f : mn0, nb1 = mn1 == -INFINITY ? 0.f : mn1;
    m0 = mn0;
    m1 = mn1;
    float rs0 = 0.f, rs1 = 0.f;
    uint32_t pa[DA_KS][4];  // P as A operand: k-steps of 16 keys
#pragma unroll
    for (int j = 0; j < DA_NT; ++j) {
      const float p0 = exp2f(s[j][0] - nb0), p1 = exp2f(s[j][1] - nb0);
      const float p2 = exp2f(s[j][2] - nb1), p3 = exp2f(s[j][3] - nb1);
      rs0 += p0 + p1;
      rs1 += p2 + p3;
      const int ks = j >> 1, hi = j & 1;
      pa[ks][hi * 2 + 0] = pack_bf16(p0, p1);
      pa[ks][hi * 2 + 1] = pack_bf16(p2, p3);
    }
    l0 = l0 * al0 + rs0;
    l1 = l1 * al1 + rs1;
#pragma unroll
    for (int j = 0; j < NT_O; ++j) {
      o[j][0] *= al0;
      o[j][1] *= al0;
      o[j][2] *= al1;
      o[j][3] *= al1;
    }
    // ---- O += P V  (16 x HD, k = DA_TILE keys)
#pragma unroll
    for (int ks = 0; ks < DA_KS; ++ks) {
#pragma unroll
      for (int j = 0; j < NT_O; j += 2) {
        // matrices: (keys ks*16.., dims j*8), (keys +8, dims j*8),
        //           (keys ks*16.., dims (j+1)*8), (keys +8, dims (j+1)*8)
        const int mat = lane >> 3, r = lane & 7;
        const int key = ks * 16 + (mat & 1) * 8 + r;
        const int ch = j + (mat >> 1);
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(vt + da_off<HD>(key, ch), b0, b1, b2, b3);
        mma_bf16_16816(o[j], pa[ks], b0, b1);
        mma_bf16_16816(o[j + 1], pa[ks], b2, b3);
      }
    }
    __syncwarp();
    stage = stage + 1 == DA_STAGES ? 0 : stage + 1;
  }
  cp_async_wait<0>();
  // row sums over the quad
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  __syncthreads();  // every warp is done with its tiles: reuse smem

  // ---- merge the 4 warps: per warp m, l [16] and O [16][HD] (fp32)
  float* wo = reinterpret_cast<float*>(smem);                 // [4][16][HD]
  float* wm = wo + DA_WARPS * 16 * HD;                        // [4][16]
  float* wl = wm + DA_WARPS * 16;                             // [4][16]
  {
    const int r0 = lane >> 2, r1 = r0 + 8, c = (lane & 3) * 2;
    float* base = wo + warp * 16 * HD;
#pragma unroll
    for (int j = 0; j < NT_O; ++j) {
      base[r0 * HD + j * 8 + c] = o[j][0];
      base[r0 * HD + j * 8 + c + 1] = o[j][1];
      base[r1 * HD + j * 8 + c] = o[j][2];
      base[r1 * HD + j * 8 + c + 1] = o[j][3];
    }
    if ((lane & 3) == 0) {
      wm[warp * 16 + r0] = m0;
      wm[warp * 16 + r1] = m1;
      wl[warp * 16 + r0] = l0;
      wl[warp * 16 + r1] = l1;
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < G * HD; idx += DA_WARPS * 32) {
    const int g = idx / HD, d = idx % HD;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < DA_WARPS; ++w) M = fmaxf(M, wm[w * 16 + g]);
    float L = 0.f, O = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < DA_WARPS; ++w) {
        const float mw = wm[w * 16 + g];
        const float f = mw == -INFINITY ? 0.f : exp2f(mw - M);
        L += f * wl[w * 16 + g];
        O += f * wo[(w * 16 + g) * HD + d];
      }
    }
    if (a.n_split == 1) {
      const float inv = L > 0.f ? 1.f / L : 0.f;
      a.out[(int64_t)req * a.out_stride + (int64_t)(kvh * G + g) * HD + d] =
          __float2bfloat16(O * inv);
    } else {
      const int64_t part = ((int64_t)(req * a.hkv + kvh) * a.n_split + split) * G + g;
      a.ws[part * HD + d] = O;
      if (d == 0) {
        float* ml = a.ws + (int64_t)a.n_req * a.hkv * a.n_split * G * HD;
        ml[2 * part] = M;
        ml[2 * part + 1] = L;
      }
    }
  }
}

// merge the splits of every (request, query head): out = sum_s w_s O_s / sum_s w_s l_s
template <int HD>
__global__ void decode_attn_merge_kernel(const DecodeArgs a) {
  pdl_wait();
  pdl_trigger();
  const int req = blockIdx.x, h = blockIdx.y, d = threadIdx.x;
  const int kvh = h / a.G, g = h % a.G;
  const float* ml = a.ws + (int64_t)a.n_req * a.hkv * a.n_split * a.G * HD;
  const int64_t p0 = ((int64_t)(req * a.hkv + kvh) * a.n_split) * a.G + g;
  float M = -INFINITY;
  for (int s = 0; s < a.n_split; ++s) M = fmaxf(M, ml[2 * (p0 + (int64_t)s * a.G)]);
  float L = 0.f, O = 0.f;
  if (M != -INFINITY) {
    for (int s = 0; s < a.n_split; ++s) {
      const int64_t p = p0 + (int64_t)s * a.G;
      const float ms = ml[2 * p];
      const float f = ms == -INFINITY ? 0.f : exp2f(ms - M);
      L += f * ml[2 * p + 1];
      O += f * a.ws[p * HD + d];
    }
  }
  a.out[(int64_t)req * a.out_stride + (int64_t)h * HD + d] =
      __float2bfloat16(L > 0.f ? O / L : 0.f);
}

// Split count: CTAs of one launch run in waves of `slots` (resident CTAs
// per SM x SMs); a wave lasts about (tiles per split + DA_SPLIT_OVH) tile
// times, so pick the split count minimising waves x (tiles/split + OVH).
// (A fixed target of 4 x SMs CTAs left the last wave 44 % full at 40
// requests x 4 KV heads: 0.68 of HBM.)  EMM_DECODE_SPLITS forces a count.
#ifndef DA_SPLIT_OVH
#define DA_SPLIT_OVH 20  // fitted: split counts 4-16 at 40 x 4400 (profiles/r02/decode_split_ab.txt)
#endif
static void decode_plan(int n_req, int hkv, int max_len, int slots, int* n_split,
                        int* tiles_per_split) {
  const int tiles = (max_len + DA_TILE - 1) / DA_TILE;
  const int pairs = n_req * hkv > 0 ? n_req * hkv : 1;
  int max_ns = (tiles + DA_WARPS - 1) / DA_WARPS;  // >= one tile per warp
  if (max_ns < 1) max_ns = 1;
  if (max_ns > 64) max_ns = 64;
  static const int forced = [] {
    const char* e = getenv("EMM_DECODE_SPLITS");
    return e ? atoi(e) : 0;
  }();
  int ns = 1;
  if (forced > 0) {
    ns = forced < max_ns ? forced : max_ns;
  } else {
    long best = -1;
    for (int c = 1; c <= max_ns; ++c) {
      const long tps = (tiles + c - 1) / c;
      const long ctas = (long)pairs * c;
      const long waves = (ctas + slots - 1) / slots;
      const long cost = waves * (tps + DA_SPLIT_OVH);
      if (best < 0 || cost < best) {
        best = cost;
        ns = c;
      }
    }
  }
  int tps = (tiles + ns - 1) / ns;
  ns = tiles > 0 ? (tiles + tps - 1) / tps : 1;
  *n_split = ns;
  *tiles_per_split = tps > 0 ? tps : 1;
}

template <int HD>
constexpr int decode_smem() {
  constexpr int SMEM_TILES = DA_WARPS * DA_STAGES * 2 * DA_TILE * HD * 2;
  constexpr int SMEM_MERGE = (DA_WARPS * 16 * HD + 2 * DA_WARPS * 16) * 4;
  return SMEM_TILES > SMEM_MERGE ? SMEM_TILES : SMEM_MERGE;
}

template <int HD>
static int decode_attr() {
  static bool attr_done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_done[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(decode_attn_kernel<HD>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         decode_smem<HD>());
    if (e != cudaSuccess) return cuda_status(e, "decode attention smem attribute");
    attr_done[dev & 63] = true;
  }
  return EMM_OK;
}

// resident CTAs of the decode kernel on the whole device (per head_dim)
static int decode_slots(int hd) {
  static int cache[2][64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int& c = cache[hd == 128 ? 1 : 0][dev & 63];
  if (c == 0) {
    int n = 0;
    if (hd == 128) {
      if (decode_attr<128>() == EMM_OK)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, decode_attn_kernel<128>, DA_WARPS * 32,
                                                      decode_smem<128>());
    } else {
      if (decode_attr<64>() == EMM_OK)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, decode_attn_kernel<64>, DA_WARPS * 32,
                                                      decode_smem<64>());
    }
    cudaGetLastError();
    c = (n > 0 ? n : 1) * sm_count();
  }
  return c;
}

template <int HD>
static int launch_decode(DecodeArgs& a, int max_len, cudaStream_t st) {
  constexpr int SMEM = decode_smem<HD>();
  const int rc = decode_attr<HD>();
  if (rc != EMM_OK) return rc;
  dim3 grid(a.n_split, a.hkv, a.n_req);
  launch_pdl(decode_attn_kernel<HD>, grid, dim3(DA_WARPS * 32), SMEM, st, a);
  count_launch();
  EMM_CUDA_CHECK_LAUNCH("decode_attn_kernel");
  if (a.n_split > 1) {
    launch_pdl(decode_attn_merge_kernel<HD>, dim3(a.n_req, a.hq), dim3(HD), 0, st, a);
    count_launch();
    EMM_CUDA_CHECK_LAUNCH("decode_attn_merge_kernel");
  }
  (void)max_len;
  return EMM_OK;
}

}  // namespace emm

extern "C" int64_t emm_decode_attention_workspace(int64_t n_req, int hq, int hkv, int hd,
                                                  int64_t max_kv_len) {
  int ns = 1, tps = 1;
  emm::decode_plan((int)n_req, hkv, (int)max_kv_len, emm::decode_slots(hd), &ns, &tps);
  if (ns <= 1) return 0;
  const int64_t G = hkv > 0 ? hq / hkv : 1;
  return n_req * hkv * ns * G * ((int64_t)hd + 2) * (int64_t)sizeof(float);
}

extern "C" int emm_decode_attention_bf16(const void* q, int64_t q_stride, const void* k_plane,
                                         const void* v_plane, int64_t row_stride,
                                         const int32_t* bt, const int64_t* bt_off,
                                         const int32_t* kv_len, int64_t n_req, int hq, int hkv,
                                         int hd, int64_t max_kv_len, void* out,
                                         int64_t out_stride, void* workspace,
                                         int64_t workspace_bytes, float scale, void* stream) {
  if (n_req == 0) return EMM_OK;
  if (!q || !k_plane || !v_plane || !bt || !bt_off || !kv_len || !out || hkv <= 0 ||
      hq % hkv || hq / hkv > 16 || (hd != 64 && hd != 128) || max_kv_len < 1 ||
      (q_stride % 8) || (row_stride % 8)) {
    emm_abi::set_error("emm_decode_attention_bf16: unsupported arguments (head_dim 64/128, "
                       "q heads per kv head <= 16, 16-byte aligned rows, max_kv_len >= 1)");
    return EMM_E_INVALID;
  }
  emm::DecodeArgs a;
  a.q = reinterpret_cast<const __nv_bfloat16*>(q);
  a.q_stride = q_stride;
  a.k = reinterpret_cast<const __nv_bfloat16*>(k_plane);
  a.v = reinterpret_cast<const __nv_bfloat16*>(v_plane);
  a.row_stride = row_stride;
  a.bt = bt;
  a.bt_off = bt_off;
  a.kv_len = kv_len;
  a.out = reinterpret_cast<__nv_bfloat16*>(out);
  a.out_stride = out_stride;
  a.n_req = (int)n_req;
  a.hq = hq;
  a.hkv = hkv;
  a.G = hq / hkv;
  a.scale_log2 = scale * 1.4426950408889634f;
  emm::decode_plan(a.n_req, hkv, (int)max_kv_len, emm::decode_slots(hd), &a.n_split,
                   &a.tiles_per_split);
  a.ws = reinterpret_cast<float*>(workspace);
  if (a.n_split > 1 &&
      (!workspace || workspace_bytes < emm_decode_attention_workspace(n_req, hq, hkv, hd,
                                                                       max_kv_len))) {
    emm_abi::set_error("emm_decode_attention_bf16: workspace too small");
    return EMM_E_INVALID;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  return hd == 128 ? emm::launch_decode<128>(a, (int)max_kv_len, st)
                   : emm::launch_decode<64>(a, (int)max_kv_len, st);
}
