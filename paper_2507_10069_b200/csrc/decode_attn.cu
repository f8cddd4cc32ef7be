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
//  * persistent CTAs (resident slots of the device) over work items (split,
//    kv_head, request): all G = hq/hkv query heads of a KV head share one
//    pass over its rows (GQA: K/V read once, not G times); each request's
//    key range is cut into splits sized from ITS length (the plan is made on
//    the device from kv_len, so a CUDA graph replays it for any lengths):
//    a batch of mixed lengths no longer waits on splits sized for the
//    longest row;
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
//  * warps merge in shared memory; splits merge in a second small kernel
//    (requests with one split are written by the attention kernel itself).
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
  float* ws;               // split partials: O [items_cap][G][hd], (m, l) pairs, plan
  int n_req, hq, hkv, G;
  int items_cap;           // partial slots in ws (>= any plan's item count)
  float scale_log2;
};

// work plan (every CTA derives the same one from kv_len after pdl_wait):
// request r is cut into ns_r = max(1, ceil(tiles_r / tps)) splits of about
// equal size, one item per (split, kv head); the persistent CTAs take items
// round-robin.  tps minimises waves(items) x (largest item + DA_SPLIT_OVH)
// over DA_WARPS * 32 candidates, one per thread.
#ifndef DA_MAX_REQ
#define DA_MAX_REQ 512  // requests per launch (the ABI loops over larger batches)
#endif
#ifndef DA_SPLIT_OVH
#define DA_SPLIT_OVH 40  // per-item cost in tile times (20-60 measured within 1 %, profiles/r02/decode_plan.txt)
#endif
#ifndef DA_PLAN_PREWAIT
#define DA_PLAN_PREWAIT 0  // experiment: plan from kv_len before griddepcontrol.wait
#endif
#ifndef DA_TRIGGER_LATE
#define DA_TRIGGER_LATE 1  // launch dependents after the item loop (measured 1-7 us faster)
#endif
#ifndef DA_MAX_WAVES
#define DA_MAX_WAVES 8  // items_cap = hkv * n_req + DA_MAX_WAVES * grid
#endif

struct DecodePlan {
  int tiles[DA_MAX_REQ];   // 16-key tiles of request r
  int cum[DA_MAX_REQ + 1]; // first split of request r (per kv head); cum[n] = splits
  unsigned long long best;
  int red[DA_WARPS];
};

__device__ __forceinline__ int da_ceil_div(int a, int b) { return (a + b - 1) / b; }

// s.cum / s.tiles for this launch; returns the split count per kv head
__device__ int decode_make_plan(const DecodeArgs& a, DecodePlan& s) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = a.n_req;
  int mx = 0;
  for (int r = tid; r < n; r += DA_WARPS * 32) {
    const int t = da_ceil_div(a.kv_len[r], DA_TILE);
    s.tiles[r] = t;
    mx = max(mx, t);
  }
  if (tid == 0) s.best = ~0ull;
#pragma unroll
  for (int d = 16; d; d >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
  if (lane == 0) s.red[warp] = mx;
  __syncthreads();
  int max_tiles = 0;
#pragma unroll
  for (int w = 0; w < DA_WARPS; ++w) max_tiles = max(max_tiles, s.red[w]);
  // candidate tiles-per-split: the longest request cut into tid + 1 splits
  // (>= DA_WARPS tiles, one per warp)
  constexpr int NC = DA_WARPS * 32;
  auto cand = [&](int c) { return max(min(max_tiles, DA_WARPS), da_ceil_div(max_tiles, c + 1)); };
  int tps = max(cand(tid), 1);
  {
    // ns = ceil(t / tps) through a float reciprocal (+ exact correction):
    // an integer division per request and candidate costs ~10 us at 512
    long long splits = 0;
    int longest = 1;
    const float inv = 1.0f / (float)tps;
    for (int r = 0; r < n; ++r) {
      const int t = s.tiles[r];
      int ns = (int)ceilf((float)t * inv);
      ns += (ns * tps < t) - ((ns - 1) * tps >= t && ns > 1);
      splits += ns > 1 ? ns : 1;
      longest = max(longest, t);
    }
    const int big = min(tps, longest);  // the largest item (splits are even, <= tps)
    const long long items = splits * a.hkv;
    if (items <= a.items_cap) {
      const long long waves = (items + gridDim.x - 1) / gridDim.x;
      const unsigned long long cost = (unsigned long long)(waves * (big + DA_SPLIT_OVH));
      atomicMin(&s.best, (cost << 24) | ((unsigned long long)tid << 12));
    }
  }
  __syncthreads();
  // the winner's tps (ties -> the largest tps: fewest items)
  tps = s.best == ~0ull ? max(max_tiles, 1) : max(cand((int)((s.best >> 12) & 0xFFF)), 1);
  // prefix sum of ns_r over requests (each thread a run of consecutive r)
  constexpr int PER = DA_MAX_REQ / NC > 0 ? DA_MAX_REQ / NC : 1;
  int loc[PER];
  int run = 0;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int r = tid * PER + k;
    const int t = r < n ? s.tiles[r] : 0;
    loc[k] = r < n ? (t > tps ? da_ceil_div(t, tps) : 1) : 0;
    run += loc[k];
  }
  int inc = run;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += o;
  }
  __syncthreads();  // s.red reuse
  if (lane == 31) s.red[warp] = inc;
  __syncthreads();
  int base = inc - run;
  for (int w = 0; w < warp; ++w) base += s.red[w];
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int r = tid * PER + k;
    if (r < n) s.cum[r] = base;
    base += loc[k];
  }
  int total = 0;
#pragma unroll
  for (int w = 0; w < DA_WARPS; ++w) total += s.red[w];
  if (tid == 0) s.cum[n] = total;
  __syncthreads();
  return total;
}

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
  __shared__ DecodePlan plan;
#if DA_PLAN_PREWAIT
  const int splits = decode_make_plan(a, plan);
#endif
  pdl_wait();  // launched with programmatic serialization: inputs are ready after this
#if !DA_TRIGGER_LATE
  pdl_trigger();
#endif
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.G;
#if !DA_PLAN_PREWAIT
  const int splits = decode_make_plan(a, plan);
#endif
  if (blockIdx.x == 0) {  // the merge kernel reads the plan
    int* wplan = reinterpret_cast<int*>(a.ws + (int64_t)a.items_cap * G * (HD + 2));
    for (int r = threadIdx.x; r <= a.n_req; r += DA_WARPS * 32) wplan[r] = plan.cum[r];
  }
  const int n_items = splits * a.hkv;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
  const int p = item / a.hkv, kvh = item - p * a.hkv;
  int req = 0;
  {  // last r with cum[r] <= p
    int lo = 0, hi = a.n_req - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (plan.cum[mid] <= p) lo = mid; else hi = mid - 1;
    }
    req = lo;
  }
  const int ns = plan.cum[req + 1] - plan.cum[req];
  const int split = p - plan.cum[req];
  const int len = a.kv_len[req];
  const int64_t bt0 = a.bt_off[req];
  const int n_tiles_all = plan.tiles[req];
  const int per = ns > 1 ? da_ceil_div(n_tiles_all, ns) : n_tiles_all;
  const int t_begin = split * per;
  int t_end = t_begin + per;
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
    if (ns == 1) {
      const float inv = L > 0.f ? 1.f / L : 0.f;
      a.out[(int64_t)req * a.out_stride + (int64_t)(kvh * G + g) * HD + d] =
          __float2bfloat16(O * inv);
    } else {
      const int64_t part = (int64_t)item * G + g;
      a.ws[part * HD + d] = O;
      if (d == 0) {
        float* ml = a.ws + (int64_t)a.items_cap * G * HD;
        ml[2 * part] = M;
        ml[2 * part + 1] = L;
      }
    }
  }
  __syncthreads();  // the next item's ring overwrites the merge area
  }
#if DA_TRIGGER_LATE
  pdl_trigger();
#endif
}

// merge the splits of every (request, query head): out = sum_s w_s O_s / sum_s w_s l_s
template <int HD>
__global__ void decode_attn_merge_kernel(const DecodeArgs a) {
  pdl_wait();
  pdl_trigger();
  const int req = blockIdx.x, h = blockIdx.y, d = threadIdx.x;
  const int kvh = h / a.G, g = h % a.G;
  const int* wplan = reinterpret_cast<const int*>(a.ws + (int64_t)a.items_cap * a.G * (HD + 2));
  const int c0 = wplan[req], ns = wplan[req + 1] - c0;
  if (ns <= 1) return;  // written by the attention kernel itself
  const float* ml = a.ws + (int64_t)a.items_cap * a.G * HD;
  // item of split s = (c0 + s) * hkv + kvh; partial row = item * G + g
  const int64_t p0 = ((int64_t)c0 * a.hkv + kvh) * a.G + g;
  const int64_t step = (int64_t)a.hkv * a.G;
  float M = -INFINITY;
  for (int s = 0; s < ns; ++s) M = fmaxf(M, ml[2 * (p0 + s * step)]);
  float L = 0.f, O = 0.f;
  if (M != -INFINITY) {
    for (int s = 0; s < ns; ++s) {
      const int64_t p = p0 + s * step;
      const float ms = ml[2 * p];
      const float f = ms == -INFINITY ? 0.f : exp2f(ms - M);
      L += f * ml[2 * p + 1];
      O += f * a.ws[p * HD + d];
    }
  }
  a.out[(int64_t)req * a.out_stride + (int64_t)h * HD + d] =
      __float2bfloat16(L > 0.f ? O / L : 0.f);
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
static int launch_decode(DecodeArgs& a, int grid, cudaStream_t st) {
  constexpr int SMEM = decode_smem<HD>();
  const int rc = decode_attr<HD>();
  if (rc != EMM_OK) return rc;
  launch_pdl(decode_attn_kernel<HD>, dim3(grid), dim3(DA_WARPS * 32), SMEM, st, a);
  count_launch();
  EMM_CUDA_CHECK_LAUNCH("decode_attn_kernel");
  launch_pdl(decode_attn_merge_kernel<HD>, dim3(a.n_req, a.hq), dim3(HD), 0, st, a);
  count_launch();
  EMM_CUDA_CHECK_LAUNCH("decode_attn_merge_kernel");
  return EMM_OK;
}

// persistent grid and partial-slot capacity of one launch of <= DA_MAX_REQ requests
static void decode_grid(int n_req, int hkv, int hd, int* grid, int* items_cap) {
  const int slots = decode_slots(hd);
  const int most = n_req * hkv * 64;  // never more CTAs than a 64-way split could feed
  *grid = slots < most ? slots : (most > 0 ? most : 1);
  *items_cap = hkv * n_req + DA_MAX_WAVES * *grid;
}

static int64_t decode_ws_bytes(int n_req, int hq, int hkv, int hd) {
  int grid = 0, cap = 0;
  decode_grid(n_req, hkv, hd, &grid, &cap);
  const int64_t G = hq / hkv;
  return (int64_t)cap * G * (hd + 2) * (int64_t)sizeof(float) +
         (int64_t)(n_req + 1) * (int64_t)sizeof(int);
}

}  // namespace emm

extern "C" int64_t emm_decode_attention_workspace(int64_t n_req, int hq, int hkv, int hd,
                                                  int64_t max_kv_len) {
  (void)max_kv_len;  // the plan is made on the device from kv_len
  if (n_req <= 0 || hkv <= 0) return 0;
  const int chunk = n_req < DA_MAX_REQ ? (int)n_req : DA_MAX_REQ;
  return emm::decode_ws_bytes(chunk, hq, hkv, hd);
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
  if (!workspace || workspace_bytes < emm_decode_attention_workspace(n_req, hq, hkv, hd,
                                                                     max_kv_len)) {
    emm_abi::set_error("emm_decode_attention_bf16: workspace too small");
    return EMM_E_INVALID;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // batches beyond DA_MAX_REQ requests: consecutive launches over request
  // ranges (stream-ordered, so they can share the workspace)
  for (int64_t r0 = 0; r0 < n_req; r0 += DA_MAX_REQ) {
    const int n = (int)(n_req - r0 < DA_MAX_REQ ? n_req - r0 : DA_MAX_REQ);
    emm::DecodeArgs a;
    a.q = reinterpret_cast<const __nv_bfloat16*>(q) + r0 * q_stride;
    a.q_stride = q_stride;
    a.k = reinterpret_cast<const __nv_bfloat16*>(k_plane);
    a.v = reinterpret_cast<const __nv_bfloat16*>(v_plane);
    a.row_stride = row_stride;
    a.bt = bt;
    a.bt_off = bt_off + r0;
    a.kv_len = kv_len + r0;
    a.out = reinterpret_cast<__nv_bfloat16*>(out) + r0 * out_stride;
    a.out_stride = out_stride;
    a.n_req = n;
    a.hq = hq;
    a.hkv = hkv;
    a.G = hq / hkv;
    a.scale_log2 = scale * 1.4426950408889634f;
    a.ws = reinterpret_cast<float*>(workspace);
    int grid = 0;
    emm::decode_grid(n, hkv, hd, &grid, &a.items_cap);
    const int rc = hd == 128 ? emm::launch_decode<128>(a, grid, st)
                             : emm::launch_decode<64>(a, grid, st);
    if (rc != EMM_OK) return rc;
  }
  return EMM_OK;
}
