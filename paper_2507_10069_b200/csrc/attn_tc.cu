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

#include <map>
#include <mutex>
#include <utility>

#include "../../include/emm.h"
#include "ptx.cuh"
#include "runtime.h"

namespace emm {

constexpr int ATT_THREADS = 384;
constexpr int ATT_BM = 128;  // query rows per tile (2 tiles per CTA)
constexpr int ATT_BN = 128;  // kv rows per block
constexpr float ATT_RESCALE_THRESH = 8.0f;  // log2 units: p <= 256 between rescales
#ifndef ATT_POLY_MODE
// which exp2 PAIRS (pair i of 32-column chunk c, 16 pairs per chunk) run as a
// degree-3 polynomial on the FMA pipe instead of MUFU.EX2 (FA4's split):
//   0 none; 1 pairs i % 8 == 7 of chunks 1-2 (1/16 of the scores);
//   2 pairs i % 8 >= 6 of chunks 1-2 (1/8, FA4's hd-128 pattern);
//   3 pairs i % 8 == 7 of every chunk (1/8)
// (ATT_POLY_FROM below selects by column and can only express 1/4 steps:
//  the column index of a pair is even)
#define ATT_POLY_MODE 0
#endif
__host__ __device__ constexpr bool att_poly_pair(int c, int i) {
  return ATT_POLY_MODE == 1   ? ((c == 1 || c == 2) && (i & 7) == 7)
         : ATT_POLY_MODE == 2 ? ((c == 1 || c == 2) && (i & 7) >= 6)
         : ATT_POLY_MODE == 3 ? ((i & 7) == 7)
                              : false;
}
#ifndef ATT_POLY_FROM
// exp2 of score columns i with (i & 7) >= ATT_POLY_FROM runs as a degree-3
// polynomial on the FMA pipe instead of MUFU.EX2 (FA4's split of the 16/clk/SM
// MUFU against the FMA pipe).  8 = all MUFU: measured fastest here (tools/
// attn_bench.py: 6 -> 972, 8 -> 1058 TF/s on the Qwen GQA shape), because the
// softmax warp is issue-bound, not MUFU-bound, once FFMA2 packs the math.
#define ATT_POLY_FROM 8
#endif

#ifndef ATT_POLY_DEG
#define ATT_POLY_DEG 3
#endif

#ifndef ATT_PROF
#define ATT_PROF 0  // 1: per-phase clock64() totals (tools/attn_prof.py; a separate build)
#endif
#if ATT_PROF
__device__ unsigned long long g_att_prof[16];
#define PROF_T(v) const long long v = clock64()
#define PROF_ADD(i, a, b) prof[i] += (unsigned long long)((b) - (a))
#else
#define PROF_T(v)
#define PROF_ADD(i, a, b)
#endif

#ifndef ATT_P_SPLIT
#define ATT_P_SPLIT 2  // P handed to the PV MMAs in parts of 128 / ATT_P_SPLIT keys
#endif
#ifndef ATT_SUM_LATE
#define ATT_SUM_LATE 0  // row sum of P after P is handed to the MMA warp
#endif
#ifndef ATT_SEQ
#define ATT_SEQ 0  // the two softmax warpgroups take turns in the exp2 phase
#endif
#ifndef ATT_PACK_ALU
// 1: P packed to bf16 pairs on the ALU pipe (round-half-up add + PRMT of the
// high halves) instead of F2FP; p >= 0 and finite, so the add cannot carry
// into the sign bit
#define ATT_PACK_ALU 0
#endif
#ifndef ATT_WAIT_SLEEP
// 1: the softmax warps wait for S / O with a suspend-time hint (parked, no
// spin) so they leave the issue slots to the other tile's exponentials
#define ATT_WAIT_SLEEP 0
#endif
#if ATT_WAIT_SLEEP >= 2
#define mbar_wait mbar_wait_sleep  // every wait of the kernels (TMA, MMA, softmax)
#endif
#if ATT_WAIT_SLEEP
#define ATT_SM_WAIT mbar_wait_sleep
#else
#define ATT_SM_WAIT mbar_wait
#endif
#ifndef ATT1_PROF
#define ATT1_PROF 0  // 1: per-phase clock64() totals of the single-tile kernel (tools/attn1_prof.py)
#endif
#if ATT1_PROF
#if !ATT_PROF
__device__ unsigned long long g_att_prof[16];
#endif
#define PROF1_T(v) const long long v = clock64()
#define PROF1_ADD(i, a, b) prof1[i] += (unsigned long long)((b) - (a))
#else
#define PROF1_T(v)
#define PROF1_ADD(i, a, b)
#endif
#ifndef ATT1_POLY_FROM
#define ATT1_POLY_FROM 8  // single-tile kernel: same knob (throughput-bound there)
#endif

struct AttnArgs {
  // [n_tiles][5] = seq, q head, first q tile (of a pair), first / end KV block
  const int32_t* tiles;
  int n_tiles;
  const int2* row_bounds;  // optional per q row [lo, hi) visible KV positions
  const int32_t* q_start;
  const int32_t* q_len;
  const int32_t* kv_start;
  const int32_t* kv_len;
  __nv_bfloat16* out;
  int64_t out_tok_stride;  // elements
  int n_q_heads, group;    // group = n_q_heads / n_kv_heads
  float scale_log2;        // softmax scale * log2(e)
  int causal;
  // optional [next, done] work-queue counters (pair kernel): items are handed
  // out longest-first to whichever CTA asks next instead of round-robin
  int* sched;
};

// head_dim = CH x 64 (SW128 chunks, 16 KiB per 128 rows) + REM (0 or 16: one
// SW32 chunk of 4 KiB; head_dim 80 of the Qwen2.5-VL vision tower).
template <int HD>
struct AttnCfg {
  static constexpr int CH = HD / 64;               // 64-element SW128 chunks per row
  static constexpr int REM = HD % 64;              // SW32 tail (0 or 16 elements)
  static_assert(REM == 0 || REM == 16, "head_dim must be 64k or 64k + 16");
  static constexpr int TILE_BYTES = 128 * HD * 2;  // one 128-row bf16 tile
  // K is consumed a block earlier than V (S_{j+1} is issued right after PV_j),
  // so it gets the deeper ring; K stages are released after the S MMAs, V
  // stages after the PV MMAs.
  static constexpr int KS = 3, VS = 2;
  static constexpr int Q_OFF = 0;                  // Q0, Q1
  static constexpr int K_OFF = 2 * TILE_BYTES;
  static constexpr int V_OFF = K_OFF + KS * TILE_BYTES;
  static constexpr int BAR_OFF = V_OFF + VS * TILE_BYTES;
  // q_full, q_empty, k_full[KS], k_empty[KS], v_full[VS], v_empty[VS],
  // s_full[2], p_full[2 tiles x 4 parts], o_done[2], o_free[2],
  // sched_full[4], sched_empty[4]
  static constexpr int N_BARS = 2 + 2 * KS + 2 * VS + 14 + 8;
  // P is handed to the PV MMAs in NP parts (the PV of the first keys runs
  // while the softmax warps exponentiate the rest): head_dim 64 / 128 only
  // (at 80 the shorter PV MMAs do not pay for the extra waits: measured)
  static constexpr int NP = REM ? 1 : ATT_P_SPLIT;
  // + TMEM slot (16 B) + the 4 item ids of the scheduling ring (16 B)
  static constexpr int SMEM = BAR_OFF + N_BARS * 8 + 32 + 1024;
};

// named barriers 1 / 2 between the two softmax warpgroups (256 threads)
__device__ __forceinline__ void named_bar_sync(int id) {
  asm volatile("bar.sync %0, 256;" ::"r"(id) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id) {
  asm volatile("bar.arrive %0, 256;" ::"r"(id) : "memory");
}

__device__ __forceinline__ uint32_t pack_p(float a, float b) {
#if ATT_PACK_ALU
  const uint32_t ua = __float_as_uint(a) + 0x8000u, ub = __float_as_uint(b) + 0x8000u;
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(d) : "r"(ua), "r"(ub));
  return d;
#else
  return pack_bf16(a, b);
#endif
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// packed fp32 pairs (FFMA2 / FADD2 on sm_100: two lanes of math per issue)
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n .reg .b64 ra, rb, rc, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
      " mov.b64 rc, {%6, %7};\n fma.rn.f32x2 rd, ra, rb, rc;\n mov.b64 {%0, %1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{\n .reg .b64 ra, rb, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
      " add.rn.f32x2 rd, ra, rb;\n mov.b64 {%0, %1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}

// 2^x of a pair on the FMA pipe: x = j + f (j = round(x), |f| <= 1/2), 2^f by
// a degree-3 minimax polynomial (max rel. error 7.5e-5, far below bf16's
// 3.9e-3), 2^j added to the exponent bits.  x >= -126 (clamped here: the
// exponent add must not wrap).
__device__ __forceinline__ float2 poly_exp2x2(float2 x) {
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);  // 1.5 * 2^23
  const float2 t = fadd2(x, magic);  // round-to-nearest integer in the low mantissa bits
  const float2 jf = fadd2(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = ffma2(jf, make_float2(-1.f, -1.f), x);
#if ATT_POLY_DEG == 2
  // quadratic (rel. error ~1.7e-3, below bf16 P's 3.9e-3 spacing)
  float2 p = ffma2(make_float2(0.2402265f, 0.2402265f), f,
                   make_float2(0.6931472f, 0.6931472f));
  p = ffma2(p, f, make_float2(1.0f, 1.0f));
#else
  float2 p = ffma2(make_float2(0.055171321434035504f, 0.055171321434035504f), f,
                   make_float2(0.24261054228171025f, 0.24261054228171025f));
  p = ffma2(p, f, make_float2(0.6932609856052558f, 0.6932609856052558f));
  p = ffma2(p, f, make_float2(0.9999281093641538f, 0.9999281093641538f));
#endif
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
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
  constexpr int KS = Cfg::KS, VS = Cfg::VS;
  uint64_t* q_full = bars;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;
  uint64_t* k_empty = k_full + KS;
  uint64_t* v_full = k_empty + KS;
  uint64_t* v_empty = v_full + VS;
  uint64_t* s_full = v_empty + VS;
  uint64_t* p_full = s_full + 2;  // [4 * tile + part]
  uint64_t* o_done = p_full + 8;
  uint64_t* o_free = o_done + 2;
  uint64_t* sched_full = o_free + 2;   // [4] item id published
  uint64_t* sched_empty = sched_full + 4;  // [4] read by the MMA thread + 8 softmax warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + Cfg::N_BARS);
  volatile int* sched_ids = reinterpret_cast<volatile int*>(tmem_slot + 4);

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
    for (int i = 0; i < KS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < VS; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      for (int q = 0; q < 4; ++q) mbar_init(&p_full[4 * i + q], 4);
      mbar_init(&o_done[i], 1);
      mbar_init(&o_free[i], 4);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&sched_full[i], 1);
      mbar_init(&sched_empty[i], 9);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  // register split (setmaxnreg inside each role's branch): the producer / MMA
  // warpgroup drops to 120, the two softmax warpgroups (a 128-score row +
  // packing per thread) rise to 192 (128 x 120 + 256 x 192 = 384 x 168)
  // every role walks the same item sequence; g counts KV blocks across items
  if (warp == 0) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 120;");
    if (lane == 0) {
      // ------------------------------------------------------------- TMA
      int g = 0;
      for (int it = 0;; ++it) {
        // this CTA's next work item, published to the MMA / softmax roles
        // through a 4-deep ring: round-robin, or (a.sched) the next one of
        // the longest-first list whichever CTA gets there first
        int item = !a.sched ? blockIdx.x + it * gridDim.x
                   : it == 0 ? blockIdx.x
                             : gridDim.x + atomicAdd(a.sched, 1);
        if (item >= a.n_tiles) item = -1;
        mbar_wait(&sched_empty[it & 3], ((it >> 2) & 1) ^ 1);
        sched_ids[it & 3] = item;
        mbar_arrive(&sched_full[it & 3]);
        if (item < 0) break;
        const int seq = a.tiles[5 * item], head = a.tiles[5 * item + 1],
                  qt0 = a.tiles[5 * item + 2], blk0 = a.tiles[5 * item + 3];
        const int kvh = head / a.group;
        const int q0 = a.q_start[seq] + qt0 * ATT_BM, kv0 = a.kv_start[seq] + blk0 * ATT_BN;
        const int nblk = a.tiles[5 * item + 4] - blk0;
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
        // K runs one block ahead of V: K0 K1 V0 K2 V1 ... V_{n-1}
        auto load_k = [&](int jj) {
          const int gg = g + jj, st = gg % KS;
          mbar_wait(&k_empty[st], ((gg / KS) & 1) ^ 1);
          mbar_arrive_expect_tx(&k_full[st], Cfg::TILE_BYTES);
          for (int c = 0; c < Cfg::CH; ++c)
            tma_load_3d(smem + Cfg::K_OFF + st * Cfg::TILE_BYTES + c * 16384, &tmK, &k_full[st],
                        c * 64, kvh, kv0 + jj * ATT_BN);
          if (Cfg::REM)
            tma_load_3d(smem + Cfg::K_OFF + st * Cfg::TILE_BYTES + Cfg::CH * 16384, &tmKr,
                        &k_full[st], Cfg::CH * 64, kvh, kv0 + jj * ATT_BN);
        };
        auto load_v = [&](int jj) {
          const int gg = g + jj, st = gg % VS;
          mbar_wait(&v_empty[st], ((gg / VS) & 1) ^ 1);
          mbar_arrive_expect_tx(&v_full[st], Cfg::TILE_BYTES);
          for (int c = 0; c < Cfg::CH; ++c)
            tma_load_3d(smem + Cfg::V_OFF + st * Cfg::TILE_BYTES + c * 16384, &tmV, &v_full[st],
                        c * 64, kvh, kv0 + jj * ATT_BN);
          if (Cfg::REM)
            tma_load_3d(smem + Cfg::V_OFF + st * Cfg::TILE_BYTES + Cfg::CH * 16384, &tmVr,
                        &v_full[st], Cfg::CH * 64, kvh, kv0 + jj * ATT_BN);
        };
        for (int j = 0; j < nblk; ++j) {
          load_k(j);
          if (j) load_v(j - 1);
        }
        load_v(nblk - 1);
        g += nblk;
      }
    }
  } else if (warp == 1) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 120;");
    if (lane == 0) {
      // ------------------------------------------------------------- MMA
      constexpr uint32_t idesc_s = idesc_bf16_f32(128, ATT_BN, false, false);
      constexpr uint32_t idesc_o = idesc_bf16_f32(128, Cfg::CH * 64, false, true);
      constexpr uint32_t idesc_or = idesc_bf16_f32(128, 16, false, true);
      const uint32_t q_addr = smem_u32(smem + Cfg::Q_OFF);
      auto issue_s = [&](int t, int g) {  // S_t = Q_t K_g^T into TMEM [t*128, +128)
        const uint32_t k_addr = smem_u32(smem + Cfg::K_OFF + (g % KS) * Cfg::TILE_BYTES);
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
      // O_t += P_t V_g over keys [16 kk0, 16 kk1), P_t from TMEM
      auto issue_pv = [&](int t, int g, bool first, int kk0, int kk1) {
        const uint32_t v_addr = smem_u32(smem + Cfg::V_OFF + (g % VS) * Cfg::TILE_BYTES);
        const uint32_t o_addr = tbase + 256 + t * 128;
#pragma unroll
        for (int kk = kk0; kk < kk1; ++kk) {
          const uint64_t bdesc = desc_sw128_mnmajor(v_addr + kk * 2048, 16384);
          mma_ts(o_addr, tbase + t * 128 + kk * 8, bdesc, idesc_o, (!first) || kk != 0);
          if (Cfg::REM)  // O columns [CH*64, HD) from the SW32 tail of V
            mma_ts(o_addr + Cfg::CH * 64, tbase + t * 128 + kk * 8,
                   desc_sw32_mnmajor(v_addr + Cfg::CH * 16384 + kk * 512), idesc_or,
                   (!first) || kk != 0);
        }
      };
#if ATT_PROF
      unsigned long long prof[16] = {0};
#endif
      int g = 0;
      for (int it = 0;; ++it) {
        mbar_wait(&sched_full[it & 3], (it >> 2) & 1);
        const int item = sched_ids[it & 3];
        mbar_arrive(&sched_empty[it & 3]);
        if (item < 0) break;
        const int nblk = a.tiles[5 * item + 4] - a.tiles[5 * item + 3];
        mbar_wait(q_full, it & 1);
        mbar_wait(&k_full[g % KS], (g / KS) & 1);
        tc_fence_after();
        issue_s(0, g);
        issue_s(1, g);
        mma_commit(&k_empty[g % KS]);  // K_g free once both S MMAs are done
        if (nblk == 1) mma_commit(q_empty);
        for (int j = 0; j < nblk; ++j, ++g) {
          const bool more = j + 1 < nblk;
          PROF_T(m0);
          mbar_wait(&v_full[g % VS], (g / VS) & 1);
          PROF_T(m1);
          PROF_ADD(8, m0, m1);
          for (int t = 0; t < 2; ++t) {
            PROF_T(m2);
            if (j == 0) mbar_wait(&o_free[t], (it & 1) ^ 1);  // epilogue of the last item read O
#pragma unroll
            for (int q = 0; q < Cfg::NP; ++q) {  // PV of each part as soon as it is in TMEM
              mbar_wait(&p_full[4 * t + q], g & 1);
              if (q == Cfg::NP - 1) {
                PROF_T(m3);
                PROF_ADD(9, m2, m3);
              }
              tc_fence_after();
              issue_pv(t, g, j == 0, q * (ATT_BN / 16) / Cfg::NP, (q + 1) * (ATT_BN / 16) / Cfg::NP);
            }
            mma_commit(&o_done[t]);
            if (more) {
              if (t == 0) {
                PROF_T(m4);
                mbar_wait(&k_full[(g + 1) % KS], ((g + 1) / KS) & 1);
                tc_fence_after();
                PROF_T(m5);
                PROF_ADD(10, m4, m5);
              }
              issue_s(t, g + 1);  // in-order: reads P_t before S_t is overwritten
            }
          }
          if (more) mma_commit(&k_empty[(g + 1) % KS]);
          if (more && j + 2 == nblk) mma_commit(q_empty);  // last S of the item issued
          mma_commit(&v_empty[g % VS]);
        }
      }
#if ATT_PROF
      atomicAdd(&g_att_prof[8], prof[8]);
      atomicAdd(&g_att_prof[9], prof[9]);
      atomicAdd(&g_att_prof[10], prof[10]);
#endif
    }
  } else if (warp >= 4) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 192;");
#if ATT_PROF
    unsigned long long prof[8] = {0};
#endif
    // ------------------------------------------------------------- softmax
    const int t = (warp - 4) >> 2;               // tile of this warpgroup
    const int ew = warp & 3;                     // TMEM lane quarter
    const int r = ew * 32 + lane;                // query row in the tile
    const uint32_t lane_off = (uint32_t)(ew * 32) << 16;
    const uint32_t t_s = tbase + lane_off + t * 128;
    const uint32_t t_o = tbase + lane_off + 256 + t * 128;
    // per-item metadata one item ahead (see attn_fwd_tc1_kernel): the
    // dependent loads tile entry -> q_start / lengths -> row bounds overlap
    // the current item instead of opening the next one
    struct Meta {
      int seq, head, qt0, blk0, nblk, q_len, q0, lo, hi;
    };
    auto load_meta = [&](int item) {
      Meta m{};
      if (item >= a.n_tiles) return m;
      m.seq = a.tiles[5 * item];
      m.head = a.tiles[5 * item + 1];
      m.qt0 = a.tiles[5 * item + 2];
      m.blk0 = a.tiles[5 * item + 3];
      m.nblk = a.tiles[5 * item + 4] - m.blk0;
      m.q_len = a.q_len[m.seq];
      const int kv_len = a.kv_len[m.seq];
      m.q0 = a.q_start[m.seq];
      const int qrow = (m.qt0 + t) * ATT_BM + r;
      // visible keys of this row: positions [lo, hi) of the sequence's KV
      m.lo = 0;
      m.hi = kv_len;
      if (a.row_bounds) {
        if (qrow < m.q_len) {
          const int2 b = a.row_bounds[m.q0 + qrow];
          m.lo = b.x;
          m.hi = b.y;
        } else {
          m.hi = 0;
        }
      } else if (a.causal) {
        m.hi = min(kv_len - m.q_len + qrow + 1, kv_len);  // queries end the KV sequence
      }
      return m;
    };
    int g = 0;
    for (int it = 0;; ++it) {
      mbar_wait(&sched_full[it & 3], (it >> 2) & 1);
      const int item = sched_ids[it & 3];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sched_empty[it & 3]);
      if (item < 0) break;
      const Meta cur = load_meta(item);
      const int head = cur.head, qt0 = cur.qt0, blk0 = cur.blk0;
      const int q_len = cur.q_len, nblk = cur.nblk, lo = cur.lo, hi = cur.hi;
      const int qrow = (qt0 + t) * ATT_BM + r;   // query index within the sequence
      float m_used = -INFINITY, l_run = 0.f;
      for (int j = 0; j < nblk; ++j, ++g) {
        PROF_T(c0);
        ATT_SM_WAIT(&s_full[t], g & 1);
        tc_fence_after();
        PROF_T(c1);
        PROF_ADD(0, c0, c1);
        const int kbase = (blk0 + j) * ATT_BN;
        // the whole 128-score row in registers: one TMEM read of S per block
        uint32_t v[ATT_BN];
#pragma unroll
        for (int c = 0; c < ATT_BN / 32; ++c)
          tmem_ld32(t_s + c * 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32 * c));
        tmem_wait_ld();
        PROF_T(c2);
        PROF_ADD(1, c1, c2);
        // interior blocks (every key visible to every row of this warp) skip masking
        const bool full = __all_sync(0xffffffffu, kbase >= lo && kbase + ATT_BN <= hi);
        if (!full) {
#pragma unroll
          for (int i = 0; i < ATT_BN; ++i) {
            const int kp = kbase + i;
            if (kp < lo || kp >= hi) v[i] = __float_as_uint(-INFINITY);
          }
        }
        float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
        for (int i = 0; i < ATT_BN; i += 4) {
          mx0 = fmaxf(mx0, __uint_as_float(v[i]));
          mx1 = fmaxf(mx1, __uint_as_float(v[i + 1]));
          mx2 = fmaxf(mx2, __uint_as_float(v[i + 2]));
          mx3 = fmaxf(mx3, __uint_as_float(v[i + 3]));
        }
        // scale > 0 commutes with max
        const float mx = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3)) * a.scale_log2;
        PROF_T(c2b);
        PROF_ADD(7, c2, c2b);
        // lazy rescale: O and l only when the running max grew by > 2^8
        const bool grow = mx > m_used + ATT_RESCALE_THRESH;
        if (j == 0) {
          m_used = mx;
        } else if (__any_sync(0xffffffffu, grow)) {
          // S_t's commit covers PV_{j-1}: O_t is complete here
          const float m_new = grow ? mx : m_used;
          // (a row still fully masked keeps m = -inf: alpha must be 1, not exp2(NaN))
          const float alpha = m_new == m_used ? 1.f : fast_exp2(m_used - m_new);
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
        PROF_T(c3);
        PROF_ADD(2, c2, c3);
        // fully masked rows (m = -inf) produce p = 0 everywhere
        const float nbase = m_used == -INFINITY ? 0.f : -m_used;
        const float sc = a.scale_log2;
        // p = exp2(s*scale - m) -> bf16 pairs over the first 64 columns (P aliases S);
        // pairs of columns go through packed FFMA2 / FADD2
        const float2 sc2 = make_float2(sc, sc), nb2 = make_float2(nbase, nbase);
        float2 rsa = make_float2(0.f, 0.f), rsb = make_float2(0.f, 0.f);
        // tile 0 goes first; tile 1 waits for tile 0's exp phase of this block,
        // tile 0 for tile 1's of the previous block
        if (ATT_SEQ && (t == 1 || g > 0)) named_bar_sync(1 + t);
#pragma unroll
        for (int c = 0; c < ATT_BN / 32; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int e = 32 * c + 2 * i;
            const float2 x = ffma2(make_float2(__uint_as_float(v[e]), __uint_as_float(v[e + 1])),
                                   sc2, nb2);
            float2 pp;
            if ((e & 7) >= ATT_POLY_FROM || att_poly_pair(c, i)) {
              pp = poly_exp2x2(x);
            } else {
              pp.x = fast_exp2(x.x);
              pp.y = fast_exp2(x.y);
            }
            if (ATT_SUM_LATE) {
              v[e] = __float_as_uint(pp.x);
              v[e + 1] = __float_as_uint(pp.y);
            } else if (i & 1) {
              rsb = fadd2(rsb, pp);
            } else {
              rsa = fadd2(rsa, pp);
            }
            pk[i] = pack_p(pp.x, pp.y);
          }
          tmem_st16(t_s + c * 16, pk);
          constexpr int CPP = (ATT_BN / 32) / Cfg::NP;  // 32-key chunks per P part
          if ((c + 1) % CPP == 0 && c + 1 < ATT_BN / 32) {  // part c / CPP is in TMEM
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[4 * t + c / CPP]);
          }
        }
        if (ATT_SEQ) named_bar_arrive(2 - t);
        PROF_T(c4);
        PROF_ADD(3, c3, c4);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[4 * t + Cfg::NP - 1]);
        if (ATT_SUM_LATE) {  // off the P -> PV critical path
#pragma unroll
          for (int e = 0; e < ATT_BN; e += 4) {
            rsa = fadd2(rsa, make_float2(__uint_as_float(v[e]), __uint_as_float(v[e + 1])));
            rsb = fadd2(rsb, make_float2(__uint_as_float(v[e + 2]), __uint_as_float(v[e + 3])));
          }
        }
        l_run += (rsa.x + rsa.y) + (rsb.x + rsb.y);
        PROF_T(c5);
        PROF_ADD(4, c4, c5);
        PROF_ADD(6, 0, 1);
      }
      PROF_T(e0);
      // epilogue: O / l -> bf16, then hand O back to the MMA warp
      ATT_SM_WAIT(&o_done[t], (g - 1) & 1);
      tc_fence_after();
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      const bool ok = qrow < q_len;
      __nv_bfloat16* orow = a.out + (int64_t)(cur.q0 + qrow) * a.out_tok_stride +
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
      PROF_T(e1);
      PROF_ADD(5, e0, e1);
    }
    if (ATT_SEQ && t == 0 && g > 0) named_bar_sync(1);  // tile 1's last arrive
#if ATT_PROF
    if (lane == 0)
      for (int i = 0; i < 8; ++i) atomicAdd(&g_att_prof[i], prof[i]);
#endif
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 120;");  // warps 2, 3
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
  // the last CTA out resets the work queue for the next launch on this
  // stream (every CTA has fetched its final, out-of-range item by now)
  if (a.sched && threadIdx.x == 0 && atomicAdd(a.sched + 1, 1) == (int)gridDim.x - 1) {
    a.sched[0] = 0;
    a.sched[1] = 0;
    __threadfence();
  }
}

// ---------------------------------------------------------------------------
// Single-tile variant: one 128-query tile per work item, S double-buffered in
// TMEM (S_a cols [0,128), S_b [128,256), O [256, 256+HD)), so the tensor pipe
// computes S(j+2) while the softmax works on block j+1 and PV(j) runs as soon as
// P(j) is published: the softmax is off the MMA's critical path and the kernel
// becomes throughput-bound (MUFU / issue vs tensor) instead of latency-bound.
//   warp 0 TMA (Q once per item, K ring KS=3, V ring VS=3), warp 1 MMA,
//   warp 2 TMEM alloc, warps 4..7 softmax + epilogue (1 thread per row).
constexpr int ATT1_THREADS = 256;
#ifndef ATT1_STAGE_OUT
#define ATT1_STAGE_OUT 1  // staged, coalesced epilogue stores (packed windows 5-17 % faster)
#endif
#ifndef ATT1_QS
#define ATT1_QS 1  // Q stages of the single-tile kernel (2: the next item's Q in flight)
#endif
template <int HD>
struct Attn1Cfg {
  static constexpr int CH = HD / 64, REM = HD % 64;
  static constexpr int TILE_BYTES = 128 * HD * 2;
  static constexpr int KS = 3, VS = 3;
  // a second Q stage only where it fits next to the K / V rings (hd 64 / 80)
  static constexpr int QS = (ATT1_QS > 1 && (2 + KS + VS) * TILE_BYTES <= 200 * 1024) ? 2 : 1;
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = QS * TILE_BYTES;
  static constexpr int V_OFF = K_OFF + KS * TILE_BYTES;
  // epilogue rows staged per warp in shared memory, then written with
  // coalesced 16-byte stores (lanes walk consecutive bytes of a row instead of
  // one row each): where it fits
  static constexpr bool STAGE_OUT = ATT1_STAGE_OUT && (QS + KS + VS + 1) * TILE_BYTES <= 200 * 1024;
  static constexpr int OUT_OFF = V_OFF + VS * TILE_BYTES;
  static constexpr int BAR_OFF = OUT_OFF + (STAGE_OUT ? TILE_BYTES : 0);
  // q_full[QS], q_empty[QS], k_full[KS], k_empty[KS], v_full[VS], v_empty[VS],
  // s_full[2], p_full[2], pv_done, o_free, o_full
  static constexpr int N_BARS = 2 * QS + 2 * KS + 2 * VS + 7;
  static constexpr int SMEM = BAR_OFF + N_BARS * 8 + 16 + 1024;
};

template <int HD>
__global__ void __launch_bounds__(ATT1_THREADS, 1)
    attn_fwd_tc1_kernel(const __grid_constant__ CUtensorMap tmQ,
                        const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV,
                        const __grid_constant__ CUtensorMap tmQr,
                        const __grid_constant__ CUtensorMap tmKr,
                        const __grid_constant__ CUtensorMap tmVr, const AttnArgs a) {
  using Cfg = Attn1Cfg<HD>;
  constexpr int KS = Cfg::KS, VS = Cfg::VS, QS = Cfg::QS;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::BAR_OFF);
  uint64_t* q_full = bars;
  uint64_t* q_empty = bars + QS;
  uint64_t* k_full = bars + 2 * QS;
  uint64_t* k_empty = k_full + KS;
  uint64_t* v_full = k_empty + KS;
  uint64_t* v_empty = v_full + VS;
  uint64_t* s_full = v_empty + VS;
  uint64_t* p_full = s_full + 2;
  uint64_t* pv_done = p_full + 2;
  uint64_t* o_free = pv_done + 1;
  // committed after an item's LAST PV: the epilogue cannot wait on pv_done by
  // parity, because when the softmax finishes the last block both PV(L-1) and
  // PV(L) may still be outstanding (S(L) only orders PV(L-2)), and a parity
  // wait two phases behind passes at once
  uint64_t* o_full = o_free + 1;
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
    for (int q = 0; q < QS; ++q) {
      mbar_init(&q_full[q], 1);
      mbar_init(&q_empty[q], 1);
    }
    for (int i = 0; i < KS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < VS; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
    }
    mbar_init(pv_done, 1);
    mbar_init(o_free, 4);
    mbar_init(o_full, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------- TMA
      int g = 0, it = 0;
      for (int item = blockIdx.x; item < a.n_tiles; item += gridDim.x, ++it) {
        const int seq = a.tiles[5 * item], head = a.tiles[5 * item + 1],
                  qt = a.tiles[5 * item + 2], blk0 = a.tiles[5 * item + 3];
        const int kvh = head / a.group;
        const int q0 = a.q_start[seq] + qt * ATT_BM, kv0 = a.kv_start[seq] + blk0 * ATT_BN;
        const int nblk = a.tiles[5 * item + 4] - blk0;
        const int qs = it % QS;
        uint8_t* qdst = smem + Cfg::Q_OFF + qs * Cfg::TILE_BYTES;
        mbar_wait(&q_empty[qs], ((it / QS) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[qs], Cfg::TILE_BYTES);
        for (int c = 0; c < Cfg::CH; ++c)
          tma_load_3d(qdst + c * 16384, &tmQ, &q_full[qs], c * 64, head, q0);
        if (Cfg::REM)
          tma_load_3d(qdst + Cfg::CH * 16384, &tmQr, &q_full[qs], Cfg::CH * 64, head, q0);
        auto load = [&](const CUtensorMap* m, const CUtensorMap* mr, int off, uint64_t* full,
                        uint64_t* empty, int stages, int jj) {
          const int gg = g + jj, st = gg % stages;
          mbar_wait(&empty[st], ((gg / stages) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[st], Cfg::TILE_BYTES);
          uint8_t* dst = smem + off + st * Cfg::TILE_BYTES;
          for (int c = 0; c < Cfg::CH; ++c)
            tma_load_3d(dst + c * 16384, m, &full[st], c * 64, kvh, kv0 + jj * ATT_BN);
          if (Cfg::REM)
            tma_load_3d(dst + Cfg::CH * 16384, mr, &full[st], Cfg::CH * 64, kvh,
                        kv0 + jj * ATT_BN);
        };
        // consumption order: K0 K1 | V0 K2 | V1 K3 | ...
        for (int j = 0; j < nblk; ++j) {
          load(&tmK, &tmKr, Cfg::K_OFF, k_full, k_empty, KS, j);
          if (j >= 1) load(&tmV, &tmVr, Cfg::V_OFF, v_full, v_empty, VS, j - 1);
        }
        load(&tmV, &tmVr, Cfg::V_OFF, v_full, v_empty, VS, nblk - 1);
        g += nblk;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------- MMA
      constexpr uint32_t idesc_s = idesc_bf16_f32(128, ATT_BN, false, false);
      constexpr uint32_t idesc_o = idesc_bf16_f32(128, Cfg::CH * 64, false, true);
      constexpr uint32_t idesc_or = idesc_bf16_f32(128, 16, false, true);
      uint32_t qa = smem_u32(smem + Cfg::Q_OFF);  // this item's Q stage
      const uint32_t o_addr = tbase + 256;
      auto issue_s = [&](int g) {  // S(g) = Q K_g^T into buffer g & 1
        const uint32_t k_addr = smem_u32(smem + Cfg::K_OFF + (g % KS) * Cfg::TILE_BYTES);
        const uint32_t d = tbase + (g & 1) * 128;
        mbar_wait(&k_full[g % KS], (g / KS) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < Cfg::CH * 4; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          mma_ss(d, desc_sw128_kmajor(qa + off), desc_sw128_kmajor(k_addr + off), idesc_s,
                 kk != 0);
        }
        if (Cfg::REM) {
          const uint32_t off = Cfg::CH * 16384;
          mma_ss(d, desc_sw32_kmajor(qa + off), desc_sw32_kmajor(k_addr + off), idesc_s, true);
        }
        mma_commit(&s_full[g & 1]);
        mma_commit(&k_empty[g % KS]);
      };
      int g = 0, it = 0;
      for (int item = blockIdx.x; item < a.n_tiles; item += gridDim.x, ++it) {
        const int nblk = a.tiles[5 * item + 4] - a.tiles[5 * item + 3];
        const int qs = it % QS;
        qa = smem_u32(smem + Cfg::Q_OFF + qs * Cfg::TILE_BYTES);
        mbar_wait(&q_full[qs], (it / QS) & 1);
        issue_s(g);
        if (nblk > 1) issue_s(g + 1);
        if (nblk <= 2) mma_commit(&q_empty[qs]);
        for (int j = 0; j < nblk; ++j, ++g) {
          mbar_wait(&v_full[g % VS], (g / VS) & 1);
          mbar_wait(&p_full[g & 1], (g >> 1) & 1);
          if (j == 0) mbar_wait(o_free, (it & 1) ^ 1);  // the last item's epilogue read O
          tc_fence_after();
          const uint32_t v_addr = smem_u32(smem + Cfg::V_OFF + (g % VS) * Cfg::TILE_BYTES);
          const uint32_t p_addr = tbase + (g & 1) * 128;
#pragma unroll
          for (int kk = 0; kk < ATT_BN / 16; ++kk) {
            mma_ts(o_addr, p_addr + kk * 8, desc_sw128_mnmajor(v_addr + kk * 2048, 16384),
                   idesc_o, j != 0 || kk != 0);
            if (Cfg::REM)
              mma_ts(o_addr + Cfg::CH * 64, p_addr + kk * 8,
                     desc_sw32_mnmajor(v_addr + Cfg::CH * 16384 + kk * 512), idesc_or,
                     j != 0 || kk != 0);
          }
          mma_commit(pv_done);
          if (j + 1 == nblk) mma_commit(o_full);
          mma_commit(&v_empty[g % VS]);
          if (j + 2 < nblk) {
            issue_s(g + 2);  // over P(g): in-order after PV(g)
            if (j + 3 == nblk) mma_commit(&q_empty[qs]);
          }
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------- softmax
    const int ew = warp & 3;
    const int r = ew * 32 + lane;
    const uint32_t lane_off = (uint32_t)(ew * 32) << 16;
    const uint32_t t_o = tbase + lane_off + 256;
#if ATT1_PROF
    unsigned long long prof1[8] = {0};
#endif
    // Per-item metadata (tile entry -> q_start / lengths -> this row's key
    // bounds: three dependent global loads) is fetched one item AHEAD, so its
    // latency hides behind the current item's softmax and epilogue instead
    // of opening every item (the windowed ViT layers run ~25 one-block items
    // per CTA, where this chain was the item's critical path).
    struct Meta {
      int seq, head, qt, blk0, nblk, q_len, q0, lo, hi;
    };
    auto load_meta = [&](int item) {
      Meta m{};
      if (item >= a.n_tiles) return m;
      m.seq = a.tiles[5 * item];
      m.head = a.tiles[5 * item + 1];
      m.qt = a.tiles[5 * item + 2];
      m.blk0 = a.tiles[5 * item + 3];
      m.nblk = a.tiles[5 * item + 4] - m.blk0;
      m.q_len = a.q_len[m.seq];
      const int kv_len = a.kv_len[m.seq];
      m.q0 = a.q_start[m.seq];
      const int qrow = m.qt * ATT_BM + r;
      m.lo = 0;
      m.hi = kv_len;
      if (a.row_bounds) {
        if (qrow < m.q_len) {
          const int2 b = a.row_bounds[m.q0 + qrow];
          m.lo = b.x;
          m.hi = b.y;
        } else {
          m.hi = 0;
        }
      } else if (a.causal) {
        m.hi = min(kv_len - m.q_len + qrow + 1, kv_len);
      }
      return m;
    };
    int g = 0, it = 0;
    Meta nxt = load_meta(blockIdx.x);
    for (int item = blockIdx.x; item < a.n_tiles; item += gridDim.x, ++it) {
      const Meta cur = nxt;
      nxt = load_meta(item + gridDim.x);
      const int head = cur.head, qt = cur.qt, blk0 = cur.blk0;
      const int q_len = cur.q_len, nblk = cur.nblk, lo = cur.lo, hi = cur.hi;
      const int qrow = qt * ATT_BM + r;
      float m_used = -INFINITY, l_run = 0.f;
#if ATT1_PROF
      long long t_sready = 0;
#endif
      for (int j = 0; j < nblk; ++j, ++g) {
        const uint32_t t_s = tbase + lane_off + (g & 1) * 128;
        PROF1_T(p0);
        ATT_SM_WAIT(&s_full[g & 1], (g >> 1) & 1);
        tc_fence_after();
        PROF1_T(p1);
        PROF1_ADD(0, p0, p1);
#if ATT1_PROF
        t_sready = p1;
#endif
        const int kbase = (blk0 + j) * ATT_BN;
        uint32_t v[ATT_BN];
#pragma unroll
        for (int c = 0; c < ATT_BN / 32; ++c)
          tmem_ld32(t_s + c * 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32 * c));
        tmem_wait_ld();
        const bool full = __all_sync(0xffffffffu, kbase >= lo && kbase + ATT_BN <= hi);
        // per 32-key chunk, warp-uniform: dead (no row of the warp sees it),
        // whole (every row sees all of it) or partial (per-key mask); packed
        // windows are whole / dead chunks only, so no per-key work at all
        float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
        for (int c = 0; c < ATT_BN / 32; ++c) {
          const int c0 = kbase + 32 * c;
          if (!full) {
            if (__all_sync(0xffffffffu, c0 + 32 <= lo || c0 >= hi)) continue;  // dead
            if (!__all_sync(0xffffffffu, c0 >= lo && c0 + 32 <= hi)) {        // partial
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const int kp = c0 + i;
                if (kp < lo || kp >= hi) v[32 * c + i] = __float_as_uint(-INFINITY);
              }
            }
          }
#pragma unroll
          for (int i = 32 * c; i < 32 * c + 32; i += 4) {
            mx0 = fmaxf(mx0, __uint_as_float(v[i]));
            mx1 = fmaxf(mx1, __uint_as_float(v[i + 1]));
            mx2 = fmaxf(mx2, __uint_as_float(v[i + 2]));
            mx3 = fmaxf(mx3, __uint_as_float(v[i + 3]));
          }
        }
        const float mx = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3)) * a.scale_log2;
        const bool grow = mx > m_used + ATT_RESCALE_THRESH;
        if (j == 0) {
          m_used = mx;
        } else if (__any_sync(0xffffffffu, grow)) {
          // O must hold PV(g-1) before it is rescaled
          mbar_wait(pv_done, (g - 1) & 1);
          tc_fence_after();
          const float m_new = grow ? mx : m_used;
          const float alpha = m_new == m_used ? 1.f : fast_exp2(m_used - m_new);
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
        const float2 sc2 = make_float2(a.scale_log2, a.scale_log2), nb2 = make_float2(nbase, nbase);
        float2 rsa = make_float2(0.f, 0.f), rsb = make_float2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < ATT_BN / 32; ++c) {
          uint32_t pk[16];
          // a 32-key chunk no row of this warp can see (the other window of a
          // packed tile, a causal block's upper part, rows past the end):
          // P = 0 without the exponentials (half of every windowed block)
          const int c0 = kbase + 32 * c;
          const bool dead = !full && __all_sync(0xffffffffu, c0 + 32 <= lo || c0 >= hi);
          if (dead) {
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = 0u;
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int e = 32 * c + 2 * i;
              const float2 x = ffma2(
                  make_float2(__uint_as_float(v[e]), __uint_as_float(v[e + 1])), sc2, nb2);
              float2 pp;
              if ((e & 7) >= ATT1_POLY_FROM) {
                pp = poly_exp2x2(x);
              } else {
                pp.x = fast_exp2(x.x);
                pp.y = fast_exp2(x.y);
              }
              if (i & 1)
                rsb = fadd2(rsb, pp);
              else
                rsa = fadd2(rsa, pp);
              pk[i] = pack_bf16(pp.x, pp.y);
            }
          }
          tmem_st16(t_s + c * 16, pk);
        }
        l_run += (rsa.x + rsa.y) + (rsb.x + rsb.y);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[g & 1]);
      }
      // epilogue: O / l -> bf16 once the item's last PV is done
      PROF1_T(p2);
      mbar_wait(o_full, it & 1);
      tc_fence_after();
      PROF1_T(p3);
      PROF1_ADD(1, t_sready, p2);  // last block: softmax after its S (per item)
      PROF1_ADD(2, p2, p3);  // epilogue: wait for the last PV
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      const bool ok = qrow < q_len;
      __nv_bfloat16* orow =
          a.out + (int64_t)(cur.q0 + qrow) * a.out_tok_stride + (int64_t)head * HD;
      if constexpr (Cfg::STAGE_OUT) {
        constexpr int U = HD * 2 / 16;  // 16-byte units per row
        uint4* wbuf = reinterpret_cast<uint4*>(smem + Cfg::OUT_OFF + ew * 32 * (HD * 2));
        __syncwarp();  // the warp's previous copy-out has read wbuf
#pragma unroll 1
        for (int c = 0; c < HD / 32; ++c) {
          uint32_t o[32];
          tmem_ld32(t_o + c * 32, o);
          tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 u;
            u.x = pack_bf16(__uint_as_float(o[8 * q + 0]) * inv, __uint_as_float(o[8 * q + 1]) * inv);
            u.y = pack_bf16(__uint_as_float(o[8 * q + 2]) * inv, __uint_as_float(o[8 * q + 3]) * inv);
            u.z = pack_bf16(__uint_as_float(o[8 * q + 4]) * inv, __uint_as_float(o[8 * q + 5]) * inv);
            u.w = pack_bf16(__uint_as_float(o[8 * q + 6]) * inv, __uint_as_float(o[8 * q + 7]) * inv);
            wbuf[lane * U + c * 4 + q] = u;
          }
        }
        if (HD % 32) {
          uint32_t o[16];
          tmem_ld16(t_o + (HD / 32) * 32, o);
          tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            uint4 u;
            u.x = pack_bf16(__uint_as_float(o[8 * q + 0]) * inv, __uint_as_float(o[8 * q + 1]) * inv);
            u.y = pack_bf16(__uint_as_float(o[8 * q + 2]) * inv, __uint_as_float(o[8 * q + 3]) * inv);
            u.z = pack_bf16(__uint_as_float(o[8 * q + 4]) * inv, __uint_as_float(o[8 * q + 5]) * inv);
            u.w = pack_bf16(__uint_as_float(o[8 * q + 6]) * inv, __uint_as_float(o[8 * q + 7]) * inv);
            wbuf[lane * U + (HD / 32) * 4 + q] = u;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(o_free);  // O is in registers / smem now
        // coalesced copy-out: unit u of the warp's 32 x U block -> row u / U
        const int row0 = cur.q0 + qt * ATT_BM + ew * 32;
        const int rows_ok = min(32, q_len - (qt * ATT_BM + ew * 32));
#pragma unroll
        for (int it2 = 0; it2 < U; ++it2) {
          const int u = it2 * 32 + lane;
          const int rr = u / U, cc = u - rr * U;
          if (rr < rows_ok)
            reinterpret_cast<uint4*>(a.out + (int64_t)(row0 + rr) * a.out_tok_stride +
                                     (int64_t)head * HD)[cc] = wbuf[u];
        }
        PROF1_T(p4s);
        PROF1_ADD(3, p3, p4s);
        PROF1_ADD(4, 0, 1);
        continue;
      }
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
      if (lane == 0) mbar_arrive(o_free);
      PROF1_T(p4);
      PROF1_ADD(3, p3, p4);  // epilogue: TMEM -> bf16 -> global
      PROF1_ADD(4, 0, 1);    // items
    }
#if ATT1_PROF
    if (lane == 0)
      for (int i = 0; i < 8; ++i) atomicAdd(&g_att_prof[i], prof1[i]);
#endif
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

// [next, done] work-queue counters of the pair kernel, one pair per (device,
// stream): launches on one stream are ordered, and the last CTA of a launch
// resets its pair.  EMM_ATT_DYN=0: round-robin items instead.
static int* attn_sched_counters(cudaStream_t stream) {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("EMM_ATT_DYN");
    mode = (e && e[0] == '0') ? 0 : 1;
  }
  if (!mode) return nullptr;
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, int*> counters;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = counters.find({dev, stream});
  if (it != counters.end()) return it->second;
  int* c = nullptr;
  // zeroed on the launch stream itself: ordered before this stream's first
  // attention launch (a legacy-stream memset would not be, for non-blocking streams)
  if (cudaMalloc(&c, 2 * sizeof(int)) != cudaSuccess ||
      cudaMemsetAsync(c, 0, 2 * sizeof(int), stream) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;  // round-robin
  }
  counters[{dev, stream}] = c;
  return c;
}

template <int HD>
static int launch_attn(const void* q, int64_t q_tok_stride, const void* k, const void* v,
                       int64_t kv_tok_stride, int64_t n_q_tokens, int64_t n_kv_tokens,
                       int n_q_heads, int n_kv_heads, const AttnArgs& args, int n_tiles,
                       int tile_rows, cudaStream_t stream) {
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
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(attn_fwd_tc1_kernel<HD>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, Attn1Cfg<HD>::SMEM);

    if (e != cudaSuccess) return cuda_status(e, "attn smem attribute");
    attr_done[dev & 63] = true;
  }
  const int grid = n_tiles < sm_count() ? n_tiles : sm_count();
  if (tile_rows == 128) {
    attn_fwd_tc1_kernel<HD><<<grid, ATT1_THREADS, Attn1Cfg<HD>::SMEM, stream>>>(
        tq, tk, tv, tqr, tkr, tvr, args);
    count_launch();
    EMM_CUDA_CHECK_LAUNCH("attn_fwd_tc1_kernel");
    return EMM_OK;
  }
  AttnArgs pa = args;
  pa.sched = attn_sched_counters(stream);
  attn_fwd_tc_kernel<HD><<<grid, ATT_THREADS, Cfg::SMEM, stream>>>(tq, tk, tv, tqr, tkr, tvr,
                                                                     pa);
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
                                  const int32_t* kv_start, const int32_t* kv_len,
                                  const int32_t* row_bounds, float scale, int causal,
                                  int tile_rows, void* stream) {
  using namespace emm;
  if (n_tiles <= 0) return EMM_OK;
  if (!q || !k || !v || !out || n_kv_heads <= 0 || n_q_heads % n_kv_heads != 0 ||
      (head_dim != 64 && head_dim != 80 && head_dim != 128) || (q_tok_stride % 8) || (kv_tok_stride % 8) ||
      (out_tok_stride % 8) || (tile_rows != 128 && tile_rows != 256)) {
    emm_abi::set_error("emm_attention_bf16: head_dim 64/80/128, GQA divisibility, 16B pitches");
    return EMM_E_INVALID;
  }
  AttnArgs a;
  a.tiles = tiles;
  a.n_tiles = n_tiles;
  a.row_bounds = reinterpret_cast<const int2*>(row_bounds);
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
  a.sched = nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  if (head_dim == 128)
    return launch_attn<128>(q, q_tok_stride, k, v, kv_tok_stride, n_q_tokens, n_kv_tokens,
                            n_q_heads, n_kv_heads, a, n_tiles, tile_rows, st);
  if (head_dim == 80)
    return launch_attn<80>(q, q_tok_stride, k, v, kv_tok_stride, n_q_tokens, n_kv_tokens,
                           n_q_heads, n_kv_heads, a, n_tiles, tile_rows, st);
  return launch_attn<64>(q, q_tok_stride, k, v, kv_tok_stride, n_q_tokens, n_kv_tokens,
                         n_q_heads, n_kv_heads, a, n_tiles, tile_rows, st);
}

#if ATT_PROF || ATT1_PROF
extern "C" int emm_attn_prof(unsigned long long* out16, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out16, emm::g_att_prof, 16 * sizeof(unsigned long long));
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(emm::g_att_prof, z, sizeof(z));
  }
  return 0;
}
#endif
