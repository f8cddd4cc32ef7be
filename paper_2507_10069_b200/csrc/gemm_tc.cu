// gemm_tc.cu — persistent warp-specialised tcgen05 GEMM for sm_100a.
//
//   C[M,N] = epilogue( A[M,K] . B[N,K]^T )     bf16 in, fp32 accumulate in TMEM
//
// This is the dense contraction behind the encoder (patch embed, QKV / O /
// MLP projections) and the prefill decoder layers: the work the reference
// models analytically as encode_time / prefill_time
// (pkg/src/mmsim/costmodel.py:102-119).
//
// Layout per CTA (1 CTA / SM, persistent over 128 x BN tiles):
//   warp 0      TMA producer: A tile 128x64, B tile BNx64 per stage, SW128
//   warp 1      MMA issuer: 4 x tcgen05.mma (K = 16) per stage, M=128 N=BN
//   warp 2      TMEM allocator (2 x BN fp32 columns: double-buffered accum)
//   warps 4..7  epilogue: tcgen05.ld 32x32b -> bias / activation / residual /
//               SwiGLU -> bf16 -> global; overlaps the next tile's mainloop
// Pipelines: smem full/empty ring (TMA <-> MMA) and TMEM full/empty pair
// (MMA <-> epilogue), all mbarrier based.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <stdlib.h>

#include "../../include/emm.h"
#include "gemm_common.cuh"
#include "ptx.cuh"
#include "runtime.h"

namespace emm {

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;
#ifndef SPLITK_KA_DEFAULT
#define SPLITK_KA_DEFAULT 2  // measured: qkv / o-proj 5-8 % faster than 1 (profiles/r02/gemm_ka.txt)
#endif
#ifndef GEMM_PAIR_STAGES
#define GEMM_PAIR_STAGES 6  // 32 KiB per stage (A 16 + half of B 16)
#endif
#ifndef GEMM_EPI_GROUPS
#define GEMM_EPI_GROUPS 1  // 2: eight epilogue warps, two per TMEM lane quarter
#endif
constexpr int GEMM_EPI_G = GEMM_EPI_GROUPS;
constexpr int GEMM_THREADS = 128 + 128 * GEMM_EPI_G;
constexpr int GEMM_GROUP_M = 16;

struct GemmArgs {
  int M, N, K;
  // rows of the A box per TMA load (64 when M <= 64, e.g. decode: the MMA
  // still reads 128 rows, rows >= M are never stored)
  int a_box_rows;
  __nv_bfloat16* C;
  int64_t ldc;
  const __nv_bfloat16* bias;
  const __nv_bfloat16* residual;
  int64_t ldr;
  int epi;
  int num_m, num_n, num_tiles;
  // folded RMSNorm: scale row m by rsqrt(row_ss_in[m] / rms_dim + eps)
  const float* row_ss_in;
  float rms_inv_dim, rms_eps;
  // sum of squares of the stored output rows (the next layer's RMSNorm)
  float* row_ss_out;
  // EMM_EPI_QKV_ROPE: split + rotate-half RoPE + KV-cache write
  __nv_bfloat16* q_out;
  int64_t ld_q;
  __nv_bfloat16* k_out;
  __nv_bfloat16* v_out;
  int64_t ld_kv;
  const int32_t* kv_row;
  const int32_t* pos;
  const float2* rope_cs;  // [pos][hd/2] (cos, sin)
  int hq, hkv, hd;
  // multimodal RoPE: rotary pair i uses pos (i < s0), pos_h (i < s0+s1) or pos_w
  const int32_t* pos_h;
  const int32_t* pos_w;
  int mrope_s0, mrope_s1;
  // split-K (small-M GEMMs, e.g. decode): work item w = tile * ksplit + ks
  // covers k-blocks [ks*nkb/ksplit, (ks+1)*nkb/ksplit); every item stores its
  // fp32 partial tile (column-major [BN][128]) to ws, and the last of a
  // tile's ksplit items to arrive (cnt[tile]) adds the others' partials to
  // its TMEM accumulator and runs the normal epilogue.
  int ksplit;
  float* ws;
  int* cnt;
  float* row_ss_zero;
  // 2-D vision RoPE on adjacent column pairs of columns [0, rope2_cols)
  const float2* rope2_cs;
  int rope2_cols, rope2_hd;
};

struct SplitAcc {
  const float* ws;  // the tile's partials, ksplit x [BN][128] (nullptr: no split)
  int parts, self, row_local;
};

// KA > 1 (decode-size split-K, M <= 64): every stage carries KA consecutive
// 64-column K atoms (KA x 128 contiguous bytes of every weight row per stage
// instead of 128) with 64-row A atoms; the MMA of an A atom reads rows
// 64..127 from the next atom / the stage's B buffer (discarded rows >= M)
template <int BN, int STAGES, int KA = 1>
struct GemmCfg {
  static constexpr int A_ATOM = (KA > 1 ? 64 : GEMM_BM) * GEMM_BK * 2;
  static constexpr int B_ATOM = BN * GEMM_BK * 2;
  static constexpr int A_BYTES = A_ATOM * KA;
  static constexpr int B_BYTES = B_ATOM * KA;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int SMEM = BAR_OFF + (2 * STAGES + 4) * 8 + 16 + 1024;
  static constexpr int TMEM_COLS = 2 * BN;
};

// grouped rasterisation: bands of GEMM_GROUP_M m-blocks, n-major inside a band
__device__ __forceinline__ void tile_coords(int t, int num_m, int num_n, int& mb, int& nb) {
  const int span = GEMM_GROUP_M * num_n;
  const int band = t / span;
  const int first = band * GEMM_GROUP_M;
  const int rows = min(GEMM_GROUP_M, num_m - first);
  const int local = t - band * span;
  mb = first + local % rows;
  nb = local / rows;
}

__device__ __forceinline__ void load_bf16x32(const __nv_bfloat16* p, float (&v)[32]) {
  const uint4* q = reinterpret_cast<const uint4*>(p);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint4 u = __ldg(q + i);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 f = __bfloat1622float2(h[j]);
      v[i * 8 + 2 * j] = f.x;
      v[i * 8 + 2 * j + 1] = f.y;
    }
  }
}

#ifndef EMM_EPI_PREFETCH
#define EMM_EPI_PREFETCH 1
#endif
// raw 64-byte row chunk (issued early: the epilogue prefetches the next
// chunk's bias / residual while it works on the current one)
__device__ __forceinline__ void ldg_raw64(const __nv_bfloat16* p, uint4 (&u)[4]) {
  const uint4* q = reinterpret_cast<const uint4*>(p);
#pragma unroll
  for (int i = 0; i < 4; ++i) u[i] = __ldg(q + i);
}
__device__ __forceinline__ void unpack_bf16x32(const uint4 (&u)[4], float (&v)[32]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u[i]);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 f = __bfloat1622float2(h[j]);
      v[i * 8 + 2 * j] = f.x;
      v[i * 8 + 2 * j + 1] = f.y;
    }
  }
}

__device__ __forceinline__ void store_bf16x32(__nv_bfloat16* p, const float (&v)[32]) {
  uint4* q = reinterpret_cast<uint4*>(p);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint4 u;
    u.x = pack_bf16(v[i * 8 + 0], v[i * 8 + 1]);
    u.y = pack_bf16(v[i * 8 + 2], v[i * 8 + 3]);
    u.z = pack_bf16(v[i * 8 + 4], v[i * 8 + 5]);
    u.w = pack_bf16(v[i * 8 + 6], v[i * 8 + 7]);
    q[i] = u;
  }
}

// split-K: add the other items' partials of columns [col, col+32) of this row
// Two partials per round trip (64 L2 loads in flight per thread instead of
// 32: the last arriver's reduction is the split GEMM's tail); same addition
// order as one partial at a time, so results are unchanged bit for bit.
template <int BN>
__device__ __forceinline__ void add_partials(const SplitAcc& sp, int col, uint32_t (&r)[32]) {
  if (!sp.ws) return;
  const float* base = sp.ws + (size_t)col * 128 + sp.row_local;
  const int n = sp.parts - 1;  // the other items, in k order (self skipped)
  int i = 0;
  for (; i + 2 <= n; i += 2) {
    const int k0 = i < sp.self ? i : i + 1;
    const int k1 = i + 1 < sp.self ? i + 1 : i + 2;
    const float* p0 = base + (size_t)k0 * 128 * BN;
    const float* p1 = base + (size_t)k1 * 128 * BN;
    float a[32], b[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) a[j] = __ldcg(p0 + j * 128);
#pragma unroll
    for (int j = 0; j < 32; ++j) b[j] = __ldcg(p1 + j * 128);
#pragma unroll
    for (int j = 0; j < 32; ++j) r[j] = __float_as_uint((__uint_as_float(r[j]) + a[j]) + b[j]);
  }
  if (i < n) {
    const int k0 = i < sp.self ? i : i + 1;
    const float* p = base + (size_t)k0 * 128 * BN;
#pragma unroll
    for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) + __ldcg(p + j * 128));
  }
}

// Epilogue of one accumulator tile: this thread owns output row `row`, the
// tile's columns start at nb*BN; t_row = TMEM address of (row, column 0).
// grp: this warp's epilogue group (GEMM_EPI_G groups split the tile's
// column chunks / heads round-robin; each group owns every row once)
template <int BN>
__device__ __forceinline__ void epilogue_tile(const GemmArgs& args, uint32_t t_row, int row,
                                              int nb, const SplitAcc& sp = SplitAcc{},
                                              int grp = 0) {
  const bool row_ok = row < args.M;
  if (args.row_ss_zero && nb == 0 && row_ok && grp == 0) args.row_ss_zero[row] = 0.f;
  float rs = 1.f;  // folded RMSNorm row scale
  if (args.row_ss_in && row_ok)
    rs = rsqrtf(__ldg(args.row_ss_in + row) * args.rms_inv_dim + args.rms_eps);
  if (args.epi == EMM_EPI_QKV_ROPE) {
    const int hd = args.hd, half = hd >> 1;
    const int q_dim = args.hq * hd, kv_dim = args.hkv * hd;
    int64_t kvr = 0;
    int p = 0, ph = 0, pw = 0;
    if (row_ok) {
      kvr = args.kv_row[row];
      p = args.pos ? args.pos[row] : 0;
      ph = args.pos_h ? args.pos_h[row] : p;
      pw = args.pos_w ? args.pos_w[row] : p;
    }
    const int s0 = args.mrope_s0, s01 = args.mrope_s0 + args.mrope_s1;
#pragma unroll 1
    for (int h = grp; h < BN / hd; h += GEMM_EPI_G) {
      const int col_h = nb * BN + h * hd;  // first column of this head
      if (col_h >= args.N) break;
      const int sect = col_h < q_dim ? 0 : (col_h < q_dim + kv_dim ? 1 : 2);
      __nv_bfloat16* dst;
      if (sect == 0)
        dst = args.q_out + (int64_t)row * args.ld_q + col_h;
      else if (sect == 1)
        dst = args.k_out + kvr * args.ld_kv + (col_h - q_dim);
      else
        dst = args.v_out + kvr * args.ld_kv + (col_h - q_dim - kv_dim);
#pragma unroll 1
      for (int ic = 0; ic < half / 32; ++ic) {
        uint32_t ra[32], rb[32];
        tmem_ld32(t_row + h * hd + ic * 32, ra);
        tmem_ld32(t_row + h * hd + half + ic * 32, rb);
        tmem_wait_ld();
        add_partials<BN>(sp, h * hd + ic * 32, ra);
        add_partials<BN>(sp, h * hd + half + ic * 32, rb);
        float a[32], b[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          a[j] = __uint_as_float(ra[j]) * rs;
          b[j] = __uint_as_float(rb[j]) * rs;
        }
        if (args.bias) {
          float ba[32], bb[32];
          load_bf16x32(args.bias + col_h + ic * 32, ba);
          load_bf16x32(args.bias + col_h + half + ic * 32, bb);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            a[j] += ba[j];
            b[j] += bb[j];
          }
        }
        if (sect < 2 && args.rope_cs && row_ok) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int i = ic * 32 + j;  // rotary pair (section of the M-RoPE position)
            const int pp = i < s0 ? p : (i < s01 ? ph : pw);
            const float2 c = __ldg(args.rope_cs + (int64_t)pp * half + i);
            const float x = a[j], y = b[j];
            a[j] = x * c.x - y * c.y;
            b[j] = y * c.x + x * c.y;
          }
        }
        if (row_ok) {
          store_bf16x32(dst + ic * 32, a);
          store_bf16x32(dst + half + ic * 32, b);
        }
      }
    }
  } else if (args.epi == EMM_EPI_GLU_SILU) {
    const int n_out = args.N >> 1;
#pragma unroll 1
    for (int c = grp; c < BN / 64; c += GEMM_EPI_G) {
      const int ocol = nb * (BN / 2) + c * 32;
      if (ocol >= n_out) break;
      uint32_t rg[32], ru[32];
      tmem_ld32(t_row + c * 32, rg);
      tmem_ld32(t_row + BN / 2 + c * 32, ru);
      tmem_wait_ld();
      add_partials<BN>(sp, c * 32, rg);
      add_partials<BN>(sp, BN / 2 + c * 32, ru);
      float g[32], u[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        g[j] = __uint_as_float(rg[j]) * rs;
        u[j] = __uint_as_float(ru[j]) * rs;
      }
      if (args.bias) {
        float bg[32], bu[32];
        load_bf16x32(args.bias + nb * BN + c * 32, bg);
        load_bf16x32(args.bias + nb * BN + BN / 2 + c * 32, bu);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          g[j] += bg[j];
          u[j] += bu[j];
        }
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) g[j] = act_silu(g[j]) * u[j];
      if (row_ok) store_bf16x32(args.C + (int64_t)row * args.ldc + ocol, g);
    }
  } else {
    float ss = 0.f;
    // software pipeline: chunk c+1's bias / residual loads are in flight
    // while chunk c is read from TMEM and processed (their global latency
    // used to serialise with every chunk)
    const bool has_res = args.residual && row_ok;
    uint4 bnext[4], rnext[4];
    const int col0 = nb * BN + grp * 32;
    if (EMM_EPI_PREFETCH && args.bias && col0 < args.N) ldg_raw64(args.bias + col0, bnext);
    if (EMM_EPI_PREFETCH && has_res && col0 < args.N)
      ldg_raw64(args.residual + (int64_t)row * args.ldr + col0, rnext);
#pragma unroll 1
    for (int c = grp; c < BN / 32; c += GEMM_EPI_G) {
      const int col = nb * BN + c * 32;
      if (col >= args.N) break;
      uint4 bcur[4], rcur[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        bcur[i] = bnext[i];
        rcur[i] = rnext[i];
      }
      constexpr int STEP = 32 * GEMM_EPI_G;
      const bool more = EMM_EPI_PREFETCH && c + GEMM_EPI_G < BN / 32 && col + STEP < args.N;
      if (!EMM_EPI_PREFETCH) {  // A/B switch: plain loads of this chunk
        if (args.bias) ldg_raw64(args.bias + col, bcur);
        if (has_res) ldg_raw64(args.residual + (int64_t)row * args.ldr + col, rcur);
      }
      if (more && args.bias) ldg_raw64(args.bias + col + STEP, bnext);
      if (more && has_res) ldg_raw64(args.residual + (int64_t)row * args.ldr + col + STEP, rnext);
      // 2-D RoPE (cos, sin) of this chunk's 16 pairs: loads issued before the
      // TMEM read so their (L2) latency overlaps it
      const bool rope2 = args.rope2_cs && col < args.rope2_cols && row_ok;
      float2 csv[16];
      if (rope2) {
        const int hd = args.rope2_hd, half = hd >> 1, quarter = hd >> 2;
        const int ph = args.pos_h[row], pw = args.pos_w[row];
        const int i0 = (col % hd) >> 1;  // rotary pair of the chunk's first column
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int i = i0 + j >= half ? i0 + j - half : i0 + j;  // < 16 pairs: one wrap
          const bool hrow = i < quarter;
          csv[j] =
              __ldg(args.rope2_cs + (int64_t)(hrow ? ph : pw) * quarter + (hrow ? i : i - quarter));
        }
      }
      uint32_t r[32];
      tmem_ld32(t_row + c * 32, r);
      tmem_wait_ld();
      add_partials<BN>(sp, c * 32, r);
      float v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]) * rs;
      if (args.bias) {
        float b[32];
        unpack_bf16x32(bcur, b);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] += b[j];
      }
      if (rope2) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float x = v[2 * j], y = v[2 * j + 1];
          v[2 * j] = x * csv[j].x - y * csv[j].y;
          v[2 * j + 1] = y * csv[j].x + x * csv[j].y;
        }
      }
      switch (args.epi) {
        case EMM_EPI_GELU_TANH:
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = act_gelu_tanh(v[j]);
          break;
        case EMM_EPI_QUICK_GELU:
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = act_quick_gelu(v[j]);
          break;
        case EMM_EPI_GELU_ERF:
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = act_gelu_erf(v[j]);
          break;
        default:
          break;
      }
      if (row_ok) {
        if (has_res) {
          float rr[32];
          unpack_bf16x32(rcur, rr);
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] += rr[j];
        }
        store_bf16x32(args.C + (int64_t)row * args.ldc + col, v);
        if (args.row_ss_out) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {  // sum of squares of the stored bf16 values
            const float q = __bfloat162float(__float2bfloat16(v[j]));
            ss += q * q;
          }
        }
      }
    }
    if (args.row_ss_out && row_ok) atomicAdd(args.row_ss_out + row, ss);
  }
}

template <int BN, int STAGES, int KA = 1>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_bf16_tc_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB, const GemmArgs args) {
  using Cfg = GemmCfg<BN, STAGES, KA>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4 * GEMM_EPI_G);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // programmatic dependent launch: the prologue above overlapped the previous
  // kernel; global memory is touched only after it completed
  pdl_wait();
  pdl_trigger();
  const uint32_t tmem_base = *tmem_slot;
  const int nkb = (args.K + GEMM_BK * KA - 1) / (GEMM_BK * KA);  // stages of K
  const int ks_n = args.ksplit > 1 ? args.ksplit : 1;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int w = blockIdx.x; w < args.num_tiles * ks_n; w += gridDim.x) {
        const int t = w / ks_n, ks = w - t * ks_n;
        int mb, nb;
        tile_coords(t, args.num_m, args.num_n, mb, nb);
        const int kb0 = ks * nkb / ks_n, kb1 = (ks + 1) * nkb / ks_n;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
          mbar_arrive_expect_tx(&full[stage],
                                KA * (args.a_box_rows * GEMM_BK * 2 + Cfg::B_ATOM));
#pragma unroll
          for (int a = 0; a < KA; ++a) {
            const int kc = (kb * KA + a) * GEMM_BK;
            tma_load_2d(sa + a * Cfg::A_ATOM, &tmA, &full[stage], kc, mb * GEMM_BM);
            tma_load_2d(sa + Cfg::A_BYTES + a * Cfg::B_ATOM, &tmB, &full[stage], kc, nb * BN);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA issuer
      constexpr uint32_t idesc = idesc_bf16_f32(GEMM_BM, BN, false, false);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int w = blockIdx.x; w < args.num_tiles * ks_n; w += gridDim.x, ++it) {
        const int ks = w % ks_n;
        const int kb0 = ks * nkb / ks_n, kb1 = (ks + 1) * nkb / ks_n;
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + stage * Cfg::STAGE_BYTES);
#pragma unroll
          for (int a = 0; a < KA; ++a) {
            const uint64_t adesc = desc_sw128_kmajor(a_addr + a * Cfg::A_ATOM);
            const uint64_t bdesc = desc_sw128_kmajor(a_addr + Cfg::A_BYTES + a * Cfg::B_ATOM);
#pragma unroll
            for (int k = 0; k < GEMM_BK / 16; ++k) {
              // +32 B per K=16 step inside the 128 B swizzle atom
              mma_ss(d_tmem, adesc + (uint64_t)(2 * k), bdesc + (uint64_t)(2 * k), idesc,
                     (kb != kb0) || (a != 0) || (k != 0));
            }
          }
          mma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue
    const int ew = warp & 3;  // TMEM lane quarter this warp may access
    const int grp = (warp - 4) >> 2;  // epilogue group (column chunks round-robin)
    __shared__ int s_last;
    int it = 0;
    for (int w = blockIdx.x; w < args.num_tiles * ks_n; w += gridDim.x, ++it) {
      const int t = w / ks_n, ks = w - t * ks_n;
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      int mb, nb;
      tile_coords(t, args.num_m, args.num_n, mb, nb);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = mb * GEMM_BM + ew * 32 + lane;
      const uint32_t t_row = tmem_base + ((uint32_t)(ew * 32) << 16) + (uint32_t)(acc * BN);
      if (ks_n == 1) {
        epilogue_tile<BN>(args, t_row, row, nb, SplitAcc{}, grp);
      } else {
        const int rl = ew * 32 + lane;
        float* tile_ws = args.ws + (size_t)t * ks_n * 128 * BN;
        float* mine = tile_ws + (size_t)ks * 128 * BN;
#pragma unroll 1
        for (int c = grp; c < BN / 32; c += GEMM_EPI_G) {
          uint32_t r[32];
          tmem_ld32(t_row + c * 32, r);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) __stcg(mine + (size_t)(c * 32 + j) * 128 + rl,
                                              __uint_as_float(r[j]));
        }
        __threadfence();
        asm volatile("bar.sync 1, %0;\n" ::"n"(128 * GEMM_EPI_G) : "memory");
        if (threadIdx.x == 128) {
          const int old = atomicAdd(args.cnt + t, 1);
          s_last = old == ks_n - 1;
          if (old == ks_n - 1) args.cnt[t] = 0;  // ready for the next launch
        }
        asm volatile("bar.sync 1, %0;\n" ::"n"(128 * GEMM_EPI_G) : "memory");
        if (s_last) {
          __threadfence();
          epilogue_tile<BN>(args, t_row, row, nb, SplitAcc{tile_ws, ks_n, ks, rl}, grp);
        }
        asm volatile("bar.sync 1, %0;\n" ::"n"(128 * GEMM_EPI_G) : "memory");  // s_last reuse
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

static bool gemm_small_a_box() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EMM_GEMM_SMALL_A_BOX");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

template <int BN, int STAGES, int KA = 1>
static int launch_gemm(const void* A, int64_t lda, const void* B, int64_t ldb, GemmArgs args,
                       cudaStream_t stream) {
  using Cfg = GemmCfg<BN, STAGES, KA>;
  CUtensorMap ta, tb;
  args.a_box_rows = (KA > 1 || (args.M <= 64 && gemm_small_a_box())) ? 64 : GEMM_BM;
  if (!make_tmap_2d(&ta, A, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)args.K,
                    (uint64_t)args.M, (uint64_t)lda * 2, GEMM_BK, args.a_box_rows,
                    CU_TENSOR_MAP_SWIZZLE_128B))
    return EMM_E_INVALID;
  if (!make_tmap_2d(&tb, B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)args.K,
                    (uint64_t)args.N, (uint64_t)ldb * 2, GEMM_BK, BN,
                    CU_TENSOR_MAP_SWIZZLE_128B))
    return EMM_E_INVALID;
  static bool attr_done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_done[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(gemm_bf16_tc_kernel<BN, STAGES, KA>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return cuda_status(e, "gemm smem attribute");
    attr_done[dev & 63] = true;
  }
  args.num_m = (args.M + GEMM_BM - 1) / GEMM_BM;
  args.num_n = (args.N + BN - 1) / BN;
  args.num_tiles = args.num_m * args.num_n;
  const int items = args.num_tiles * (args.ksplit > 1 ? args.ksplit : 1);
  const int grid = items < sm_count() ? items : sm_count();
  launch_pdl(gemm_bf16_tc_kernel<BN, STAGES, KA>, dim3(grid), dim3(GEMM_THREADS), Cfg::SMEM,
             stream, ta, tb, args);
  count_launch();
  EMM_CUDA_CHECK_LAUNCH("gemm_bf16_tc_kernel launch");
  return EMM_OK;
}

// ---------------------------------------------------------------------------
// CTA-pair variant (cluster of 2, tcgen05 cta_group::2): the pair computes a
// 256 x BN tile; CTA r holds A rows [128r, 128r+128) and B rows
// [r*BN/2, (r+1)*BN/2) of the tile, so each SM stages only half of B per
// k-block (32 KiB/stage instead of 48) and arithmetic intensity per SM rises
// from 85 to 128 FLOP/byte.  The leader (rank 0) issues every MMA; its
// commits multicast to both CTAs' barriers.  Each CTA's TMEM holds its 128
// rows x BN fp32 (double buffered) and runs its own epilogue.
template <int BN, int STAGES>
struct GemmPairCfg {
  static constexpr int A_BYTES = GEMM_BM * GEMM_BK * 2;        // 16 KiB
  static constexpr int B_BYTES = (BN / 2) * GEMM_BK * 2;       // 16 KiB at BN=256
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int SMEM = BAR_OFF + (2 * STAGES + 4) * 8 + 16 + 1024;
  static constexpr int TMEM_COLS = 2 * BN;
};

template <int BN, int STAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GEMM_THREADS, 1)
    gemm_bf16_tc2_kernel(const __grid_constant__ CUtensorMap tmA,
                         const __grid_constant__ CUtensorMap tmB, const GemmArgs args) {
  using Cfg = GemmPairCfg<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 2);   // one arrive per CTA (+ both CTAs' TMA bytes), leader's used
      mbar_init(&empty[s], 1);  // leader's MMA commit, multicast to both
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);   // leader's MMA commit, multicast to both
      mbar_init(&tempty[a], 8 * GEMM_EPI_G);  // epilogue warps x 2 CTAs, leader's used
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  pdl_wait();
  pdl_trigger();
  const uint32_t tmem_base = *tmem_slot;
  const int nkb = (args.K + GEMM_BK - 1) / GEMM_BK;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer (both CTAs)
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair; t < args.num_tiles; t += n_pairs) {
        int mb, nb;
        tile_coords(t, args.num_m, args.num_n, mb, nb);
        const int m0 = mb * 2 * GEMM_BM + (int)rank * GEMM_BM;
        const int n0 = nb * BN + (int)rank * (BN / 2);
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
          if (leader)
            mbar_arrive_expect_tx(&full[stage], 2 * Cfg::STAGE_BYTES);
          else
            mbar_arrive_cluster(&full[stage], 0);
          tma_load_2d_pair(sa, &tmA, &full[stage], kb * GEMM_BK, m0);
          tma_load_2d_pair(sa + Cfg::A_BYTES, &tmB, &full[stage], kb * GEMM_BK, n0);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ------------------------------------------------ MMA issuer (leader only)
      constexpr uint32_t idesc = idesc_bf16_f32(2 * GEMM_BM, BN, false, false);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = pair; t < args.num_tiles; t += n_pairs, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + stage * Cfg::STAGE_BYTES);
          const uint64_t adesc = desc_sw128_kmajor(a_addr);
          const uint64_t bdesc = desc_sw128_kmajor(a_addr + Cfg::A_BYTES);
#pragma unroll
          for (int k = 0; k < GEMM_BK / 16; ++k)
            mma_ss_pair(d_tmem, adesc + (uint64_t)(2 * k), bdesc + (uint64_t)(2 * k), idesc,
                        (kb | k) != 0);
          mma_commit_pair(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit_pair(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ epilogue (both CTAs)
    const int ew = warp & 3;
    int it = 0;
    for (int t = pair; t < args.num_tiles; t += n_pairs, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      int mb, nb;
      tile_coords(t, args.num_m, args.num_n, mb, nb);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = mb * 2 * GEMM_BM + (int)rank * GEMM_BM + ew * 32 + lane;
      const uint32_t t_row = tmem_base + ((uint32_t)(ew * 32) << 16) + (uint32_t)(acc * BN);
      epilogue_tile<BN>(args, t_row, row, nb, SplitAcc{}, (warp - 4) >> 2);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&tempty[acc], 0);
    }
  }
  tc_fence_before();
  __syncwarp();  // role lanes reconverge before the warp-aligned cluster barrier
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, Cfg::TMEM_COLS);
  }
}

template <int BN, int STAGES>
static int launch_gemm_pair(const void* A, int64_t lda, const void* B, int64_t ldb,
                            GemmArgs args, cudaStream_t stream) {
  using Cfg = GemmPairCfg<BN, STAGES>;
  CUtensorMap ta, tb;
  if (!make_tmap_2d(&ta, A, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)args.K,
                    (uint64_t)args.M, (uint64_t)lda * 2, GEMM_BK, GEMM_BM,
                    CU_TENSOR_MAP_SWIZZLE_128B))
    return EMM_E_INVALID;
  if (!make_tmap_2d(&tb, B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)args.K,
                    (uint64_t)args.N, (uint64_t)ldb * 2, GEMM_BK, BN / 2,
                    CU_TENSOR_MAP_SWIZZLE_128B))
    return EMM_E_INVALID;
  static bool attr_done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_done[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(gemm_bf16_tc2_kernel<BN, STAGES>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return cuda_status(e, "gemm pair smem attribute");
    attr_done[dev & 63] = true;
  }
  args.num_m = (args.M + 2 * GEMM_BM - 1) / (2 * GEMM_BM);  // 256-row pair tiles
  args.num_n = (args.N + BN - 1) / BN;
  args.num_tiles = args.num_m * args.num_n;
  int pairs = sm_count() / 2;
  if (args.num_tiles < pairs) pairs = args.num_tiles;
  launch_pdl(gemm_bf16_tc2_kernel<BN, STAGES>, dim3(2 * pairs), dim3(GEMM_THREADS), Cfg::SMEM,
             stream, ta, tb, args);
  count_launch();
  EMM_CUDA_CHECK_LAUNCH("gemm_bf16_tc2_kernel launch");
  return EMM_OK;
}

}  // namespace emm

// EMM_GEMM_PAIR: 0 = never use CTA pairs, 2 = always (tests), default = when
// the 256x256 pair tiles still fill the machine
static int pair_mode() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EMM_GEMM_PAIR");
    v = (e && e[0] == '0') ? 0 : ((e && e[0] == '2') ? 2 : 1);
  }
  return v;
}

static bool splitk_bn64() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EMM_GEMM_SPLITK_BN64");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// EMM_GEMM_KS: force the split count of split-K GEMMs (experiments; 0 = model)
static int splitk_force() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EMM_GEMM_KS");
    v = e ? atoi(e) : 0;
  }
  return v;
}

// EMM_GEMM_KA: 64-column K atoms per pipeline stage of the decode-size
// split-K GEMMs (1, 2 or 4; needs K % (64 KA) == 0 and M <= 64)
static int splitk_ka() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EMM_GEMM_KA");
    v = e ? atoi(e) : SPLITK_KA_DEFAULT;
    if (v != 2 && v != 4) v = 1;
  }
  return v;
}

// EMM_GEMM_SKINNY=0: decode-size GEMMs on the 128-row-tile kernel instead
static int skinny_mode() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EMM_GEMM_SKINNY");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v;
}

static int splitk_mode() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EMM_GEMM_SPLITK");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v;
}

// per-device split-K workspace + self-resetting tile counters (allocated on
// first use, so a CUDA-graph capture after a warm-up call allocates nothing);
// split GEMMs of one device must be stream-ordered, which the library's
// callers guarantee (one stream per GPU)
bool emm::splitk_workspace(size_t ws_bytes, size_t n_cnt, cudaStream_t st, float** ws,
                           int** cnt) {
  struct Buf {
    float* ws = nullptr;
    size_t ws_bytes = 0;
    int* cnt = nullptr;
    size_t n_cnt = 0;
  };
  static std::map<int, Buf> bufs;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  cudaGetDevice(&dev);
  Buf& b = bufs[dev];
  if (b.ws_bytes < ws_bytes) {
    if (b.ws) {
      cudaStreamSynchronize(st);
      cudaFree(b.ws);
    }
    const size_t want = ws_bytes < (16u << 20) ? (16u << 20) : ws_bytes;
    if (cudaMalloc(&b.ws, want) != cudaSuccess) {
      emm_abi::set_error("split-K workspace allocation failed");
      b.ws = nullptr;
      b.ws_bytes = 0;
      return false;
    }
    b.ws_bytes = want;
  }
  if (b.n_cnt < n_cnt) {
    if (b.cnt) {
      cudaStreamSynchronize(st);
      cudaFree(b.cnt);
    }
    const size_t want = n_cnt < 4096 ? 4096 : n_cnt;
    if (cudaMalloc(&b.cnt, want * sizeof(int)) != cudaSuccess) {
      emm_abi::set_error("split-K counter allocation failed");
      b.cnt = nullptr;
      b.n_cnt = 0;
      return false;
    }
    cudaMemsetAsync(b.cnt, 0, want * sizeof(int), st);
    b.n_cnt = want;
  }
  *ws = b.ws;
  *cnt = b.cnt;
  return true;
}

extern "C" int emm_gemm_bf16_ex(const void* A, int64_t lda, const void* B, int64_t ldb,
                                void* C, int64_t ldc, int64_t M, int64_t N, int64_t K,
                                const emm_gemm_epilogue* e, void* stream) {
  using namespace emm;
  if (M <= 0 || N <= 0) return EMM_OK;
  const int epi = e ? e->kind : EMM_EPI_NONE;
  const bool qkv = epi == EMM_EPI_QKV_ROPE;
  if (!A || !B || (!C && !qkv) || K <= 0 || (N % 32) != 0 || (K % 8) != 0 || (lda % 8) != 0 ||
      (ldb % 8) != 0 || (!qkv && (ldc % 8) != 0) || (e && e->residual && (e->ldr % 8) != 0) ||
      (reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15) ||
      (reinterpret_cast<uintptr_t>(C) & 15) || M > (1ll << 31) || N > (1ll << 31)) {
    emm_abi::set_error("emm_gemm_bf16: need N%32==0, K%8==0, 16B-aligned pointers/pitches");
    return EMM_E_INVALID;
  }
  if (epi == EMM_EPI_GLU_SILU && (N % 256) != 0) {
    emm_abi::set_error("emm_gemm_bf16: GLU epilogue needs N % 256 == 0 (128-row interleave)");
    return EMM_E_INVALID;
  }
  if (qkv && (!e->q_out || !e->k_out || !e->v_out || !e->kv_row || (e->hd != 64 && e->hd != 128) ||
              N != (int64_t)(e->hq + 2 * e->hkv) * e->hd || (e->ld_q % 8) || (e->ld_kv % 8))) {
    emm_abi::set_error("emm_gemm_bf16: QKV epilogue needs q/k/v outputs, kv_row, hd 64/128, "
                       "N == (hq + 2 hkv) hd");
    return EMM_E_INVALID;
  }
  GemmArgs args{};
  args.M = (int)M;
  args.N = (int)N;
  args.K = (int)K;
  args.C = reinterpret_cast<__nv_bfloat16*>(C);
  args.ldc = ldc;
  args.epi = epi;
  if (e) {
    args.bias = reinterpret_cast<const __nv_bfloat16*>(e->bias);
    args.residual = reinterpret_cast<const __nv_bfloat16*>(e->residual);
    args.ldr = e->ldr;
    args.row_ss_in = e->row_ss_in;
    args.rms_inv_dim = e->rms_dim > 0 ? 1.f / (float)e->rms_dim : 0.f;
    args.rms_eps = e->rms_eps;
    args.row_ss_out = e->row_ss_out;
    args.row_ss_zero = e->row_ss_zero;
    args.q_out = reinterpret_cast<__nv_bfloat16*>(e->q_out);
    args.ld_q = e->ld_q;
    args.k_out = reinterpret_cast<__nv_bfloat16*>(e->k_out);
    args.v_out = reinterpret_cast<__nv_bfloat16*>(e->v_out);
    args.ld_kv = e->ld_kv;
    args.kv_row = e->kv_row;
    args.pos = e->pos;
    args.rope_cs = reinterpret_cast<const float2*>(e->rope_cs);
    args.hq = e->hq;
    args.hkv = e->hkv;
    args.hd = e->hd;
    args.pos_h = e->pos_h;
    args.pos_w = e->pos_w;
    args.rope2_cs = reinterpret_cast<const float2*>(e->rope2_cs);
    args.rope2_cols = e->rope2_cols;
    args.rope2_hd = e->rope2_hd;
    // 1-D RoPE: every pair in the first section
    args.mrope_s0 = e->pos_h ? e->mrope_t : (1 << 30);
    args.mrope_s1 = e->pos_h ? e->mrope_h : 0;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int64_t sms = sm_count();
  // decode-size M: the transposed weight-stream kernel (gemm_skinny.cu)
  if (M <= 64 && (K % 64) == 0 && !args.rope2_cs && skinny_mode() != 0) {
    SkinnyArgs sa{};
    sa.M = args.M;
    sa.N = args.N;
    sa.K = args.K;
    sa.C = args.C;
    sa.ldc = args.ldc;
    sa.bias = args.bias;
    sa.residual = args.residual;
    sa.ldr = args.ldr;
    sa.epi = args.epi;
    sa.row_ss_in = args.row_ss_in;
    sa.rms_inv_dim = args.rms_inv_dim;
    sa.rms_eps = args.rms_eps;
    sa.row_ss_out = args.row_ss_out;
    sa.row_ss_zero = args.row_ss_zero;
    sa.q_out = args.q_out;
    sa.ld_q = args.ld_q;
    sa.k_out = args.k_out;
    sa.v_out = args.v_out;
    sa.ld_kv = args.ld_kv;
    sa.kv_row = args.kv_row;
    sa.pos = args.pos;
    sa.rope_cs = args.rope_cs;
    sa.hq = args.hq;
    sa.hkv = args.hkv;
    sa.hd = args.hd;
    sa.pos_h = args.pos_h;
    sa.pos_w = args.pos_w;
    sa.mrope_s0 = args.mrope_s0;
    sa.mrope_s1 = args.mrope_s1;
    return launch_gemm_skinny(A, lda, B, ldb, sa, st);
  }
  // split-K when the (M, N) tiles cannot fill half the SMs and K is long
  // (decode-size M): the weight stream is then spread over ~all SMs
  {
    const int64_t tiles128 = ((M + 127) / 128) * ((N + 127) / 128);
    const int64_t nkb = (K + GEMM_BK - 1) / GEMM_BK;
    if (epi != EMM_EPI_GLU_SILU && tiles128 * 2 <= sms && nkb >= 8 && splitk_mode() != 0) {
      // BN = 64 tiles (non-QKV epilogues, K <= 8192: the o-projection):
      // twice the tiles, half the splits, so each item streams a longer K
      // range and the last arriver adds fewer partials (64 x 3584 x 3584:
      // 16.6 -> 12.5 us); the long-K down projection keeps BN = 128
      // (measured 3 % slower with 64)
      if (!qkv && N % 64 == 0 && K <= 8192 && splitk_bn64()) {
        const int64_t tiles64 = ((M + 127) / 128) * ((N + 63) / 64);
        int64_t ks = sms / tiles64;
        if (ks > nkb / 4) ks = nkb / 4;
        if (ks > 16) ks = 16;
        if (splitk_force() > 0) ks = splitk_force() < nkb ? splitk_force() : nkb;
        if (ks < 1) ks = 1;
        float* ws = nullptr;
        int* cnt = nullptr;
        if (!splitk_workspace((size_t)tiles64 * ks * 128 * 64 * 4, (size_t)tiles64, st, &ws,
                              &cnt))
          return EMM_E_CUDA;
        args.ksplit = (int)ks;
        args.ws = ks > 1 ? ws : nullptr;
        args.cnt = cnt;
        const int ka = M <= 64 ? splitk_ka() : 1;
        if (ka == 4 && K % (GEMM_BK * 4) == 0 && ks <= nkb / 4)
          return launch_gemm<64, 3, 4>(A, lda, B, ldb, args, st);
        if (ka == 2 && K % (GEMM_BK * 2) == 0 && ks <= nkb / 2)
          return launch_gemm<64, 6, 2>(A, lda, B, ldb, args, st);
        return launch_gemm<64, 8>(A, lda, B, ldb, args, st);
      }
      int64_t ks = sms / tiles128;
      if (ks > nkb / 4) ks = nkb / 4;
      if (ks > 16) ks = 16;
      if (splitk_force() > 0) ks = splitk_force() < nkb ? splitk_force() : nkb;
      if (ks >= 2) {
        float* ws = nullptr;
        int* cnt = nullptr;
        if (!splitk_workspace((size_t)tiles128 * ks * 128 * 128 * 4, (size_t)tiles128, st, &ws,
                              &cnt))
          return EMM_E_CUDA;
        args.ksplit = (int)ks;
        args.ws = ws;
        args.cnt = cnt;
        const int ka = M <= 64 ? splitk_ka() : 1;
        if (ka == 4 && K % (GEMM_BK * 4) == 0 && ks <= nkb / 4)
          return launch_gemm<128, 2, 4>(A, lda, B, ldb, args, st);
        if (ka == 2 && K % (GEMM_BK * 2) == 0 && ks <= nkb / 2)
          return launch_gemm<128, 4, 2>(A, lda, B, ldb, args, st);
        return launch_gemm<128, 6>(A, lda, B, ldb, args, st);
      }
    }
  }
  // wave-quantisation aware tile choice: est ~ waves * (BN + fixed per-tile cost)
  const int64_t t256 = ((M + 127) / 128) * ((N + 255) / 256);
  const int64_t t128 = ((M + 127) / 128) * ((N + 127) / 128);
  const int64_t est256 = ((t256 + sms - 1) / sms) * (256 + 32);
  const int64_t est128 = ((t128 + sms - 1) / sms) * (128 + 32);
  const bool pick256 = epi == EMM_EPI_GLU_SILU || (qkv && (256 % e->hd) == 0 && est256 <= est128) ||
                       (!qkv && est256 <= est128);
  if (pick256 && pair_mode() != 0) {
    // the pair kernel stages half of B per SM (128 instead of 85 FLOP/byte)
    // and measured faster than the single-CTA BN=256 kernel even where the
    // wave count says "equal or one more" (tools/gemm_pair_choice.py: 5-27 %
    // on the decoder shapes, +0.9 % on C3): take it for every M above one
    // pair tile; small M keeps the wave comparison
    const int64_t tpair = ((M + 255) / 256) * ((N + 255) / 256);
    const int64_t est_pair = ((tpair + sms / 2 - 1) / (sms / 2)) * (256 + 32);
    if (M > 256 || est_pair <= est256 || pair_mode() == 2)
      return launch_gemm_pair<256, GEMM_PAIR_STAGES>(A, lda, B, ldb, args, st);
  }
  if (pick256)
    return launch_gemm<256, 4>(A, lda, B, ldb, args, st);
  return launch_gemm<128, 6>(A, lda, B, ldb, args, st);
}

extern "C" int emm_gemm_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, void* C,
                             int64_t ldc, int64_t M, int64_t N, int64_t K, const void* bias,
                             const void* residual, int64_t ldr, int epi, void* stream) {
  emm_gemm_epilogue e{};
  e.kind = epi;
  e.bias = bias;
  e.residual = residual;
  e.ldr = ldr;
  return emm_gemm_bf16_ex(A, lda, B, ldb, C, ldc, M, N, K, &e, stream);
}
