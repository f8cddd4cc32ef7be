// gemm_skinny.cu — decode-size GEMMs (M <= 64 activation rows) on tcgen05,
// computed transposed as a weight stream:
//
//   D^T[n, m] = B[n, :] . A[m, :]      C[m, n] = epilogue(D[m, n])
//
// The weight rows fill the MMA's 128 lanes (M = 128) and the few activation
// rows are its N (32 or 64), so every staged byte of B is a byte the MMA
// uses — the 128-row activation tiles of gemm_tc.cu stage 2-4x the A bytes
// and spend half of every accumulator on rows >= M.  A decode step streams
// the whole decoder from HBM once (profiles/r02/gemm_stream.txt), so this
// kernel's roofline is the HBM copy rate of B.
//
// Work: a unit is one 128-row tile of B (EMM_EPI_GLU_SILU: a 256-row gate /
// up pair, both accumulated, gate rows first); its K range is split ks ways
// so units x ks items cover the SMs (o-proj 28 x 5, QKV 36 x 4, down 28 x 5,
// gate/up 148 x 1).  With ks > 1 every item stores its fp32 partial tile,
// arrives on the unit's counter and waits for the other ks - 1 (all items
// are resident: units x ks <= SMs, one CTA per SM); then item s reduces the
// 8-row groups s, s + ks, ... of the tile in a fixed split order (results do
// not depend on arrival order) and runs the epilogue for them.
//
// Per CTA: warp 0 TMA producer (B tiles 128 x 64 and the A tile NT x 64 per
// K atom, SW128), warp 1 MMA issuer (tcgen05.mma M=128 N=NT K=16), warp 2
// TMEM allocator (2 accumulators, double-buffered across items), warps 4..7
// epilogue (TMEM lane n = weight row n of the unit; 32 lanes = 32 adjacent
// output columns, so each output row segment is one 64-byte store per warp).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdlib.h>

#include "../../include/emm.h"
#include "gemm_common.cuh"
#include "ptx.cuh"
#include "runtime.h"

namespace emm {

constexpr int SK_ROWS = 128;  // weight rows per tile = TMEM lanes
constexpr int SK_BK = 64;     // K per atom (128 B rows, SW128)
constexpr int SK_THREADS = 256;
constexpr int SK_PIPE_BYTES = 200 * 1024;
constexpr int SK_RCH = 8;     // rows per reduction group (ks > 1)

template <int NT, int G, int KA>
struct SkCfg {
  static constexpr int W_ATOM = SK_ROWS * SK_BK * 2;  // 16 KiB
  static constexpr int X_ATOM = NT * SK_BK * 2;
  static constexpr int W_BYTES = W_ATOM * G * KA;
  static constexpr int STAGE_BYTES = W_BYTES + X_ATOM * KA;
  static constexpr int STAGES_FIT = SK_PIPE_BYTES / STAGE_BYTES;
  static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
  static constexpr int XCH_OFF = STAGES * STAGE_BYTES;  // epilogue staging, 3 x [16][128]
  static constexpr int XCH_BYTES = 3 * 16 * SK_ROWS * 4;
  static constexpr int ROWS_OFF = XCH_OFF + XCH_BYTES;  // SkRows
  static constexpr int BAR_OFF = ROWS_OFF + 1280;
  static constexpr int SMEM = BAR_OFF + (2 * STAGES + 4) * 8 + 16 + 1024;
  static constexpr int ACC_COLS = G * NT;
  static constexpr int TMEM_COLS = 2 * ACC_COLS;
};

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SK_STAMP(i)                                                               \
  do {                                                                            \
    if (args.prof) args.prof[blockIdx.x * 16 + (i)] = gtime();                     \
  } while (0)

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Per-row values of the activation rows, staged once per CTA in shared
// memory while the first weight tiles stream in (M <= 64)
struct SkRows {
  float rs[64];    // folded RMSNorm scale (1 without row_ss_in)
  int pos[64], pos_h[64], pos_w[64], kv_row[64];
};

template <int KIND>
__device__ __forceinline__ float sk_act(float x) {
  if constexpr (KIND == EMM_EPI_GELU_TANH) return act_gelu_tanh(x);
  else if constexpr (KIND == EMM_EPI_QUICK_GELU) return act_quick_gelu(x);
  else if constexpr (KIND == EMM_EPI_GELU_ERF) return act_gelu_erf(x);
  else return x;
}

// The epilogue runs once per launch on every SM, so its instructions are
// fetched cold, and one warp per scheduler leaves no other warp to hide a
// dependent chain: it is a short unrolled staging step followed by a per-row
// loop unrolled 4x (an unrolled multi-kind epilogue measured several us of
// instruction-fetch stalls per launch, a rolled one ~100 cycles per row of
// dependent latency; profiles/r02/gemm_skinny.txt).
//
// Staging (this thread = weight row n_local of unit u, rows m0 .. m0+15):
//   xs0[j] = acc * rs[m] + bias            (GLU: gate)
//   xs1[j] = up * rs[m] + bias_up (GLU) | residual[m][n] | cos (QKV)
//   xs2[j] = sin (QKV)
struct SkStage {
  float* xs0;
  float* xs1;
  float* xs2;
};

template <int G, int CW>
__device__ __forceinline__ void sk_stage(const SkinnyArgs& a, const SkStage& st, int n_local,
                                         int m0, const float (&v)[G][CW], const SkRows* rows,
                                         float b0, float b1, const float (&rr)[CW]) {
#pragma unroll
  for (int j = 0; j < CW; ++j) {
    const float rs = rows->rs[m0 + j < a.M ? m0 + j : 0];
    st.xs0[j * SK_ROWS + n_local] = v[0][j] * rs + b0;
    if constexpr (G == 2) {
      st.xs1[j * SK_ROWS + n_local] = v[G - 1][j] * rs + b1;
    } else {
      st.xs1[j * SK_ROWS + n_local] = rr[j];
    }
  }
}

// rotary (cos, sin) of rows m0 .. m0+CW-1 for this thread's pair
template <int CW>
__device__ __forceinline__ void sk_stage_rope(const SkinnyArgs& a, const SkStage& st, int n_local,
                                              int m0, const SkRows* rows) {
  const int half = a.hd >> 1;
  const int i = n_local & (half - 1);
  const int s0 = a.mrope_s0, s01 = a.mrope_s0 + a.mrope_s1;
  const int* pv = i < s0 ? rows->pos : (i < s01 ? rows->pos_h : rows->pos_w);
  float2 cs[CW];
#pragma unroll
  for (int j = 0; j < CW; ++j)
    cs[j] = (a.rope_cs && m0 + j < a.M) ? __ldg(a.rope_cs + (int64_t)pv[m0 + j] * half + i)
                                        : make_float2(1.f, 0.f);
#pragma unroll
  for (int j = 0; j < CW; ++j) {
    st.xs1[j * SK_ROWS + n_local] = cs[j].x;
    st.xs2[j * SK_ROWS + n_local] = cs[j].y;
  }
}

// Rows m0 .. m0+cnt-1 of this thread's output column from the staged values.
// Same arithmetic as gemm_tc.cu's epilogue_tile: folded RMSNorm scale, bias,
// activation / SwiGLU / RoPE, residual, sum of squares of the stored bf16
// values.
template <int KIND>
__device__ __forceinline__ void sk_rows(const SkinnyArgs& a, const SkStage& st, int u,
                                        int n_local, int m0, int cnt, const SkRows* rows) {
  if constexpr (KIND == EMM_EPI_GLU_SILU) {
    __nv_bfloat16* dst = a.C + (int64_t)m0 * a.ldc + u * SK_ROWS + n_local;
#pragma unroll 4
    for (int j = 0; j < cnt; ++j) {
      const float g = st.xs0[j * SK_ROWS + n_local], up = st.xs1[j * SK_ROWS + n_local];
      dst[(int64_t)j * a.ldc] = __float2bfloat16(act_silu(g) * up);
    }
  } else if constexpr (KIND == EMM_EPI_QKV_ROPE) {
    const int n = u * SK_ROWS + n_local;
    if (n >= a.N) return;
    const int hd = a.hd, half = hd >> 1;
    const int q_dim = a.hq * hd, kv_dim = a.hkv * hd;
    const int col_h = n - (n_local & (hd - 1));  // first column of this head
    const int sect = col_h < q_dim ? 0 : (col_h < q_dim + kv_dim ? 1 : 2);
    const bool first = (n_local & half) == 0;
    const float sgn = first ? -1.f : 1.f;
    __nv_bfloat16* base = sect == 0 ? a.q_out + n
                                    : (sect == 1 ? a.k_out + (n - q_dim)
                                                 : a.v_out + (n - q_dim - kv_dim));
    const int64_t ld = sect == 0 ? a.ld_q : a.ld_kv;
#pragma unroll 4
    for (int j = 0; j < cnt; ++j) {
      const int m = m0 + j;
      const float x = st.xs0[j * SK_ROWS + n_local];
      float o = x;
      if (sect < 2 && a.rope_cs) {
        // the rotate-half partner: column n ^ half of the same head
        const float y = st.xs0[j * SK_ROWS + (n_local ^ half)];
        o = x * st.xs1[j * SK_ROWS + n_local] + sgn * y * st.xs2[j * SK_ROWS + n_local];
      }
      base[(int64_t)(sect == 0 ? m : rows->kv_row[m]) * ld] = __float2bfloat16(o);
    }
  } else {
    const int n = u * SK_ROWS + n_local;
    const bool n_ok = n < a.N;
    __nv_bfloat16* dst = a.C + (int64_t)m0 * a.ldc + n;
#pragma unroll 4
    for (int j = 0; j < cnt; ++j) {
      const float val = sk_act<KIND>(st.xs0[j * SK_ROWS + n_local]) + st.xs1[j * SK_ROWS + n_local];
      float q = 0.f;
      if (n_ok) {
        const __nv_bfloat16 h = __float2bfloat16(val);
        if (!(a.dbg & 2)) dst[(int64_t)j * a.ldc] = h;
        q = __bfloat162float(h);
      }
      if (a.row_ss_out) {  // warp-uniform
        float s = q * q;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if ((n_local & 31) == 0) atomicAdd(a.row_ss_out + m0 + j, s);
      }
    }
  }
}

// stage rows m0 .. m0+CW-1 (accumulator values v, residual rr) and write them
template <int G, int CW>
__device__ __forceinline__ void skinny_epilogue(const SkinnyArgs& a, const SkStage& st, int u,
                                                int n_local, int m0, const float (&v)[G][CW],
                                                const SkRows* rows, float b0, float b1,
                                                const float (&rr)[CW]) {
  const int cnt = a.M - m0 < CW ? a.M - m0 : CW;
  if (a.row_ss_zero && u == 0 && n_local < cnt) a.row_ss_zero[m0 + n_local] = 0.f;
  const bool qkv = G == 1 && a.epi == EMM_EPI_QKV_ROPE;
  if (qkv) epi_bar();  // the previous rows' partner reads are done
  sk_stage<G, CW>(a, st, n_local, m0, v, rows, b0, b1, rr);
  if constexpr (G == 2) {
    sk_rows<EMM_EPI_GLU_SILU>(a, st, u, n_local, m0, cnt, rows);
  } else {
    if (qkv) {
      sk_stage_rope<CW>(a, st, n_local, m0, rows);
      epi_bar();
      sk_rows<EMM_EPI_QKV_ROPE>(a, st, u, n_local, m0, cnt, rows);
      return;
    }
    switch (a.epi) {
      case EMM_EPI_GELU_TANH: sk_rows<EMM_EPI_GELU_TANH>(a, st, u, n_local, m0, cnt, rows); break;
      case EMM_EPI_QUICK_GELU: sk_rows<EMM_EPI_QUICK_GELU>(a, st, u, n_local, m0, cnt, rows); break;
      case EMM_EPI_GELU_ERF: sk_rows<EMM_EPI_GELU_ERF>(a, st, u, n_local, m0, cnt, rows); break;
      default: sk_rows<EMM_EPI_NONE>(a, st, u, n_local, m0, cnt, rows); break;
    }
  }
}

// residual values of rows m0 .. m0+CW-1 of column n (0 where absent)
template <int CW>
__device__ __forceinline__ void load_residual(const SkinnyArgs& a, int n, int m0, float (&rr)[CW]) {
  const bool ok = a.residual && n < a.N && !(a.dbg & 4);
#pragma unroll
  for (int j = 0; j < CW; ++j)
    rr[j] = (ok && m0 + j < a.M) ? __bfloat162float(a.residual[(int64_t)(m0 + j) * a.ldr + n])
                                 : 0.f;
}

__device__ __forceinline__ void red_release_gpu(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int NT, int G, int KA>
__global__ void __launch_bounds__(SK_THREADS, 1)
    gemm_skinny_kernel(const __grid_constant__ CUtensorMap tmW,
                       const __grid_constant__ CUtensorMap tmX, const SkinnyArgs args) {
  using Cfg = SkCfg<NT, G, KA>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* xch = reinterpret_cast<float*>(smem + Cfg::XCH_OFF);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) SK_STAMP(0);
  if (threadIdx.x == 0) {
    tma_prefetch(&tmW);
    tma_prefetch(&tmX);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) SK_STAMP(1);
  const uint32_t tmem_base = *tmem_slot;
  const int nst = args.K / (SK_BK * KA);  // pipeline stages along K
  const int ks = args.ks;
  const int items = args.units * ks;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int w = blockIdx.x; w < items; w += gridDim.x) {
        const int u = w / ks, s = w - u * ks;
        const int k0 = s * nst / ks, k1 = (s + 1) * nst / ks;
        for (int kb = k0; kb < k1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * Cfg::STAGE_BYTES;
          mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES);
#pragma unroll
          for (int a = 0; a < KA; ++a) {
            const int kc = (kb * KA + a) * SK_BK;
#pragma unroll
            for (int g = 0; g < G; ++g)
              tma_load_2d(st + (a * G + g) * Cfg::W_ATOM, &tmW, &full[stage], kc,
                          (u * G + g) * SK_ROWS);
            tma_load_2d(st + Cfg::W_BYTES + a * Cfg::X_ATOM, &tmX, &full[stage], kc, 0);
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
      constexpr uint32_t idesc = idesc_bf16_f32(SK_ROWS, NT, false, false);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int w = blockIdx.x; w < items; w += gridDim.x, ++it) {
        const int s = w % ks;
        const int k0 = s * nst / ks, k1 = (s + 1) * nst / ks;
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * Cfg::ACC_COLS;
        for (int kb = k0; kb < k1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (it == 0 && kb == k0) SK_STAMP(2);
          const uint32_t base = smem_u32(smem + stage * Cfg::STAGE_BYTES);
#pragma unroll
          for (int a = 0; a < KA; ++a) {
            const uint64_t bdesc = desc_sw128_kmajor(base + Cfg::W_BYTES + a * Cfg::X_ATOM);
#pragma unroll
            for (int g = 0; g < G; ++g) {
              const uint64_t adesc = desc_sw128_kmajor(base + (a * G + g) * Cfg::W_ATOM);
#pragma unroll
              for (int k = 0; k < SK_BK / 16; ++k)
                mma_ss(d_tmem + g * NT, adesc + (uint64_t)(2 * k), bdesc + (uint64_t)(2 * k),
                       idesc, (kb != k0) || (a != 0) || (k != 0));
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
    const int ew = warp & 3;
    const int n_local = ew * 32 + lane;
    SkRows* rows = reinterpret_cast<SkRows*>(smem + Cfg::ROWS_OFF);
    const SkStage stg{xch, xch + 16 * SK_ROWS, xch + 32 * SK_ROWS};
    {
      const int e = threadIdx.x - 128;
      if (e < args.M) {
        rows->rs[e] = args.row_ss_in
                          ? rsqrtf(__ldg(args.row_ss_in + e) * args.rms_inv_dim + args.rms_eps)
                          : 1.f;
        if (args.epi == EMM_EPI_QKV_ROPE) {
          const int p = args.pos ? args.pos[e] : 0;
          rows->pos[e] = p;
          rows->pos_h[e] = args.pos_h ? args.pos_h[e] : p;
          rows->pos_w[e] = args.pos_w ? args.pos_w[e] : p;
          rows->kv_row[e] = args.kv_row[e];
        }
      }
      epi_bar();
    }
    int it = 0;
    for (int w = blockIdx.x; w < items; w += gridDim.x, ++it) {
      const int u = w / ks, s = w - u * ks;
      const int acc = it & 1;
      float b0 = 0.f, b1 = 0.f;  // bias, loaded before the accumulator is ready
      if (args.bias) {
        if (G == 2) {
          b0 = __bfloat162float(args.bias[u * 2 * SK_ROWS + n_local]);
          b1 = __bfloat162float(args.bias[u * 2 * SK_ROWS + SK_ROWS + n_local]);
        } else if (u * SK_ROWS + n_local < args.N) {
          b0 = __bfloat162float(args.bias[u * SK_ROWS + n_local]);
        }
      }
      const uint32_t t_base =
          tmem_base + ((uint32_t)(ew * 32) << 16) + (uint32_t)(acc * Cfg::ACC_COLS);
      if (args.dbg & 1) {
        mbar_wait(&tfull[acc], (it >> 1) & 1);
        tc_fence_after();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      } else if (ks == 1) {
        const int n = u * SK_ROWS + n_local;
        float rr[16];
        load_residual<16>(args, n, 0, rr);
        mbar_wait(&tfull[acc], (it >> 1) & 1);
        tc_fence_after();
        if (threadIdx.x == 128 && it == 0) SK_STAMP(3);
#pragma unroll 1
        for (int m0 = 0; m0 < args.M; m0 += 16) {
          uint32_t r[G][16];
#pragma unroll
          for (int g = 0; g < G; ++g) tmem_ld16(t_base + g * NT + m0, r[g]);
          float rn[16];  // the next chunk's residual, in flight during this one
          load_residual<16>(args, n, m0 + 16, rn);
          tmem_wait_ld();
          float v[G][16];
#pragma unroll
          for (int g = 0; g < G; ++g)
#pragma unroll
            for (int j = 0; j < 16; ++j) v[g][j] = __uint_as_float(r[g][j]);
          skinny_epilogue<G, 16>(args, stg, u, n_local, m0, v, rows, b0, b1, rr);
#pragma unroll
          for (int j = 0; j < 16; ++j) rr[j] = rn[j];
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      } else {
        // this item reduces the 8-row groups s, s + ks, ...
        const int n = u * SK_ROWS + n_local;
        float rr[SK_RCH];
        load_residual<SK_RCH>(args, n, s * SK_RCH, rr);
        mbar_wait(&tfull[acc], (it >> 1) & 1);
        tc_fence_after();
        if (threadIdx.x == 128 && it == 0) SK_STAMP(3);
        const size_t tile = (size_t)args.M * SK_ROWS;  // one accumulator's partial
        float* unit_ws = args.ws + (size_t)u * ks * G * tile;
        float* mine = unit_ws + (size_t)s * G * tile;
#pragma unroll 1
        for (int m0 = 0; m0 < args.M; m0 += 16) {
          uint32_t r[G][16];
#pragma unroll
          for (int g = 0; g < G; ++g) tmem_ld16(t_base + g * NT + m0, r[g]);
          tmem_wait_ld();
#pragma unroll
          for (int g = 0; g < G; ++g)
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (m0 + j < args.M)
                __stcg(mine + g * tile + (size_t)(m0 + j) * SK_ROWS + n_local,
                       __uint_as_float(r[g][j]));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        epi_bar();
        if (threadIdx.x == 128) {
          SK_STAMP(4);
          red_release_gpu(args.cnt + u, 1);  // publishes the 128 threads' partials
          while (ld_acquire_gpu(args.cnt + u) < ks) __nanosleep(20);
          SK_STAMP(5);
        }
        epi_bar();
        // reduce in split order 0 .. ks-1 (independent of arrival order)
#pragma unroll 1
        for (int m0 = s * SK_RCH; m0 < args.M; m0 += ks * SK_RCH) {
          float v[G][SK_RCH];
#pragma unroll
          for (int g = 0; g < G; ++g)
#pragma unroll
            for (int j = 0; j < SK_RCH; ++j) v[g][j] = 0.f;
#pragma unroll 1
          for (int p0 = 0; p0 < ks; p0 += 8) {
            float t[8][G][SK_RCH];
#pragma unroll
            for (int q = 0; q < 8; ++q)
#pragma unroll
              for (int g = 0; g < G; ++g)
#pragma unroll
                for (int j = 0; j < SK_RCH; ++j)
                  t[q][g][j] = (p0 + q < ks && m0 + j < args.M)
                                   ? __ldcg(unit_ws + ((size_t)(p0 + q) * G + g) * tile +
                                            (size_t)(m0 + j) * SK_ROWS + n_local)
                                   : 0.f;
#pragma unroll
            for (int q = 0; q < 8; ++q)
#pragma unroll
              for (int g = 0; g < G; ++g)
#pragma unroll
                for (int j = 0; j < SK_RCH; ++j)
                  if (p0 + q < ks) v[g][j] += t[q][g][j];
          }
          float rn[SK_RCH];
          load_residual<SK_RCH>(args, n, m0 + ks * SK_RCH, rn);
          skinny_epilogue<G, SK_RCH>(args, stg, u, n_local, m0, v, rows, b0, b1, rr);
#pragma unroll
          for (int j = 0; j < SK_RCH; ++j) rr[j] = rn[j];
        }
        epi_bar();
        if (threadIdx.x == 128) {
          if (atomicAdd(args.cnt + args.units + u, 1) == ks - 1) {
            args.cnt[u] = 0;  // ready for the next launch
            args.cnt[args.units + u] = 0;
          }
        }
      }
    }
  }
  if (threadIdx.x == 128) SK_STAMP(6);
  if (threadIdx.x == 0) SK_STAMP(9);
  __syncthreads();
  if (threadIdx.x == 128) SK_STAMP(7);
  if (threadIdx.x == 0) SK_STAMP(8);
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

template <int NT, int G, int KA>
static int launch_skinny_t(const void* A, int64_t lda, const void* B, int64_t ldb,
                           const SkinnyArgs& args, cudaStream_t stream) {
  using Cfg = SkCfg<NT, G, KA>;
  CUtensorMap tw, tx;
  if (!make_tmap_2d(&tw, B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)args.K,
                    (uint64_t)args.N, (uint64_t)ldb * 2, SK_BK, SK_ROWS,
                    CU_TENSOR_MAP_SWIZZLE_128B))
    return EMM_E_INVALID;
  if (!make_tmap_2d(&tx, A, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)args.K,
                    (uint64_t)args.M, (uint64_t)lda * 2, SK_BK, NT, CU_TENSOR_MAP_SWIZZLE_128B))
    return EMM_E_INVALID;
  static bool attr_done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_done[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(gemm_skinny_kernel<NT, G, KA>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return cuda_status(e, "gemm skinny smem attribute");
    attr_done[dev & 63] = true;
  }
  const SkinnyArgs& a = args;
  const int items = a.units * a.ks;
  const int grid = items < sm_count() ? items : sm_count();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(SK_THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  cudaLaunchKernelEx(&cfg, gemm_skinny_kernel<NT, G, KA>, tw, tx, a);
  count_launch();
  EMM_CUDA_CHECK_LAUNCH("gemm_skinny_kernel launch");
  return EMM_OK;
}

// EMM_SKINNY_PROF=1: per-CTA timestamps of the last launch (tools/skinny_prof.py)
static unsigned long long* g_prof = nullptr;
static unsigned long long* skinny_prof_buf() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("EMM_SKINNY_PROF");
    on = (e && e[0] == '1') ? 1 : 0;
    if (on && cudaMalloc(&g_prof, 16 * 1024 * sizeof(unsigned long long)) != cudaSuccess) on = 0;
  }
  return on ? g_prof : nullptr;
}

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

int launch_gemm_skinny(const void* A, int64_t lda, const void* B, int64_t ldb,
                       const SkinnyArgs& in, cudaStream_t stream) {
  static const int ka_env = env_int("EMM_SKINNY_KA", 1);
  static const int ks_env = env_int("EMM_SKINNY_KS", 0);
  static const int dbg_env = env_int("EMM_SKINNY_DBG", 0);
  SkinnyArgs args = in;
  const bool glu = args.epi == EMM_EPI_GLU_SILU;
  const int G = glu ? 2 : 1;
  const int ka = (!glu && ka_env == 2 && args.K % (2 * SK_BK) == 0) ? 2 : 1;
  const int nst = args.K / (SK_BK * ka);
  const int sms = sm_count();
  args.units = glu ? args.N / (2 * SK_ROWS) : (args.N + SK_ROWS - 1) / SK_ROWS;
  // split K when the units leave more than half the SMs idle; every split
  // keeps >= 4 atoms of K and units x ks <= SMs (the splits of a unit wait
  // for each other, so all of them must be resident)
  int ks = 1;
  if (args.units * 2 <= sms) {
    ks = sms / args.units;
    if (ks > args.K / (SK_BK * 4)) ks = args.K / (SK_BK * 4);
    if (ks > 16) ks = 16;
  }
  if (ks_env > 0) ks = ks_env * args.units <= sms ? ks_env : sms / args.units;
  if (ks > nst) ks = nst;
  if (ks < 1) ks = 1;
  args.ks = ks;
  args.dbg = dbg_env;
  args.prof = skinny_prof_buf();
  args.ws = nullptr;
  args.cnt = nullptr;
  if (ks > 1) {
    const size_t ws_bytes = (size_t)args.units * ks * G * args.M * SK_ROWS * 4;
    if (!splitk_workspace(ws_bytes, (size_t)2 * args.units, stream, &args.ws, &args.cnt))
      return EMM_E_CUDA;
  }
  if (args.M <= 32) {
    if (glu) return launch_skinny_t<32, 2, 1>(A, lda, B, ldb, args, stream);
    if (ka == 2) return launch_skinny_t<32, 1, 2>(A, lda, B, ldb, args, stream);
    return launch_skinny_t<32, 1, 1>(A, lda, B, ldb, args, stream);
  }
  if (glu) return launch_skinny_t<64, 2, 1>(A, lda, B, ldb, args, stream);
  if (ka == 2) return launch_skinny_t<64, 1, 2>(A, lda, B, ldb, args, stream);
  return launch_skinny_t<64, 1, 1>(A, lda, B, ldb, args, stream);
}

}  // namespace emm

extern "C" int emm_skinny_prof_read(unsigned long long* host, int n) {
  if (!emm::g_prof || n > 16 * 1024) return -1;
  return cudaMemcpy(host, emm::g_prof, (size_t)n * 8, cudaMemcpyDeviceToHost) == cudaSuccess ? 0
                                                                                          : -1;
}
