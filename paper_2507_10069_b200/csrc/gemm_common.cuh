// gemm_common.cuh — pieces shared by the two tcgen05 GEMM kernels:
// gemm_tc.cu (tiles of 128 activation rows) and gemm_skinny.cu (decode-size
// M <= 64, computed transposed so the weight rows fill the MMA's 128 lanes).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace emm {

__device__ __forceinline__ float act_gelu_tanh(float x) {
  // 0.5 x (1 + tanh(u)) = x * sigmoid(2u)
  const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
  return __fdividef(x, 1.f + __expf(-2.f * u));
}
__device__ __forceinline__ float act_quick_gelu(float x) {
  return __fdividef(x, 1.f + __expf(-1.702f * x));
}
__device__ __forceinline__ float act_gelu_erf(float x) {
  return 0.5f * x * (1.f + erff(x * 0.7071067811865476f));
}
__device__ __forceinline__ float act_silu(float x) { return __fdividef(x, 1.f + __expf(-x)); }

// Arguments of the decode-size kernel (gemm_skinny.cu).  A "unit" is one
// 128-row tile of the weight matrix B (EMM_EPI_GLU_SILU: a 256-row gate/up
// pair, the gate rows first); every unit's K range is split ks ways.
struct SkinnyArgs {
  int M, N, K;
  int units, ks;
  __nv_bfloat16* C;
  int64_t ldc;
  const __nv_bfloat16* bias;
  const __nv_bfloat16* residual;
  int64_t ldr;
  int epi;
  const float* row_ss_in;
  float rms_inv_dim, rms_eps;
  float* row_ss_out;
  float* row_ss_zero;
  __nv_bfloat16* q_out;
  int64_t ld_q;
  __nv_bfloat16* k_out;
  __nv_bfloat16* v_out;
  int64_t ld_kv;
  const int32_t* kv_row;
  const int32_t* pos;
  const float2* rope_cs;
  int hq, hkv, hd;
  const int32_t* pos_h;
  const int32_t* pos_w;
  int mrope_s0, mrope_s1;
  // ks > 1: partials [unit][ks][G][M][128] fp32 and 2 x units counters
  // (arrivals, then completions; the last completion re-zeroes both)
  float* ws;
  int* cnt;
  int dbg;  // EMM_SKINNY_DBG experiments: 1 no epilogue, 2 no stores, 4 no residual
  unsigned long long* prof;  // EMM_SKINNY_PROF: per-CTA %globaltimer stamps (8 per CTA)
};

// Launch the decode-size kernel; A = activations [M, K] (lda), B = weights
// [N, K] (ldb).  args.units / ks / ws / cnt are filled by the caller.
int launch_gemm_skinny(const void* A, int64_t lda, const void* B, int64_t ldb,
                       const SkinnyArgs& args, cudaStream_t stream);
// per-device split-K workspace and self-resetting counters (gemm_tc.cu)
bool splitk_workspace(size_t ws_bytes, size_t n_cnt, cudaStream_t st, float** ws, int** cnt);

}  // namespace emm
