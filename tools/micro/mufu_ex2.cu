#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cstdio>
__global__ void k_f32(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a[i])); a[i] = y * -0.5f; }
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_f16x2(float* out, int iters) {
  uint32_t a[8];
  for (int i = 0; i < 8; ++i) { __half2 h = __floats2half2_rn(-0.001f * (threadIdx.x + i), -0.002f); a[i] = *reinterpret_cast<uint32_t*>(&h); }
  const uint32_t mh = 0xB800B800u; // -0.5 half2
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { uint32_t y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(a[i])); asm volatile("mul.rn.f16x2 %0, %1, %2;" : "=r"(a[i]) : "r"(y), "r"(mh)); }
  }
  float s = 0; for (int i = 0; i < 8; ++i) { __half2 h = *reinterpret_cast<__half2*>(&a[i]); s += __low2float(h) + __high2float(h); }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_bf16x2(float* out, int iters) {
  uint32_t a[8];
  for (int i = 0; i < 8; ++i) { __nv_bfloat162 h = __floats2bfloat162_rn(-0.001f * (threadIdx.x + i), -0.002f); a[i] = *reinterpret_cast<uint32_t*>(&h); }
  const uint32_t mh = 0xBF00BF00u; // -0.5 bf16x2
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { uint32_t y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(a[i])); asm volatile("mul.rn.bf16x2 %0, %1, %2;" : "=r"(a[i]) : "r"(y), "r"(mh)); }
  }
  float s = 0; for (int i = 0; i < 8; ++i) { __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&a[i]); s += __low2float(h) + __high2float(h); }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(e0); k_f32<<<148 * 8, 1024>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double n = 148.0 * 8 * 1024 * iters * 8;
    printf("f32   ex2: %.1f Gexp/s  %.2f exp/clk/SM @1.9GHz\n", n / ms / 1e6, n / (ms * 1e-3) / 148 / 1.9e9);
    cudaEventRecord(e0); k_f16x2<<<148 * 8, 1024>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("f16x2 ex2: %.1f Gexp/s  %.2f exp/clk/SM (values, x2)\n", 2 * n / ms / 1e6, 2 * n / (ms * 1e-3) / 148 / 1.9e9);
    cudaEventRecord(e0); k_bf16x2<<<148 * 8, 1024>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("bf16x2 ex2: %.1f Gexp/s  %.2f exp/clk/SM (values, x2)\n", 2 * n / ms / 1e6, 2 * n / (ms * 1e-3) / 148 / 1.9e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
