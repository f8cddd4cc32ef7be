// tma_stream_probe.cu — how fast can one CTA per SM stream a decode-size
// weight matrix W[N][K] (bf16) out of HBM through TMA, with no math?  The
// ceiling for the split-K decode GEMMs (profiles/r02/gemm_stream.txt).
//
// Every CTA owns one (row tile, k range) item: rows [r0, r0+R) x k [k0, k1),
// loaded as boxes of (64 k x R rows, SWIZZLE_128B) — KA boxes per stage —
// into a ring of S stages; a consumer warp releases each stage as soon as it
// lands.  Timed over rotating copies of W (> L2 in total).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_stream_probe \
//        tools/tma_stream_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n}\n" ::"r"(su32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0,
                                      int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(su32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}

struct P {
  int N, K, R, ks, S, KA, tiles;
};

__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, P p,
                                                       int* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = raw + ((1024 - (su32(raw) & 1023)) & 1023);
  const int box = p.R * 128;
  const int stage_bytes = box * p.KA;
  uint64_t* full = (uint64_t*)(sm + p.S * stage_bytes);
  uint64_t* empty = full + p.S;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nkb = p.K / (64 * p.KA);
  for (int w = blockIdx.x; w < p.tiles * p.ks; w += gridDim.x) {
    const int t = w / p.ks, s_ = w % p.ks;
    const int kb0 = s_ * nkb / p.ks, kb1 = (s_ + 1) * nkb / p.ks;
    // per-item ring restart keeps the probe simple (one item per CTA anyway)
    if (threadIdx.x == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&empty[st], ph ^ 1);
        mbar_expect(&full[st], stage_bytes);
        for (int a = 0; a < p.KA; ++a)
          tma2d(sm + st * stage_bytes + a * box, &tm, &full[st], (kb * p.KA + a) * 64, t * p.R);
        if (++st == p.S) {
          st = 0;
          ph ^= 1;
        }
      }
    } else if (threadIdx.x == 32) {
      int st = 0;
      uint32_t ph = 0;
      int acc = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[st], ph);
        acc += sm[st * stage_bytes];
        mbar_arrive(&empty[st]);
        if (++st == p.S) {
          st = 0;
          ph ^= 1;
        }
      }
      if (acc == 12345) sink[0] = acc;
    }
    __syncthreads();
    // re-init barriers for the next item of this CTA
    if (threadIdx.x == 0) {
      for (int s = 0; s < p.S; ++s) {
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(su32(&full[s])));
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(su32(&empty[s])));
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                          CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                          CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  EncFn enc = (EncFn)fp;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  int* sink;
  CK(cudaMalloc(&sink, 4));
  struct Shape {
    const char* name;
    int N, K;
  } shapes[] = {{"qkv", 4608, 3584}, {"o", 3584, 3584}, {"down", 3584, 18944},
                {"gate_up", 37888, 3584}};
  // (R rows per box, KA boxes per stage, S stages, ks override (0 = fill))
  struct Cfg {
    int R, KA, S, ks;
  } cfgs[] = {{128, 1, 8, 0}, {128, 1, 12, 0}, {128, 2, 6, 0}, {128, 4, 3, 0}, {64, 1, 16, 0},
              {64, 2, 8, 0},  {64, 4, 6, 0},   {256, 1, 6, 0}, {128, 1, 12, 1}, {128, 2, 6, 2}};
  for (auto& sh : shapes) {
    const size_t bytes = (size_t)sh.N * sh.K * 2;
    int copies = (int)(600e6 / bytes) + 2;
    std::vector<void*> ws(copies);
    for (auto& w : ws) {
      CK(cudaMalloc(&w, bytes));
      CK(cudaMemset(w, 1, bytes));
    }
    for (auto& c : cfgs) {
      if (c.R * 128 * c.KA * c.S + 2048 > 227 * 1024) continue;
      P p;
      p.N = sh.N;
      p.K = sh.K;
      p.R = c.R;
      p.KA = c.KA;
      p.S = c.S;
      p.tiles = (sh.N + c.R - 1) / c.R;
      const int nkb = sh.K / (64 * c.KA);
      int ks = c.ks ? c.ks : sms / p.tiles;
      if (ks < 1) ks = 1;
      if (ks > nkb) ks = nkb;
      p.ks = ks;
      const int items = p.tiles * ks;
      const int grid = items < sms ? items : sms;
      std::vector<CUtensorMap> tms(copies);
      for (int i = 0; i < copies; ++i) {
        cuuint64_t dims[2] = {(cuuint64_t)sh.K, (cuuint64_t)sh.N};
        cuuint64_t str[1] = {(cuuint64_t)sh.K * 2};
        cuuint32_t box[2] = {64, (cuuint32_t)(c.R > 256 ? 256 : c.R)};
        cuuint32_t es[2] = {1, 1};
        if (enc(&tms[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ws[i], dims, str, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != 0) {
          fprintf(stderr, "encode failed\n");
          return 1;
        }
      }
      const int smem = c.R * 128 * c.KA * c.S + 2048;
      for (int i = 0; i < copies; ++i)
        stream_kernel<<<grid, 64, smem>>>(tms[i], p, sink);
      CK(cudaDeviceSynchronize());
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      const int reps = 3 * copies;
      cudaEventRecord(e0);
      for (int i = 0; i < reps; ++i) stream_kernel<<<grid, 64, smem>>>(tms[i % copies], p, sink);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double us = ms * 1e3 / reps;
      printf("%-8s N=%6d K=%6d R=%3d KA=%d S=%2d ks=%2d grid=%3d inflight=%3d KB: %7.1f us %6.0f GB/s\n",
             sh.name, sh.N, sh.K, c.R, c.KA, c.S, ks, grid, c.R * 128 * c.KA * (c.S - 1) / 1024, us,
             bytes / us / 1e3);
      fflush(stdout);
    }
    for (auto& w : ws) cudaFree(w);
  }
  return 0;
}
