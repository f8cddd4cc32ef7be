// runtime.h — host-side helpers shared by the launch wrappers: TMA tensor-map
// encoding through the driver entry point (no -lcuda), SM count, the launch
// counter behind emm_launch_count(), and CUDA error mapping.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace emm_abi {
void set_error(const std::string& s);
}

namespace emm {

void count_launch(uint64_t n = 1);
int sm_count();  // of the current device (cached per device)

// 2-D tensor map over a row-major [outer][inner] array with a row pitch in
// bytes; box = [box_outer][box_inner] elements.
bool make_tmap_2d(CUtensorMap* map, const void* ptr, CUtensorMapDataType dtype, int elem_bytes,
                  uint64_t inner, uint64_t outer, uint64_t row_pitch_bytes, uint32_t box_inner,
                  uint32_t box_outer, CUtensorMapSwizzle swizzle);
// 3-D tensor map [d2][d1][d0] with pitches (bytes) for d1 and d2.
bool make_tmap_3d(CUtensorMap* map, const void* ptr, CUtensorMapDataType dtype, int elem_bytes,
                  uint64_t d0, uint64_t d1, uint64_t d2, uint64_t pitch1, uint64_t pitch2,
                  uint32_t b0, uint32_t b1, uint32_t b2, CUtensorMapSwizzle swizzle);

// map the last CUDA error to EMM_E_CUDA with a message
int cuda_status(cudaError_t e, const char* what);

// Programmatic dependent launch (EMM_PDL, default on): kernels launched with
// launch_pdl may start their prologue (barrier init, TMEM alloc, descriptor
// prefetch) while the previous kernel in the stream drains; every such
// kernel executes pdl_wait() before touching global memory and
// pdl_trigger() once all its CTAs are resident.
bool pdl_enabled();

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

}  // namespace emm

#ifdef __CUDACC__
// griddepcontrol: no-ops when the kernel was launched without the attribute
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
#endif

#define EMM_CUDA_CHECK_LAUNCH(what)                                   \
  do {                                                                \
    cudaError_t _e = cudaGetLastError();                              \
    if (_e != cudaSuccess) return emm::cuda_status(_e, what);         \
  } while (0)
