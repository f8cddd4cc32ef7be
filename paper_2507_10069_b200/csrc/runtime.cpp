// runtime.cpp — see runtime.h
#include "runtime.h"

#include <stdlib.h>

#include <atomic>
#include <mutex>
#include <string>

#include "../../include/emm.h"

namespace emm {

static std::atomic<uint64_t> g_launches{0};
void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

bool make_tmap_2d(CUtensorMap* map, const void* ptr, CUtensorMapDataType dtype, int elem_bytes,
                  uint64_t inner, uint64_t outer, uint64_t row_pitch_bytes, uint32_t box_inner,
                  uint32_t box_outer, CUtensorMapSwizzle swizzle) {
  (void)elem_bytes;
  EncodeTiledFn fn = encode_fn();
  if (!fn) {
    emm_abi::set_error("cuTensorMapEncodeTiled unavailable");
    return false;
  }
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_pitch_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, dtype, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    emm_abi::set_error("cuTensorMapEncodeTiled(2d) failed: " + std::to_string((int)r) +
                       " inner=" + std::to_string(inner) + " outer=" + std::to_string(outer) +
                       " pitch=" + std::to_string(row_pitch_bytes));
    return false;
  }
  return true;
}

bool make_tmap_3d(CUtensorMap* map, const void* ptr, CUtensorMapDataType dtype, int elem_bytes,
                  uint64_t d0, uint64_t d1, uint64_t d2, uint64_t pitch1, uint64_t pitch2,
                  uint32_t b0, uint32_t b1, uint32_t b2, CUtensorMapSwizzle swizzle) {
  (void)elem_bytes;
  EncodeTiledFn fn = encode_fn();
  if (!fn) {
    emm_abi::set_error("cuTensorMapEncodeTiled unavailable");
    return false;
  }
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {pitch1, pitch2};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, dtype, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    emm_abi::set_error("cuTensorMapEncodeTiled(3d) failed: " + std::to_string((int)r));
    return false;
  }
  return true;
}

int cuda_status(cudaError_t e, const char* what) {
  emm_abi::set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return EMM_E_CUDA;
}

bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EMM_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

}  // namespace emm

extern "C" uint64_t emm_launch_count(void) { return emm::g_launches.load(); }

extern "C" int emm_device_sm_count(int device, int* sms) {
  int n = 0;
  cudaError_t e = cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) return emm::cuda_status(e, "cudaDeviceGetAttribute");
  *sms = n;
  return EMM_OK;
}

// Enable device `dev` to address `peer`'s memory (K6 over NVLink P2P).
extern "C" int emm_enable_peer_access(int dev, int peer) {
  int can = 0;
  cudaError_t e = cudaDeviceCanAccessPeer(&can, dev, peer);
  if (e != cudaSuccess) return emm::cuda_status(e, "cudaDeviceCanAccessPeer");
  if (!can) {
    emm_abi::set_error("peer access not supported between these devices");
    return EMM_E_INVALID;
  }
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(dev);
  e = cudaDeviceEnablePeerAccess(peer, 0);
  cudaSetDevice(prev);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return EMM_OK;
  }
  if (e != cudaSuccess) return emm::cuda_status(e, "cudaDeviceEnablePeerAccess");
  return EMM_OK;
}
