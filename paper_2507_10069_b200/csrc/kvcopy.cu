// kvcopy.cu — K3 (paged KV gather / scatter) and K6 (KV migration) row copies.
//
// A KV "row" is one token's K (or V) for one layer: kv_heads*head_dim bf16,
// contiguous (1 KiB at Qwen2.5-VL-7B shape, 8 KiB at Llama-7B shape).  The
// pool is [layer][K|V][slot][row], request buffers [layer][K|V][row][row].
// The copy is staged through shared memory with 1-D TMA bulk copies
// (cp.async.bulk global->shared, completion on an mbarrier, then
// shared->global bulk stores): no register traffic, one issuing thread per
// CTA, S stages of up to 16 KiB in flight per CTA.  Either side may be a
// peer GPU's memory (NVLink P2P), which makes the same kernel the
// migration path.
#include <cuda_runtime.h>

#include "../../include/emm.h"
#include "ptx.cuh"
#include "runtime.h"

namespace emm {

constexpr int KVC_STAGES = 6;
constexpr int KVC_STAGE_BYTES = 16384;

struct KvCopyArgs {
  const uint8_t* src;
  int64_t src_stride;
  const int32_t* src_rows;
  uint8_t* dst;
  int64_t dst_stride;
  const int32_t* dst_rows;
  int64_t n_rows;
  int64_t row_bytes;
  int64_t n_items;  // n_layers * 2 * n_rows
  int rows_per_stage;
  int64_t chunks_per_cta;
};

__device__ __forceinline__ void kvc_addr(const KvCopyArgs& a, int64_t item, const uint8_t*& s,
                                         uint8_t*& d) {
  const int64_t lh = item / a.n_rows;
  const int64_t r = item - lh * a.n_rows;
  const int64_t sr = a.src_rows ? (int64_t)a.src_rows[r] : r;
  const int64_t dr = a.dst_rows ? (int64_t)a.dst_rows[r] : r;
  s = a.src + lh * a.src_stride + sr * a.row_bytes;
  d = a.dst + lh * a.dst_stride + dr * a.row_bytes;
}

__global__ void __launch_bounds__(32) kv_copy_rows_kernel(const KvCopyArgs a) {
  extern __shared__ __align__(128) uint8_t kvc_smem[];
  uint8_t(*buf)[KVC_STAGE_BYTES] = reinterpret_cast<uint8_t(*)[KVC_STAGE_BYTES]>(kvc_smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(kvc_smem + KVC_STAGES * KVC_STAGE_BYTES);
  if (threadIdx.x != 0) return;
  const int64_t total_chunks = (a.n_items + a.rows_per_stage - 1) / a.rows_per_stage;
  const int64_t c0 = (int64_t)blockIdx.x * a.chunks_per_cta;
  const int64_t c1 = min(c0 + a.chunks_per_cta, total_chunks);
  if (c0 >= c1) return;
  for (int s = 0; s < KVC_STAGES; ++s) mbar_init(&bar[s], 1);
  fence_mbar_init();
  const uint32_t rb = (uint32_t)a.row_bytes;

  auto issue_load = [&](int64_t c) {
    const int st = (int)((c - c0) % KVC_STAGES);
    const int64_t i0 = c * a.rows_per_stage;
    const int64_t i1 = min(i0 + a.rows_per_stage, a.n_items);
    mbar_arrive_expect_tx(&bar[st], (uint32_t)(i1 - i0) * rb);
    for (int64_t i = i0; i < i1; ++i) {
      const uint8_t* s;
      uint8_t* d;
      kvc_addr(a, i, s, d);
      bulk_load(&buf[st][(i - i0) * rb], s, rb, &bar[st]);
    }
  };
  const int64_t n = c1 - c0;
  for (int64_t c = c0; c < c0 + min(n, (int64_t)KVC_STAGES); ++c) issue_load(c);
  for (int64_t c = c0; c < c1; ++c) {
    const int64_t k = c - c0;
    const int st = (int)(k % KVC_STAGES);
    mbar_wait(&bar[st], (uint32_t)((k / KVC_STAGES) & 1));
    const int64_t i0 = c * a.rows_per_stage;
    const int64_t i1 = min(i0 + a.rows_per_stage, a.n_items);
    for (int64_t i = i0; i < i1; ++i) {
      const uint8_t* s;
      uint8_t* d;
      kvc_addr(a, i, s, d);
      bulk_store(d, &buf[st][(i - i0) * rb], rb);
    }
    bulk_commit();
    if (c + KVC_STAGES < c1) {
      bulk_wait_read<0>();  // stage st drained before it is refilled
      issue_load(c + KVC_STAGES);
    }
  }
  bulk_wait<0>();
}

// Small rows (<= 2 KiB, e.g. 1 KiB per token-layer at the Qwen2.5-VL-7B
// shape): one 16-byte vector per thread, U independent loads in flight before
// the stores, grid (row chunks, layer x K/V) so no per-thread division by the
// row count; row_bytes / 16 is a power of two (a shift).  Single-thread TMA
// bulk issue is too slow for 1 KiB rows (one bulk op per KiB).
constexpr int KVV_THREADS = 256, KVV_U = 4;
__global__ void __launch_bounds__(KVV_THREADS) kv_copy_rows_vec_kernel(const KvCopyArgs a,
                                                                        int upr_shift) {
  const int64_t lh = blockIdx.y;
  const uint8_t* src = a.src + lh * a.src_stride;
  uint8_t* dst = a.dst + lh * a.dst_stride;
  const int64_t units = a.n_rows << upr_shift;
  const int64_t base = (int64_t)blockIdx.x * KVV_U * KVV_THREADS + threadIdx.x;
  const int upr_mask = (1 << upr_shift) - 1;
  uint4 v[KVV_U];
  int64_t doff[KVV_U];
#pragma unroll
  for (int k = 0; k < KVV_U; ++k) {
    const int64_t u = base + (int64_t)k * KVV_THREADS;
    doff[k] = -1;
    if (u < units) {
      const int64_t r = u >> upr_shift;
      const int w = (int)(u & upr_mask);
      const int64_t sr = a.src_rows ? (int64_t)__ldg(a.src_rows + r) : r;
      const int64_t dr = a.dst_rows ? (int64_t)__ldg(a.dst_rows + r) : r;
      v[k] = __ldcs(reinterpret_cast<const uint4*>(src + sr * a.row_bytes) + w);
      doff[k] = dr * a.row_bytes + (int64_t)w * 16;
    }
  }
#pragma unroll
  for (int k = 0; k < KVV_U; ++k)
    if (doff[k] >= 0) __stcs(reinterpret_cast<uint4*>(dst + doff[k]), v[k]);
}

int kv_copy_rows_launch(const void* src, int64_t src_stride, const int32_t* src_rows, void* dst,
                        int64_t dst_stride, const int32_t* dst_rows, int64_t n_rows,
                        int64_t row_bytes, int64_t n_layers, cudaStream_t stream) {
  if (n_rows <= 0 || n_layers <= 0) return EMM_OK;
  if (row_bytes <= 0 || row_bytes % 16 != 0 || row_bytes > KVC_STAGE_BYTES ||
      (reinterpret_cast<uintptr_t>(src) & 15) || (reinterpret_cast<uintptr_t>(dst) & 15) ||
      (src_stride % 16) || (dst_stride % 16)) {
    emm_abi::set_error("emm_kv_copy_rows: rows must be 16-byte multiples <= 16 KiB, aligned");
    return EMM_E_INVALID;
  }
  const int64_t upr = row_bytes / 16;
  const bool small = row_bytes <= 2048 && (upr & (upr - 1)) == 0;
  KvCopyArgs a;
  a.src = reinterpret_cast<const uint8_t*>(src);
  a.src_stride = src_stride;
  a.src_rows = src_rows;
  a.dst = reinterpret_cast<uint8_t*>(dst);
  a.dst_stride = dst_stride;
  a.dst_rows = dst_rows;
  a.n_rows = n_rows;
  a.row_bytes = row_bytes;
  a.n_items = n_layers * 2 * n_rows;
  a.rows_per_stage = (int)(KVC_STAGE_BYTES / row_bytes);
  if (small) {
    int shift = 0;
    while ((1ll << shift) < upr) ++shift;
    const int64_t units = n_rows * upr;
    const int64_t per_cta = (int64_t)KVV_U * KVV_THREADS;
    dim3 grid((unsigned)((units + per_cta - 1) / per_cta), (unsigned)(n_layers * 2));
    kv_copy_rows_vec_kernel<<<grid, KVV_THREADS, 0, stream>>>(a, shift);
    count_launch();
    EMM_CUDA_CHECK_LAUNCH("kv_copy_rows_vec_kernel");
    return EMM_OK;
  }
  const int64_t chunks = (a.n_items + a.rows_per_stage - 1) / a.rows_per_stage;
  const int64_t max_ctas = (int64_t)sm_count() * 2;  // 96 KiB smem per CTA -> 2 CTAs per SM
  int64_t ctas = chunks < max_ctas ? chunks : max_ctas;
  a.chunks_per_cta = (chunks + ctas - 1) / ctas;
  ctas = (chunks + a.chunks_per_cta - 1) / a.chunks_per_cta;
  constexpr int smem = KVC_STAGES * KVC_STAGE_BYTES + KVC_STAGES * 8;
  static bool attr_done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_done[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(kv_copy_rows_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return cuda_status(e, "kv copy smem attribute");
    attr_done[dev & 63] = true;
  }
  kv_copy_rows_kernel<<<(unsigned)ctas, 32, smem, stream>>>(a);
  count_launch();
  EMM_CUDA_CHECK_LAUNCH("kv_copy_rows_kernel");
  return EMM_OK;
}

}  // namespace emm

extern "C" int emm_kv_copy_rows(const void* src, int64_t src_stride, const int32_t* src_rows,
                                void* dst, int64_t dst_stride, const int32_t* dst_rows,
                                int64_t n_rows, int64_t row_bytes, int64_t n_layers,
                                void* stream) {
  return emm::kv_copy_rows_launch(src, src_stride, src_rows, dst, dst_stride, dst_rows, n_rows,
                                  row_bytes, n_layers, (cudaStream_t)stream);
}

extern "C" int emm_kv_copy_planes_ce(const void* src, int64_t src_stride, void* dst,
                                     int64_t dst_stride, int64_t n_rows, int64_t row_bytes,
                                     int64_t n_layers, void* stream) {
  if (n_rows < 0 || row_bytes <= 0 || n_layers <= 0 || (n_rows > 0 && (!src || !dst)) ||
      src_stride < n_rows * row_bytes || dst_stride < n_rows * row_bytes) {
    emm_abi::set_error("emm_kv_copy_planes_ce: bad arguments");
    return EMM_E_INVALID;
  }
  if (n_rows == 0) return EMM_OK;
  cudaError_t e = cudaMemcpy2DAsync(dst, (size_t)dst_stride, src, (size_t)src_stride,
                                    (size_t)(n_rows * row_bytes), (size_t)(2 * n_layers),
                                    cudaMemcpyDefault, (cudaStream_t)stream);
  if (e != cudaSuccess) return emm::cuda_status(e, "cudaMemcpy2DAsync (K6 copy engine)");
  return EMM_OK;
}

// ---------------------------------------------------------------------------
// Migration checksum ("exact copying ... checksums"; SURVEY
// §5 debug mode): XXH64 of every moved row, seeded with its plane (layer * 2
// + K/V) and LOGICAL row index, summed mod 2^64.  The source rows (through
// src_rows) and the destination rows (through dst_rows) give the same sum
// iff every (position, bytes) pair arrived; the sum does not depend on the
// order threads finish.  One thread per (plane, row) runs the XXH64 stripe
// loop over its row with 16-byte loads (the second half of every 32-byte
// sector is an L1 hit): 4.1 TB/s = 0.63 of HBM on 4.6 GB (tools/
// kv_checksum_bench.py), bound by L1 wavefronts of the 32-rows-per-warp
// access (16 useful bytes per sector request); unrolled loads measured equal.
namespace emm {

constexpr uint64_t XXP1 = 0x9E3779B185EBCA87ull, XXP2 = 0xC2B2AE3D27D4EB4Full,
                   XXP3 = 0x165667B19E3779F9ull, XXP4 = 0x85EBCA77C2B2AE63ull,
                   XXP5 = 0x27D4EB2F165667C5ull;

__device__ __forceinline__ uint64_t xx_rotl(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
__device__ __forceinline__ uint64_t xx_round(uint64_t acc, uint64_t in) {
  acc += in * XXP2;
  return xx_rotl(acc, 31) * XXP1;
}
__device__ __forceinline__ uint64_t xx_merge(uint64_t h, uint64_t v) {
  h ^= xx_round(0, v);
  return h * XXP1 + XXP4;
}

// XXH64 of a row of `len` bytes (len % 8 == 0, 16-byte aligned)
__device__ uint64_t xxh64_row(const uint8_t* p, int64_t len, uint64_t seed) {
  const uint4* q = reinterpret_cast<const uint4*>(p);
  uint64_t h;
  int64_t off = 0;
  if (len >= 32) {
    uint64_t v1 = seed + XXP1 + XXP2, v2 = seed + XXP2, v3 = seed, v4 = seed - XXP1;
    for (; off + 32 <= len; off += 32) {
      const uint4 a = __ldg(q + off / 16), b = __ldg(q + off / 16 + 1);
      v1 = xx_round(v1, ((uint64_t)a.y << 32) | a.x);
      v2 = xx_round(v2, ((uint64_t)a.w << 32) | a.z);
      v3 = xx_round(v3, ((uint64_t)b.y << 32) | b.x);
      v4 = xx_round(v4, ((uint64_t)b.w << 32) | b.z);
    }
    h = xx_rotl(v1, 1) + xx_rotl(v2, 7) + xx_rotl(v3, 12) + xx_rotl(v4, 18);
    h = xx_merge(h, v1);
    h = xx_merge(h, v2);
    h = xx_merge(h, v3);
    h = xx_merge(h, v4);
  } else {
    h = seed + XXP5;
  }
  h += (uint64_t)len;
  for (; off + 8 <= len; off += 8) {
    const uint64_t k = *reinterpret_cast<const uint64_t*>(p + off);
    h ^= xx_round(0, k);
    h = xx_rotl(h, 27) * XXP1 + XXP4;
  }
  h ^= h >> 33;
  h *= XXP2;
  h ^= h >> 29;
  h *= XXP3;
  h ^= h >> 32;
  return h;
}

__global__ void kv_checksum_kernel(const uint8_t* __restrict__ base, int64_t plane_stride,
                                   const int32_t* __restrict__ rows, int64_t n_rows,
                                   int64_t row_bytes, int64_t n_items,
                                   unsigned long long* __restrict__ out) {
  uint64_t acc = 0;
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < n_items;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int64_t plane = it / n_rows, i = it - plane * n_rows;
    const int64_t row = rows ? rows[i] : i;
    acc += xxh64_row(base + plane * plane_stride + row * row_bytes, row_bytes,
                     ((uint64_t)plane << 32) + (uint64_t)i);
  }
#pragma unroll
  for (int d = 16; d; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, (unsigned long long)acc);
}

}  // namespace emm

extern "C" int emm_kv_checksum(const void* planes, int64_t plane_stride, const int32_t* rows,
                               int64_t n_rows, int64_t row_bytes, int64_t n_layers,
                               uint64_t* out_device, void* stream) {
  if (n_rows < 0 || row_bytes <= 0 || (row_bytes % 16) || n_layers <= 0 || !out_device ||
      (n_rows > 0 && !planes) || (plane_stride % 16) ||
      (reinterpret_cast<uintptr_t>(planes) % 16)) {
    emm_abi::set_error("emm_kv_checksum: bad arguments (16-byte aligned planes and rows)");
    return EMM_E_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(out_device, 0, sizeof(uint64_t), st);
  if (e != cudaSuccess) return emm::cuda_status(e, "cudaMemsetAsync (kv checksum)");
  const int64_t n_items = n_rows * 2 * n_layers;
  if (n_items == 0) return EMM_OK;
  int64_t blocks = (n_items + 255) / 256;
  const int64_t cap = (int64_t)emm::sm_count() * 8;
  if (blocks > cap) blocks = cap;
  emm::kv_checksum_kernel<<<(unsigned)blocks, 256, 0, st>>>(
      reinterpret_cast<const uint8_t*>(planes), plane_stride, rows, n_rows, row_bytes, n_items,
      reinterpret_cast<unsigned long long*>(out_device));
  emm::count_launch();
  EMM_CUDA_CHECK_LAUNCH("kv_checksum_kernel");
  return EMM_OK;
}
