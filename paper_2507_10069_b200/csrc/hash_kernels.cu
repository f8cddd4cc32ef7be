// hash_kernels.cu — K1: block hashes of unified sequences and image-content
// digests (definitions in emm_hash.h; CPU restatement in oracle/hash_oracle.c).
//
// Block hash: one CTA per sequence; the chained polynomial
//   P(i) = P(i-1) * B + x_i  (mod 2^61-1)
// is an affine map h -> h*a + c, so a CTA-wide inclusive scan over
// (a, c) pairs gives every position's prefix hash in O(log n) depth; a
// running carry links successive 256-symbol chunks.  Weights are
// prefix-summed in the same pass (cumw = KV-token end of each symbol).
//
// Pixel digest: one warp per 8 KiB segment, 32 consecutive 8-byte words per
// step (coalesced 256 B warp loads); partial (h, len) per segment, then one
// thread per image folds its segments in order.
#include <cuda_runtime.h>

#include <vector>

#include "../../include/emm.h"
#include "emm_hash.h"
#include "runtime.h"

namespace emm {

struct Aff {  // h -> h*a + c
  uint64_t a, c;
};

__device__ __forceinline__ Aff aff_then(Aff f, Aff g) {  // apply f then g
  return Aff{emm_mulmod61(f.a, g.a), emm_addmod61(emm_mulmod61(f.c, g.a), g.c)};
}

__device__ __forceinline__ Aff shfl_up_aff(Aff v, int d) {
  Aff r;
  r.a = __shfl_up_sync(0xffffffffu, v.a, d);
  r.c = __shfl_up_sync(0xffffffffu, v.c, d);
  return r;
}

constexpr int HASH_THREADS = 256;

__global__ void __launch_bounds__(HASH_THREADS) block_hash_kernel(
    const uint64_t* __restrict__ keys, const int64_t* __restrict__ weights,
    const int64_t* __restrict__ seq_off, uint64_t* __restrict__ h0, uint64_t* __restrict__ h1,
    int64_t* __restrict__ cumw) {
  __shared__ Aff warp_tot[2][HASH_THREADS / 32];
  __shared__ int64_t warp_w[HASH_THREADS / 32];
  __shared__ Aff carry_s[2];
  __shared__ int64_t carry_w;
  const int s = blockIdx.x;
  const int64_t beg = seq_off[s], end = seq_off[s + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    carry_s[0] = Aff{1, EMM_H0};  // h starts at the seed: represent as constant map
    carry_s[1] = Aff{1, EMM_H1};
    carry_w = 0;
  }
  __syncthreads();
  for (int64_t base = beg; base < end; base += HASH_THREADS) {
    const int64_t j = base + tid;
    const bool ok = j < end;
    const uint64_t k = ok ? keys[j] : 0;
    const int64_t w = ok ? weights[j] : 0;
    Aff f[2];
    f[0] = ok ? Aff{EMM_B0, emm_sym_term(k, (uint64_t)w, 0)} : Aff{1, 0};
    f[1] = ok ? Aff{EMM_B1, emm_sym_term(k, (uint64_t)w, 1)} : Aff{1, 0};
    int64_t ws = w;
    // warp inclusive scan
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
      for (int l = 0; l < 2; ++l) {
        Aff o = shfl_up_aff(f[l], d);
        if (lane >= d) f[l] = aff_then(o, f[l]);
      }
      int64_t ow = __shfl_up_sync(0xffffffffu, ws, d);
      if (lane >= d) ws += ow;
    }
    if (lane == 31) {
      warp_tot[0][warp] = f[0];
      warp_tot[1][warp] = f[1];
      warp_w[warp] = ws;
    }
    __syncthreads();
    // prefix over earlier warps + chunk carry
    Aff pre[2] = {carry_s[0], carry_s[1]};
    int64_t pw = carry_w;
    for (int q = 0; q < warp; ++q) {
      pre[0] = aff_then(pre[0], warp_tot[0][q]);
      pre[1] = aff_then(pre[1], warp_tot[1][q]);
      pw += warp_w[q];
    }
    const Aff tot0 = aff_then(pre[0], f[0]);
    const Aff tot1 = aff_then(pre[1], f[1]);
    if (ok) {
      // carry maps are constant maps (a applied to h=... folded into c)
      h0[j] = tot0.c;
      h1[j] = tot1.c;
      cumw[j] = pw + ws;
    }
    __syncthreads();
    // invalid lanes carry identity maps, so the last thread holds the chunk total
    if (tid == HASH_THREADS - 1) {
      carry_s[0] = Aff{1, tot0.c};
      carry_s[1] = Aff{1, tot1.c};
      carry_w = pw + ws;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- pixels
constexpr int SEG_WORDS = 1024;  // 8 KiB per warp segment

__device__ __forceinline__ uint64_t powmod61(uint64_t b, uint64_t e) {
  uint64_t r = 1;
  while (e) {
    if (e & 1) r = emm_mulmod61(r, b);
    b = emm_mulmod61(b, b);
    e >>= 1;
  }
  return r;
}

__device__ __forceinline__ uint64_t load_word(const uint8_t* p, int64_t nbytes, int64_t w) {
  const int64_t off = w * 8;
  if (off + 8 <= nbytes) {
    uint64_t v;
    memcpy(&v, p + off, 8);  // 8-byte aligned when the image start is
    return v;
  }
  uint64_t v = 0;
  for (int b = 0; b < 8 && off + b < nbytes; ++b) v |= (uint64_t)p[off + b] << (8 * b);
  return v;
}

// grid: one warp per (image, segment); seg_base[i] = first global segment of image i
__global__ void pixel_segments_kernel(const uint8_t* __restrict__ bytes,
                                      const int64_t* __restrict__ img_start,
                                      const int64_t* __restrict__ img_len,
                                      const int64_t* __restrict__ seg_base, int n_imgs,
                                      int64_t n_segs, uint64_t* __restrict__ part) {
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x / 32);
  const int lane = threadIdx.x & 31;
  if (gw >= n_segs) return;
  // find the image owning this segment (few images: linear search)
  int img = 0;
  while (img + 1 < n_imgs && seg_base[img + 1] <= gw) ++img;
  const int64_t seg = gw - seg_base[img];
  const uint8_t* p = bytes + img_start[img];
  const int64_t nbytes = img_len[img];
  const int64_t nwords = (nbytes + 7) / 8;
  const int64_t w0 = seg * SEG_WORDS;
  const int64_t w1 = min(w0 + (int64_t)SEG_WORDS, nwords);
  // lane power B^(31-lane) for a full 32-word step
  const uint64_t pl0 = powmod61(EMM_C0, 31 - lane), pl1 = powmod61(EMM_C1, 31 - lane);
  const uint64_t p32_0 = powmod61(EMM_C0, 32), p32_1 = powmod61(EMM_C1, 32);
  uint64_t acc0 = 0, acc1 = 0;
  int64_t w = w0;
  for (; w + 32 <= w1; w += 32) {
    const uint64_t x = load_word(p, nbytes, w + lane);
    uint64_t t0 = emm_mulmod61(emm_pix_term(x, 0), pl0);
    uint64_t t1 = emm_mulmod61(emm_pix_term(x, 1), pl1);
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
      t0 = emm_addmod61(t0, __shfl_xor_sync(0xffffffffu, t0, d));
      t1 = emm_addmod61(t1, __shfl_xor_sync(0xffffffffu, t1, d));
    }
    acc0 = emm_addmod61(emm_mulmod61(acc0, p32_0), t0);
    acc1 = emm_addmod61(emm_mulmod61(acc1, p32_1), t1);
  }
  // tail (< 32 words): lane 0 folds sequentially
  if (lane == 0) {
    for (; w < w1; ++w) {
      const uint64_t x = load_word(p, nbytes, w);
      acc0 = emm_addmod61(emm_mulmod61(acc0, EMM_C0), emm_pix_term(x, 0));
      acc1 = emm_addmod61(emm_mulmod61(acc1, EMM_C1), emm_pix_term(x, 1));
    }
    part[2 * gw] = acc0;
    part[2 * gw + 1] = acc1;
  }
}

__global__ void pixel_fold_kernel(const int64_t* __restrict__ img_len,
                                  const int64_t* __restrict__ seg_base, int n_imgs,
                                  const uint64_t* __restrict__ part, uint64_t* __restrict__ out) {
  const int img = blockIdx.x * blockDim.x + threadIdx.x;
  if (img >= n_imgs) return;
  const int64_t nbytes = img_len[img];
  const int64_t nwords = (nbytes + 7) / 8;
  const int64_t nseg = seg_base[img + 1] - seg_base[img];
  const uint64_t full0 = powmod61(EMM_C0, SEG_WORDS), full1 = powmod61(EMM_C1, SEG_WORDS);
  uint64_t d0 = EMM_G0, d1 = EMM_G1;
  for (int64_t s = 0; s < nseg; ++s) {
    const int64_t len = min((int64_t)SEG_WORDS, nwords - s * SEG_WORDS);
    const uint64_t m0 = len == SEG_WORDS ? full0 : powmod61(EMM_C0, len);
    const uint64_t m1 = len == SEG_WORDS ? full1 : powmod61(EMM_C1, len);
    d0 = emm_addmod61(emm_mulmod61(d0, m0), part[2 * (seg_base[img] + s)]);
    d1 = emm_addmod61(emm_mulmod61(d1, m1), part[2 * (seg_base[img] + s) + 1]);
  }
  d0 = emm_addmod61(emm_mulmod61(d0, EMM_C0), emm_red61(emm_mix64((uint64_t)nbytes ^ EMM_Q0)));
  d1 = emm_addmod61(emm_mulmod61(d1, EMM_C1), emm_red61(emm_mix64((uint64_t)nbytes ^ EMM_Q1)));
  out[2 * img] = d0;
  out[2 * img + 1] = d1;
}

}  // namespace emm

extern "C" int emm_block_hash(const uint64_t* keys, const int64_t* weights,
                              const int64_t* seq_off, int64_t n_seqs, uint64_t* h0, uint64_t* h1,
                              int64_t* cumw, void* stream) {
  if (n_seqs <= 0) return EMM_OK;
  if (!keys || !weights || !seq_off || !h0 || !h1 || !cumw) {
    emm_abi::set_error("emm_block_hash: null pointer");
    return EMM_E_INVALID;
  }
  emm::block_hash_kernel<<<(unsigned)n_seqs, emm::HASH_THREADS, 0, (cudaStream_t)stream>>>(
      keys, weights, seq_off, h0, h1, cumw);
  emm::count_launch();
  EMM_CUDA_CHECK_LAUNCH("block_hash_kernel");
  return EMM_OK;
}

static int64_t pixel_total_segments(const int64_t* img_len_host, int64_t n_imgs,
                                    std::vector<int64_t>* base) {
  int64_t total = 0;
  for (int64_t i = 0; i < n_imgs; ++i) {
    if (base) base->push_back(total);
    const int64_t nwords = (img_len_host[i] + 7) / 8;
    total += (nwords + emm::SEG_WORDS - 1) / emm::SEG_WORDS;
  }
  if (base) base->push_back(total);
  return total;
}

extern "C" int64_t emm_pixel_digest_scratch_bytes(const int64_t* img_len_host, int64_t n_imgs) {
  const int64_t segs = pixel_total_segments(img_len_host, n_imgs, nullptr);
  return (n_imgs + 1) * 8 + segs * 16 + 16;
}

extern "C" int emm_pixel_digest(const uint8_t* bytes, const int64_t* img_start_dev,
                                const int64_t* img_len_dev, const int64_t* img_start_host,
                                const int64_t* img_len_host, int64_t n_imgs, void* scratch_dev,
                                uint64_t* out, void* stream) {
  if (n_imgs <= 0) return EMM_OK;
  for (int64_t i = 0; i < n_imgs; ++i) {
    if (img_start_host[i] % 8 != 0 || img_len_host[i] < 0) {
      emm_abi::set_error("emm_pixel_digest: image starts must be 8-byte aligned");
      return EMM_E_INVALID;
    }
  }
  std::vector<int64_t> base;
  const int64_t total = pixel_total_segments(img_len_host, n_imgs, &base);
  int64_t* seg_base_dev = reinterpret_cast<int64_t*>(scratch_dev);
  uint64_t* part_dev = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(seg_base_dev + n_imgs + 1) + 15) & ~(uintptr_t)15);
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(seg_base_dev, base.data(), (n_imgs + 1) * 8,
                                  cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return emm::cuda_status(e, "pixel digest segment upload");
  if (total > 0) {
    const int warps = 8;
    const unsigned grid = (unsigned)((total + warps - 1) / warps);
    emm::pixel_segments_kernel<<<grid, warps * 32, 0, st>>>(
        bytes, img_start_dev, img_len_dev, seg_base_dev, (int)n_imgs, total, part_dev);
    emm::count_launch();
    EMM_CUDA_CHECK_LAUNCH("pixel_segments_kernel");
  }
  emm::pixel_fold_kernel<<<(unsigned)((n_imgs + 127) / 128), 128, 0, st>>>(
      img_len_dev, seg_base_dev, (int)n_imgs, part_dev, out);
  emm::count_launch();
  EMM_CUDA_CHECK_LAUNCH("pixel_fold_kernel");
  return EMM_OK;
}
