// hash_kernels.cu — K1: block hashes of unified sequences and image-content
// digests (definitions in emm_hash.h; CPU restatement in oracle/hash_oracle.c).
//
// Block hash: one CTA per sequence; the chained polynomial
//   P(i) = P(i-1) * B + x_i  (mod 2^61-1)
// is an affine map h -> h*a + c.  Each thread folds a run of 8 consecutive
// symbols with plain Horner steps, the CTA scans the per-run maps, and every
// thread fixes its 8 local values up with the hash entering its run; a
// running carry links successive 2048-symbol chunks.  Weights are
// prefix-summed in the same pass (cumw = KV-token end of each symbol).
//
// Pixel digest: one warp per 8 KiB segment, coalesced 256 B warp loads; each
// lane runs its own Horner chain (base C^32) over every 32nd word and the
// lanes combine once per segment; then one thread per image folds its
// segments in order.
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

__device__ __forceinline__ Aff shfl_aff(Aff v, int src) {
  return Aff{__shfl_sync(0xffffffffu, v.a, src), __shfl_sync(0xffffffffu, v.c, src)};
}

// One CTA per sequence, HB_CHUNK symbols per pass.  Thread t owns the run
// [t*R, t*R + R): it folds its symbols with plain Horner steps (local prefix
// values starting from 0, i.e. the affine map h -> h*B^m + c of the run),
// the CTA scans the per-thread maps (warp shuffle scan, then warp 0 scans
// the 8 warp totals, prefixed by the carry of the previous pass), and each
// thread fixes its local values up with the incoming hash:
//   P(i) = P_in * B^(j+1) + local_j.
// Per symbol that is two Horner steps instead of a log-depth affine scan.
struct HashSmem {
  Aff warp_tot[2][HASH_THREADS / 32];
  int64_t warp_w[HASH_THREADS / 32];
  Aff warp_pre[2][HASH_THREADS / 32];
  int64_t warp_pw[HASH_THREADS / 32];
  uint64_t carry_h[2];
  int64_t carry_w;
};

template <int HB_R>
__device__ __forceinline__ void block_hash_seq(const uint64_t* __restrict__ keys,
                                               const int64_t* __restrict__ weights, int64_t beg,
                                               int64_t end, uint64_t* __restrict__ h0,
                                               uint64_t* __restrict__ h1,
                                               int64_t* __restrict__ cumw, HashSmem& sm) {
  constexpr int HB_CHUNK = HASH_THREADS * HB_R;  // symbols per CTA pass
  auto& warp_tot = sm.warp_tot;
  auto& warp_w = sm.warp_w;
  auto& warp_pre = sm.warp_pre;
  auto& warp_pw = sm.warp_pw;
  auto& carry_h = sm.carry_h;
  auto& carry_w = sm.carry_w;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    carry_h[0] = EMM_H0;
    carry_h[1] = EMM_H1;
    carry_w = 0;
  }
  uint64_t bp0[HB_R], bp1[HB_R];  // B^1 .. B^R
  bp0[0] = EMM_B0;
  bp1[0] = EMM_B1;
#pragma unroll
  for (int j = 1; j < HB_R; ++j) {
    bp0[j] = emm_mulmod61(bp0[j - 1], EMM_B0);
    bp1[j] = emm_mulmod61(bp1[j - 1], EMM_B1);
  }
  __syncthreads();
  for (int64_t base = beg; base < end; base += HB_CHUNK) {
    const int64_t j0 = base + (int64_t)tid * HB_R;
    const int m = (int)max((int64_t)0, min((int64_t)HB_R, end - j0));  // valid symbols
    uint64_t l0[HB_R], l1[HB_R];
    int64_t lw[HB_R];
    uint64_t c0 = 0, c1 = 0;
    int64_t ws = 0;
#pragma unroll
    for (int j = 0; j < HB_R; ++j) {
      if (j < m) {
        const uint64_t k = keys[j0 + j];
        const int64_t w = weights[j0 + j];
        c0 = emm_addmod61(emm_mulmod61(c0, EMM_B0), emm_sym_term(k, (uint64_t)w, 0));
        c1 = emm_addmod61(emm_mulmod61(c1, EMM_B1), emm_sym_term(k, (uint64_t)w, 1));
        ws += w;
      }
      l0[j] = c0;
      l1[j] = c1;
      lw[j] = ws;
    }
    // this run's map h -> h*B^m + c (identity when m == 0); B^m picked by an
    // unrolled select so bp0 / bp1 stay in registers
    uint64_t bm0 = 1, bm1 = 1;
#pragma unroll
    for (int j = 0; j < HB_R; ++j)
      if (j < m) {
        bm0 = bp0[j];
        bm1 = bp1[j];
      }
    Aff f[2] = {Aff{bm0, c0}, Aff{bm1, c1}};
    int64_t fw = ws;
    // inclusive warp scan of the run maps
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
      for (int l = 0; l < 2; ++l) {
        Aff o = shfl_up_aff(f[l], d);
        if (lane >= d) f[l] = aff_then(o, f[l]);
      }
      const int64_t ow = __shfl_up_sync(0xffffffffu, fw, d);
      if (lane >= d) fw += ow;
    }
    if (lane == 31) {
      warp_tot[0][warp] = f[0];
      warp_tot[1][warp] = f[1];
      warp_w[warp] = fw;
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the warp totals, after the carry
      constexpr int NW = HASH_THREADS / 32;
      Aff t[2] = {Aff{1, 0}, Aff{1, 0}};
      int64_t tw = 0;
      if (lane < NW) {
        t[0] = warp_tot[0][lane];
        t[1] = warp_tot[1][lane];
        tw = warp_w[lane];
      }
#pragma unroll
      for (int d = 1; d < NW; d <<= 1) {
#pragma unroll
        for (int l = 0; l < 2; ++l) {
          Aff o = shfl_up_aff(t[l], d);
          if (lane >= d) t[l] = aff_then(o, t[l]);
        }
        const int64_t ow = __shfl_up_sync(0xffffffffu, tw, d);
        if (lane >= d) tw += ow;
      }
      // exclusive = inclusive of lane - 1; prefix with the constant carry map
      Aff e0 = shfl_up_aff(t[0], 1), e1 = shfl_up_aff(t[1], 1);
      int64_t ew = __shfl_up_sync(0xffffffffu, tw, 1);
      if (lane == 0) {
        e0 = Aff{1, 0};
        e1 = Aff{1, 0};
        ew = 0;
      }
      if (lane < NW) {
        warp_pre[0][lane] = aff_then(Aff{1, carry_h[0]}, e0);
        warp_pre[1][lane] = aff_then(Aff{1, carry_h[1]}, e1);
        warp_pw[lane] = carry_w + ew;
      }
    }
    __syncthreads();
    // hash entering this run = warp prefix, then the lanes before it
    Aff x0 = shfl_up_aff(f[0], 1), x1 = shfl_up_aff(f[1], 1);
    int64_t xw = __shfl_up_sync(0xffffffffu, fw, 1);
    if (lane == 0) {
      x0 = Aff{1, 0};
      x1 = Aff{1, 0};
      xw = 0;
    }
    const uint64_t in0 = aff_then(warp_pre[0][warp], x0).c;  // constant maps: value in .c
    const uint64_t in1 = aff_then(warp_pre[1][warp], x1).c;
    const int64_t inw = warp_pw[warp] + xw;
#pragma unroll
    for (int j = 0; j < HB_R; ++j) {
      if (j < m) {
        h0[j0 + j] = emm_addmod61(emm_mulmod61(in0, bp0[j]), l0[j]);
        h1[j0 + j] = emm_addmod61(emm_mulmod61(in1, bp1[j]), l1[j]);
        cumw[j0 + j] = inw + lw[j];
      }
    }
    __syncthreads();
    // the chunk's last run (the last thread: identity maps after the end)
    if (tid == HASH_THREADS - 1) {
      carry_h[0] = aff_then(Aff{1, in0}, Aff{bm0, c0}).c;
      carry_h[1] = aff_then(Aff{1, in1}, Aff{bm1, c1}).c;
      carry_w = inw + ws;
    }
    __syncthreads();
  }
}

// One CTA per sequence; the run length per thread follows the sequence
// length (short sequences keep every thread busy, long ones amortise the
// scan over 8 symbols per thread).
__global__ void __launch_bounds__(HASH_THREADS) block_hash_kernel(
    const uint64_t* __restrict__ keys, const int64_t* __restrict__ weights,
    const int64_t* __restrict__ seq_off, uint64_t* __restrict__ h0, uint64_t* __restrict__ h1,
    int64_t* __restrict__ cumw) {
  __shared__ HashSmem sm;
  const int64_t beg = seq_off[blockIdx.x], end = seq_off[blockIdx.x + 1];
  const int64_t len = end - beg;
  if (len >= 4 * HASH_THREADS)
    block_hash_seq<8>(keys, weights, beg, end, h0, h1, cumw, sm);
  else if (len >= 2 * HASH_THREADS)
    block_hash_seq<4>(keys, weights, beg, end, h0, h1, cumw, sm);
  else if (len > HASH_THREADS)
    block_hash_seq<2>(keys, weights, beg, end, h0, h1, cumw, sm);
  else
    block_hash_seq<1>(keys, weights, beg, end, h0, h1, cumw, sm);
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
  // Lane l runs its own Horner chain over words w0 + 32k + l with base C^32
  // (no cross-lane traffic per step); the segment polynomial is then
  //   sum_l acc_l * C^(31-l)   (one warp reduction per segment)
  // — the same value as folding the words one by one.
  const uint64_t p32_0 = powmod61(EMM_C0, 32), p32_1 = powmod61(EMM_C1, 32);
  uint64_t acc0 = 0, acc1 = 0;
  int64_t w = w0;
  const int64_t n_full = (w1 - w0) / 32;
  const uint64_t* p64 = reinterpret_cast<const uint64_t*>(p);
  if ((w0 + n_full * 32) * 8 <= nbytes) {  // every word of the full steps is in bounds
    // four interleaved chains per hash lane (steps k = 4q + u, base C^128)
    // so the dependent mulmods of one chain overlap the other three's
    const uint64_t p128_0 = powmod61(EMM_C0, 128), p128_1 = powmod61(EMM_C1, 128);
    uint64_t a0[4] = {0, 0, 0, 0}, a1[4] = {0, 0, 0, 0};
    const int64_t n4 = n_full / 4;
    for (int64_t q = 0; q < n4; ++q) {
      uint64_t x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = __ldg(p64 + w + 32 * (4 * q + u) + lane);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a0[u] = emm_addmod61(emm_mulmod61(a0[u], p128_0), emm_pix_term(x[u], 0));
        a1[u] = emm_addmod61(emm_mulmod61(a1[u], p128_1), emm_pix_term(x[u], 1));
      }
    }
    // sum_u a_u * C^(32 (3 - u)): the lane's chain over k = 0 .. 4 n4 - 1
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      acc0 = emm_addmod61(emm_mulmod61(acc0, p32_0), a0[u]);
      acc1 = emm_addmod61(emm_mulmod61(acc1, p32_1), a1[u]);
    }
    for (int64_t k = 4 * n4; k < n_full; ++k) {
      const uint64_t x = __ldg(p64 + w + 32 * k + lane);
      acc0 = emm_addmod61(emm_mulmod61(acc0, p32_0), emm_pix_term(x, 0));
      acc1 = emm_addmod61(emm_mulmod61(acc1, p32_1), emm_pix_term(x, 1));
    }
  } else {
    for (int64_t k = 0; k < n_full; ++k) {
      const uint64_t x = load_word(p, nbytes, w + 32 * k + lane);
      acc0 = emm_addmod61(emm_mulmod61(acc0, p32_0), emm_pix_term(x, 0));
      acc1 = emm_addmod61(emm_mulmod61(acc1, p32_1), emm_pix_term(x, 1));
    }
  }
  w += n_full * 32;
  if (n_full) {
    acc0 = emm_mulmod61(acc0, powmod61(EMM_C0, 31 - lane));
    acc1 = emm_mulmod61(acc1, powmod61(EMM_C1, 31 - lane));
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
      acc0 = emm_addmod61(acc0, __shfl_xor_sync(0xffffffffu, acc0, d));
      acc1 = emm_addmod61(acc1, __shfl_xor_sync(0xffffffffu, acc1, d));
    }
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
