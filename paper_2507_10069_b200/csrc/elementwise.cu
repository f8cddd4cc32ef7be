// elementwise.cu — the HBM-bound glue of the encoder and prefill paths:
// RMSNorm / LayerNorm, RoPE + Q/K/V split with the KV-cache write, pointer
// row gather (input-embedding assembly from text-embedding rows and image
// slabs), ViT patchify (uint8 pixels -> normalised bf16 patches), ViT token
// assembly (CLS + patches + position embeddings) and row argmax.
// All vectorised 16-byte accesses; one warp (or CTA) per row.
#include <cuda_bf16.h>

#include <cuda_runtime.h>

#include "../../include/emm.h"
#include "runtime.h"

namespace emm {

typedef __nv_bfloat16 bf16;

__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float2 t = __bfloat1622float2(h[j]);
    f[2 * j] = t.x;
    f[2 * j + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 u;
  __nv_bfloat162 t;
  t = __floats2bfloat162_rn(f[0], f[1]);
  u.x = *reinterpret_cast<uint32_t*>(&t);
  t = __floats2bfloat162_rn(f[2], f[3]);
  u.y = *reinterpret_cast<uint32_t*>(&t);
  t = __floats2bfloat162_rn(f[4], f[5]);
  u.z = *reinterpret_cast<uint32_t*>(&t);
  t = __floats2bfloat162_rn(f[6], f[7]);
  u.w = *reinterpret_cast<uint32_t*>(&t);
  return u;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

// --------------------------------------------------------------- norms
// one warp per row; D % 8 == 0 (8 elements per lane per step; per-head norms
// of head_dim 64 / 128 leave lanes idle)
template <bool LAYERNORM>
__global__ void norm_kernel(const bf16* __restrict__ x, int64_t ldx, const int32_t* rows,
                            const bf16* __restrict__ w, const bf16* __restrict__ b,
                            bf16* __restrict__ out, int64_t ldo, int T, int D, float eps) {
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= T) return;
  const int src_row = rows ? rows[row] : row;
  const uint4* xr = reinterpret_cast<const uint4*>(x + (int64_t)src_row * ldx);
  const int nv = D / 8;
  float s = 0.f, ss = 0.f;
  for (int i = lane; i < nv; i += 32) {
    float f[8];
    unpack8(xr[i], f);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      s += f[j];
      ss += f[j] * f[j];
    }
  }
  s = warp_sum(s);
  ss = warp_sum(ss);
  float mean = 0.f, rstd;
  if (LAYERNORM) {
    mean = s / D;
    rstd = rsqrtf(fmaxf(ss / D - mean * mean, 0.f) + eps);
  } else {
    rstd = rsqrtf(ss / D + eps);
  }
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  const uint4* br = reinterpret_cast<const uint4*>(b);
  uint4* orow = reinterpret_cast<uint4*>(out + (int64_t)row * ldo);
  for (int i = lane; i < nv; i += 32) {
    float f[8], g[8], bb[8];
    unpack8(xr[i], f);
    unpack8(wr[i], g);
    if (LAYERNORM) unpack8(br[i], bb);
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = (f[j] - mean) * rstd * g[j] + (LAYERNORM ? bb[j] : 0.f);
    orow[i] = pack8(f);
  }
}

// ------------------------------------------------------- rope + qkv split
// qkv row t: [q heads | k heads | v heads] * hd.  Writes q -> q_out[t],
// k/v -> k_out[kv_row[t]] / v_out[kv_row[t]] (the request KV buffer).
__global__ void rope_split_kernel(const bf16* __restrict__ qkv, int64_t ld_qkv, int T, int hq,
                                  int hkv, int hd, const int32_t* __restrict__ pos, float theta,
                                  int rope, bf16* __restrict__ q_out, int64_t ld_q,
                                  bf16* __restrict__ k_out, bf16* __restrict__ v_out,
                                  const int32_t* __restrict__ kv_row, int64_t ld_kv) {
  extern __shared__ float cs[];  // [hd/2] cos, [hd/2] sin
  const int t = blockIdx.x;
  const int half = hd / 2;
  if (rope) {
    const float p = (float)pos[t];
    for (int i = threadIdx.x; i < half; i += blockDim.x) {
      const float inv = powf(theta, -2.f * (float)i / (float)hd);
      float sn, cn;
      sincosf(p * inv, &sn, &cn);
      cs[i] = cn;
      cs[half + i] = sn;
    }
    __syncthreads();
  }
  const bf16* src = qkv + (int64_t)t * ld_qkv;
  const int64_t kr = kv_row[t];
  // q and k: rotate pairs (i, i + hd/2)
  const int n_rot = (hq + hkv) * half;
  for (int idx = threadIdx.x; idx < n_rot; idx += blockDim.x) {
    const int h = idx / half, i = idx - h * half;
    const float a = __bfloat162float(src[h * hd + i]);
    const float b = __bfloat162float(src[h * hd + i + half]);
    float ra = a, rb = b;
    if (rope) {
      const float c = cs[i], s = cs[half + i];
      ra = a * c - b * s;
      rb = b * c + a * s;
    }
    bf16* dst = h < hq ? q_out + (int64_t)t * ld_q + h * hd
                       : k_out + kr * ld_kv + (h - hq) * hd;
    dst[i] = __float2bfloat16(ra);
    dst[i + half] = __float2bfloat16(rb);
  }
  // v: plain copy, 16-byte vectors
  const uint4* vs = reinterpret_cast<const uint4*>(src + (hq + hkv) * hd);
  uint4* vd = reinterpret_cast<uint4*>(v_out + kr * ld_kv);
  for (int i = threadIdx.x; i < hkv * hd / 8; i += blockDim.x) vd[i] = vs[i];
}

// --------------------------------------------------------- row sum of squares
// one warp per row: out[row] = sum(x[row, :]^2) in fp32 (folded RMSNorm input)
__global__ void row_sumsq_kernel(const bf16* __restrict__ x, int64_t ldx, int T, int D,
                                 float* __restrict__ out) {
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= T) return;
  const uint4* xr = reinterpret_cast<const uint4*>(x + (int64_t)row * ldx);
  float ss = 0.f;
  for (int i = lane; i < D / 8; i += 32) {
    float f[8];
    unpack8(xr[i], f);
#pragma unroll
    for (int j = 0; j < 8; ++j) ss += f[j] * f[j];
  }
  ss = warp_sum(ss);
  if (lane == 0) out[row] = ss;
}

// ------------------------------------------------------------ row gather
// out[i] = *(row_bytes at src_ptr[i]); one warp per row, 16-byte vectors
__global__ void gather_rows_kernel(const int64_t* __restrict__ src_ptr, uint8_t* __restrict__ out,
                                   int64_t ldo_bytes, int T, int row_bytes) {
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= T) return;
  const uint4* s = reinterpret_cast<const uint4*>(src_ptr[row]);
  uint4* d = reinterpret_cast<uint4*>(out + (int64_t)row * ldo_bytes);
  for (int i = lane; i < row_bytes / 16; i += 32) d[i] = s[i];
}

// out[i] = table[ids[i]] (decode: embeddings of the tokens fed back from the
// previous step's argmax, on the device, no host round trip)
__global__ void embed_rows_kernel(const uint8_t* __restrict__ table, int64_t ld_bytes,
                                  const int32_t* __restrict__ ids, uint8_t* __restrict__ out,
                                  int64_t ldo_bytes, int T, int row_bytes) {
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= T) return;
  const uint4* s = reinterpret_cast<const uint4*>(table + (int64_t)ids[row] * ld_bytes);
  uint4* d = reinterpret_cast<uint4*>(out + (int64_t)row * ldo_bytes);
  for (int i = lane; i < row_bytes / 16; i += 32) d[i] = s[i];
}

// ------------------------------------------------------------- patchify
// image i: HWC uint8 at pix + pix_off[i], grid gh x gw patches of P x P;
// patch p (row-major) -> out row patch_off[i] + p, columns (c, ky, kx),
// zero-padded to k_pad.  x = (v/255 - mean[c]) / std[c].
__global__ void patchify_kernel(const uint8_t* __restrict__ pix, const int64_t* __restrict__ pix_off,
                                const int32_t* __restrict__ gh, const int32_t* __restrict__ gw,
                                const int64_t* __restrict__ patch_off, int n_img, int P, int k_pad,
                                float m0, float m1, float m2, float s0, float s1, float s2,
                                bf16* __restrict__ out) {
  const int img = blockIdx.y;
  const int p = blockIdx.x;
  if (img >= n_img || p >= gh[img] * gw[img]) return;
  const int W = gw[img] * P;
  const int py = p / gw[img], px = p - py * gw[img];
  const uint8_t* base = pix + pix_off[img];
  bf16* o = out + (patch_off[img] + p) * (int64_t)k_pad;
  const int K = 3 * P * P;
  for (int k = threadIdx.x; k < k_pad; k += blockDim.x) {
    float v = 0.f;
    if (k < K) {
      const int c = k / (P * P), r = k - c * P * P, ky = r / P, kx = r - ky * P;
      const int y = py * P + ky, x = px * P + kx;
      const float raw = (float)base[((int64_t)y * W + x) * 3 + c] * (1.f / 255.f);
      const float mean = c == 0 ? m0 : (c == 1 ? m1 : m2);
      const float sd = c == 0 ? s0 : (c == 1 ? s1 : s2);
      v = (raw - mean) / sd;
    }
    o[k] = __float2bfloat16(v);
  }
}

// ------------------------------------------- Qwen2.5-VL patchify (window order)
// out row r <- image row_img[r], raster patch row_patch[r]; columns (c, t, ky, kx)
// over `T` identical frames (Conv3d temporal patch of a still image), zero-padded.
__global__ void patchify_rows_kernel(const uint8_t* __restrict__ pix,
                                     const int64_t* __restrict__ pix_off,
                                     const int32_t* __restrict__ gw,
                                     const int32_t* __restrict__ row_img,
                                     const int32_t* __restrict__ row_patch, int P, int T,
                                     int k_pad, float m0, float m1, float m2, float s0, float s1,
                                     float s2, bf16* __restrict__ out) {
  const int64_t r = blockIdx.x;
  const int img = row_img[r], p = row_patch[r];
  const int w = gw[img];
  const int py = p / w, px = p - py * w;
  const int W = w * P;
  const uint8_t* base = pix + pix_off[img];
  bf16* o = out + r * (int64_t)k_pad;
  const int PP = P * P, K = 3 * T * PP;
  for (int k = threadIdx.x; k < k_pad; k += blockDim.x) {
    float v = 0.f;
    if (k < K) {
      const int c = k / (T * PP), rem = k % PP, ky = rem / P, kx = rem - ky * P;
      const int y = py * P + ky, x = px * P + kx;
      const float raw = (float)base[((int64_t)y * W + x) * 3 + c] * (1.f / 255.f);
      const float mean = c == 0 ? m0 : (c == 1 ? m1 : m2);
      const float sd = c == 0 ? s0 : (c == 1 ? s1 : s2);
      v = (raw - mean) / sd;
    }
    o[k] = __float2bfloat16(v);
  }
}

// ------------------------------------------------ 2-D rotary (Qwen2.5-VL ViT)
// in place on the first n_heads heads of row t (q then k of the fused QKV):
// pair (i, i + hd/2), angle = pos_h[t] * inv[i] (i < hd/4) or
// pos_w[t] * inv[i - hd/4], inv[j] = theta^(-2j / (hd/2)).  One warp per row,
// 8 pairs (two 16-byte vectors) per step.
__global__ void rope2d_kernel(bf16* __restrict__ x, int64_t ldx, int T, int n_heads, int hd,
                              const int32_t* __restrict__ pos_h,
                              const int32_t* __restrict__ pos_w, float theta) {
  extern __shared__ float cs2[];  // per warp: [half] cos, [half] sin
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + wib;
  if (row >= T) return;
  const int half = hd >> 1, quarter = hd >> 2;
  float* cs = cs2 + wib * hd;
  const float ph = (float)pos_h[row], pw = (float)pos_w[row];
  for (int i = lane; i < half; i += 32) {
    const int j = i < quarter ? i : i - quarter;
    const float inv = powf(theta, -2.f * (float)j / (float)half);
    float sn, cn;
    sincosf((i < quarter ? ph : pw) * inv, &sn, &cn);
    cs[i] = cn;
    cs[half + i] = sn;
  }
  __syncwarp();
  bf16* xr = x + (int64_t)row * ldx;
  const int per_head = half / 8;
  for (int u = lane; u < n_heads * per_head; u += 32) {
    const int h = u / per_head, c = (u - h * per_head) * 8;
    uint4* pa = reinterpret_cast<uint4*>(xr + h * hd + c);
    uint4* pb = reinterpret_cast<uint4*>(xr + h * hd + half + c);
    float a[8], b[8];
    unpack8(*pa, a);
    unpack8(*pb, b);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float cn = cs[c + e], sn = cs[half + c + e];
      const float xa = a[e], xb = b[e];
      a[e] = xa * cn - xb * sn;
      b[e] = xb * cn + xa * sn;
    }
    *pa = pack8(a);
    *pb = pack8(b);
  }
}

// ---------------------------------------------------- ViT token assembly
// image i owns output rows [tok_off[i], tok_off[i+1]) and patch rows from
// patch_off[i]; row j of image i = (j==0 && cls ? cls_emb : patch[.. + j-cls])
// + pos[j]
__global__ void vit_embed_kernel(const bf16* __restrict__ patch, const bf16* __restrict__ cls,
                                 const bf16* __restrict__ pos, bf16* __restrict__ out,
                                 const int64_t* __restrict__ tok_off,
                                 const int64_t* __restrict__ patch_off, int n_img, int has_cls,
                                 int D) {
  const int64_t row = blockIdx.x;
  int lo = 0, hi = n_img - 1;
  while (lo < hi) {  // image owning this row
    const int mid = (lo + hi + 1) >> 1;
    if (tok_off[mid] <= row)
      lo = mid;
    else
      hi = mid - 1;
  }
  const int img = lo;
  const int64_t j = row - tok_off[img];
  const uint4* src = (has_cls && j == 0)
                         ? reinterpret_cast<const uint4*>(cls)
                         : reinterpret_cast<const uint4*>(patch + (patch_off[img] + j - has_cls) * D);
  const uint4* pr = reinterpret_cast<const uint4*>(pos + j * D);
  uint4* d = reinterpret_cast<uint4*>(out + row * D);
  for (int i = threadIdx.x; i < D / 8; i += blockDim.x) {
    float a[8], b[8];
    unpack8(src[i], a);
    unpack8(pr[i], b);
#pragma unroll
    for (int e = 0; e < 8; ++e) a[e] += b[e];
    d[i] = pack8(a);
  }
}

// --------------------------------------------------------------- argmax
__global__ void argmax_rows_kernel(const bf16* __restrict__ x, int64_t ldx, int V,
                                   int32_t* __restrict__ out) {
  const int row = blockIdx.x;
  const bf16* r = x + (int64_t)row * ldx;
  float best = -INFINITY;
  int bi = 0;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    const float v = __bfloat162float(r[i]);
    if (v > best) {
      best = v;
      bi = i;
    }
  }
  __shared__ float sb[32];
  __shared__ int si[32];
#pragma unroll
  for (int d = 16; d; d >>= 1) {
    const float ob = __shfl_xor_sync(0xffffffffu, best, d);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, d);
    if (ob > best || (ob == best && oi < bi)) {
      best = ob;
      bi = oi;
    }
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sb[w] = best;
    si[w] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q)
      if (sb[q] > best || (sb[q] == best && si[q] < bi)) {
        best = sb[q];
        bi = si[q];
      }
    out[row] = bi;
  }
}


// Chunked row argmax: grid (chunks, rows), 16-byte loads; each CTA writes
// its best (value, first index) as one 64-bit key (order-preserving float
// bits above ~index: larger value, then smaller index wins) to the caller's
// workspace, and argmax_keys_kernel reduces a row's keys to the index.
// Same result as argmax_rows_kernel: the first index of the maximum, NaNs
// ignored, 0 for a row without any value above -inf.
__device__ __forceinline__ unsigned long long argmax_key(float v, int i) {
  // -0.0 and +0.0 compare equal (torch.argmax, argmax_rows_kernel): give them
  // one key so the first index of a zero maximum wins
  const uint32_t u = v == 0.0f ? 0u : __float_as_uint(v);
  const uint32_t k = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((unsigned long long)k << 32) | (0xFFFFFFFFu - (uint32_t)i);
}

__global__ void argmax_chunks_kernel(const bf16* __restrict__ x, int64_t ldx, int V, int chunk,
                                     int n_chunks, int vec, unsigned long long* ws) {
  const int c = blockIdx.x, row = blockIdx.y;
  const bf16* r = x + (int64_t)row * ldx;
  const int i0 = c * chunk, i1 = min(V, i0 + chunk);
  float best = -INFINITY;
  int bi = 0;
  if (vec) {  // row start 16-byte aligned, chunk a multiple of 8
    for (int i = i0 + threadIdx.x * 8; i < i1; i += blockDim.x * 8) {
      if (i + 8 <= i1) {
        const uint4 u = *reinterpret_cast<const uint4*>(r + i);
        const bf16* h = reinterpret_cast<const bf16*>(&u);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float v = __bfloat162float(h[k]);
          if (v > best) {
            best = v;
            bi = i + k;
          }
        }
      } else {
        for (int k = i; k < i1; ++k) {
          const float v = __bfloat162float(r[k]);
          if (v > best) {
            best = v;
            bi = k;
          }
        }
      }
    }
  } else {
    for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
      const float v = __bfloat162float(r[i]);
      if (v > best) {
        best = v;
        bi = i;
      }
    }
  }
  unsigned long long key = argmax_key(best, bi);
#pragma unroll
  for (int d = 16; d; d >>= 1) {
    const unsigned long long o = __shfl_xor_sync(0xffffffffu, key, d);
    key = o > key ? o : key;
  }
  __shared__ unsigned long long sk[32];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) sk[w] = key;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q) key = sk[q] > key ? sk[q] : key;
    ws[(int64_t)row * n_chunks + c] = key;
  }
}

// one warp per row: the max of the row's chunk keys -> its index
__global__ void argmax_keys_kernel(const unsigned long long* __restrict__ ws, int n_chunks,
                                   int T, int32_t* __restrict__ out) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= T) return;
  unsigned long long key = 0;
  for (int c = lane; c < n_chunks; c += 32) {
    const unsigned long long k = ws[(int64_t)row * n_chunks + c];
    key = k > key ? k : key;
  }
#pragma unroll
  for (int d = 16; d; d >>= 1) {
    const unsigned long long o = __shfl_xor_sync(0xffffffffu, key, d);
    key = o > key ? o : key;
  }
  if (lane == 0) out[row] = (int32_t)(0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFull));
}

}  // namespace emm

using emm::bf16;

extern "C" int emm_norm_bf16(const void* x, int64_t ldx, const int32_t* rows, const void* w,
                             const void* b, void* out, int64_t ldo, int64_t T, int64_t D,
                             float eps, int layernorm, void* stream) {
  if (T <= 0) return EMM_OK;
  if (D % 8 != 0 || ldx % 8 || ldo % 8) {
    emm_abi::set_error("emm_norm_bf16: D % 8 == 0 and 16-byte pitches required");
    return EMM_E_INVALID;
  }
  const int wpb = 8;
  dim3 grid((unsigned)((T + wpb - 1) / wpb));
  if (layernorm)
    emm::norm_kernel<true><<<grid, wpb * 32, 0, (cudaStream_t)stream>>>(
        (const bf16*)x, ldx, rows, (const bf16*)w, (const bf16*)b, (bf16*)out, ldo, (int)T,
        (int)D, eps);
  else
    emm::norm_kernel<false><<<grid, wpb * 32, 0, (cudaStream_t)stream>>>(
        (const bf16*)x, ldx, rows, (const bf16*)w, nullptr, (bf16*)out, ldo, (int)T, (int)D, eps);
  emm::count_launch();
  EMM_CUDA_CHECK_LAUNCH("norm_kernel");
  return EMM_OK;
}

extern "C" int emm_rope_split_bf16(const void* qkv, int64_t ld_qkv, int64_t T, int hq, int hkv,
                                   int hd, const int32_t* pos, float theta, int rope,
                                   void* q_out, int64_t ld_q, void* k_out, void* v_out,
                                   const int32_t* kv_row, int64_t ld_kv, void* stream) {
  if (T <= 0) return EMM_OK;
  if (hd % 16 || ld_kv % 8) {
    emm_abi::set_error("emm_rope_split_bf16: head_dim % 16 and 16-byte KV pitch required");
    return EMM_E_INVALID;
  }
  emm::rope_split_kernel<<<(unsigned)T, 256, hd * sizeof(float), (cudaStream_t)stream>>>(
      (const bf16*)qkv, ld_qkv, (int)T, hq, hkv, hd, pos, theta, rope, (bf16*)q_out, ld_q,
      (bf16*)k_out, (bf16*)v_out, kv_row, ld_kv);
  emm::count_launch();
  EMM_CUDA_CHECK_LAUNCH("rope_split_kernel");
  return EMM_OK;
}

extern "C" int emm_row_sumsq_bf16(const void* x, int64_t ldx, int64_t T, int64_t D, float* out,
                                  void* stream) {
  if (T <= 0) return EMM_OK;
  if (D % 8 || ldx % 8) return EMM_E_INVALID;
  const int wpb = 8;
  emm::row_sumsq_kernel<<<(unsigned)((T + wpb - 1) / wpb), wpb * 32, 0, (cudaStream_t)stream>>>(
      (const bf16*)x, ldx, (int)T, (int)D, out);
  emm::count_launch();
  EMM_CUDA_CHECK_LAUNCH("row_sumsq_kernel");
  return EMM_OK;
}

extern "C" int emm_gather_rows(const int64_t* src_ptr, void* out, int64_t ldo_bytes, int64_t T,
                               int64_t row_bytes, void* stream) {
  if (T <= 0) return EMM_OK;
  if (row_bytes % 16 || ldo_bytes % 16) {
    emm_abi::set_error("emm_gather_rows: 16-byte rows required");
    return EMM_E_INVALID;
  }
  const int wpb = 8;
  emm::gather_rows_kernel<<<(unsigned)((T + wpb - 1) / wpb), wpb * 32, 0, (cudaStream_t)stream>>>(
      src_ptr, (uint8_t*)out, ldo_bytes, (int)T, (int)row_bytes);
  emm::count_launch();
  EMM_CUDA_CHECK_LAUNCH("gather_rows_kernel");
  return EMM_OK;
}

extern "C" int emm_embed_rows(const void* table, int64_t ld_bytes, const int32_t* ids,
                              void* out, int64_t ldo_bytes, int64_t T, int64_t row_bytes,
                              void* stream) {
  if (T <= 0) return EMM_OK;
  if (row_bytes % 16 || ldo_bytes % 16 || ld_bytes % 16) {
    emm_abi::set_error("emm_embed_rows: 16-byte rows required");
    return EMM_E_INVALID;
  }
  const int wpb = 8;
  emm::embed_rows_kernel<<<(unsigned)((T + wpb - 1) / wpb), wpb * 32, 0, (cudaStream_t)stream>>>(
      (const uint8_t*)table, ld_bytes, ids, (uint8_t*)out, ldo_bytes, (int)T, (int)row_bytes);
  emm::count_launch();
  EMM_CUDA_CHECK_LAUNCH("embed_rows_kernel");
  return EMM_OK;
}

// decode: advance every request of a batch by one token on the device (so a
// captured decode step replays without host input): the new token's arena
// row is the request's next reserved slot, its RoPE position the next one.
__global__ void decode_advance_kernel(const int32_t* __restrict__ bt,
                                      const int64_t* __restrict__ bt_off,
                                      int32_t* __restrict__ kv_len, int32_t* __restrict__ next_pos,
                                      int32_t* __restrict__ slot, int32_t* __restrict__ pos,
                                      int n) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int len = kv_len[r];
  slot[r] = bt[bt_off[r] + len];
  kv_len[r] = len + 1;
  const int p = next_pos[r];
  pos[r] = p;
  next_pos[r] = p + 1;
}

extern "C" int emm_decode_advance(const int32_t* bt, const int64_t* bt_off, int32_t* kv_len,
                                  int32_t* next_pos, int32_t* slot, int32_t* pos, int64_t n,
                                  void* stream) {
  if (n <= 0) return EMM_OK;
  decode_advance_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      bt, bt_off, kv_len, next_pos, slot, pos, (int)n);
  emm::count_launch();
  EMM_CUDA_CHECK_LAUNCH("decode_advance_kernel");
  return EMM_OK;
}

extern "C" int emm_patchify(const uint8_t* pix, const int64_t* pix_off, const int32_t* gh,
                            const int32_t* gw, const int64_t* patch_off, int n_img,
                            int max_patches, int patch, int k_pad, const float* mean3,
                            const float* std3, void* out, void* stream) {
  if (n_img <= 0) return EMM_OK;
  dim3 grid((unsigned)max_patches, (unsigned)n_img);
  emm::patchify_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      pix, pix_off, gh, gw, patch_off, n_img, patch, k_pad, mean3[0], mean3[1], mean3[2],
      std3[0], std3[1], std3[2], (bf16*)out);
  emm::count_launch();
  EMM_CUDA_CHECK_LAUNCH("patchify_kernel");
  return EMM_OK;
}

extern "C" int emm_vit_embed(const void* patch, const void* cls, const void* pos, void* out,
                             const int64_t* tok_off, const int64_t* patch_off, int n_img,
                             int64_t n_rows, int has_cls, int D, void* stream) {
  if (n_img <= 0 || n_rows <= 0) return EMM_OK;
  if (D % 8) return EMM_E_INVALID;
  emm::vit_embed_kernel<<<(unsigned)n_rows, 128, 0, (cudaStream_t)stream>>>(
      (const bf16*)patch, (const bf16*)cls, (const bf16*)pos, (bf16*)out, tok_off, patch_off,
      n_img, has_cls, D);
  emm::count_launch();
  EMM_CUDA_CHECK_LAUNCH("vit_embed_kernel");
  return EMM_OK;
}

extern "C" int emm_argmax_rows(const void* x, int64_t ldx, int64_t T, int64_t V, int32_t* out,
                               void* stream) {
  if (T <= 0) return EMM_OK;
  emm::argmax_rows_kernel<<<(unsigned)T, 512, 0, (cudaStream_t)stream>>>((const bf16*)x, ldx,
                                                                         (int)V, out);
  emm::count_launch();
  EMM_CUDA_CHECK_LAUNCH("argmax_rows_kernel");
  return EMM_OK;
}

extern "C" int64_t emm_argmax_workspace_keys(int64_t T, int64_t V) {
  return T * ((V + EMM_ARGMAX_CHUNK - 1) / EMM_ARGMAX_CHUNK);
}

extern "C" int emm_argmax_rows_ws(const void* x, int64_t ldx, int64_t T, int64_t V,
                                  int32_t* out, uint64_t* ws, void* stream) {
  if (T <= 0) return EMM_OK;
  if (T > 65535 || !ws) return emm_argmax_rows(x, ldx, T, V, out, stream);
  cudaStream_t st = (cudaStream_t)stream;
  const int n_chunks = (int)((V + EMM_ARGMAX_CHUNK - 1) / EMM_ARGMAX_CHUNK);
  const int vec = ((reinterpret_cast<uintptr_t>(x) & 15) == 0 && (ldx % 8) == 0) ? 1 : 0;
  emm::argmax_chunks_kernel<<<dim3((unsigned)n_chunks, (unsigned)T), 256, 0, st>>>(
      (const bf16*)x, ldx, (int)V, EMM_ARGMAX_CHUNK, n_chunks, vec,
      reinterpret_cast<unsigned long long*>(ws));
  emm::count_launch();
  EMM_CUDA_CHECK_LAUNCH("argmax_chunks_kernel");
  emm::argmax_keys_kernel<<<(unsigned)((T + 7) / 8), 256, 0, st>>>(
      reinterpret_cast<const unsigned long long*>(ws), n_chunks, (int)T, out);
  emm::count_launch();
  EMM_CUDA_CHECK_LAUNCH("argmax_keys_kernel");
  return EMM_OK;
}

extern "C" int emm_patchify_rows(const uint8_t* pix, const int64_t* pix_off, const int32_t* gw,
                                 const int32_t* row_img, const int32_t* row_patch,
                                 int64_t n_rows, int patch, int temporal, int k_pad,
                                 const float* mean3, const float* std3, void* out,
                                 void* stream) {
  if (n_rows <= 0) return EMM_OK;
  if (k_pad < 3 * temporal * patch * patch || temporal < 1) {
    emm_abi::set_error("emm_patchify_rows: k_pad < 3 * temporal * patch^2");
    return EMM_E_INVALID;
  }
  emm::patchify_rows_kernel<<<(unsigned)n_rows, 256, 0, (cudaStream_t)stream>>>(
      pix, pix_off, gw, row_img, row_patch, patch, temporal, k_pad, mean3[0], mean3[1],
      mean3[2], std3[0], std3[1], std3[2], (bf16*)out);
  emm::count_launch();
  EMM_CUDA_CHECK_LAUNCH("patchify_rows_kernel");
  return EMM_OK;
}

extern "C" int emm_rope2d_bf16(void* x, int64_t ldx, int64_t T, int n_heads, int hd,
                               const int32_t* pos_h, const int32_t* pos_w, float theta,
                               void* stream) {
  if (T <= 0) return EMM_OK;
  if (hd % 16 || ldx % 8 || hd > 256) {
    emm_abi::set_error("emm_rope2d_bf16: head_dim % 16 == 0 (<= 256), 16-byte pitch");
    return EMM_E_INVALID;
  }
  const int wpb = 8;
  emm::rope2d_kernel<<<(unsigned)((T + wpb - 1) / wpb), wpb * 32, wpb * hd * sizeof(float),
                       (cudaStream_t)stream>>>((bf16*)x, ldx, (int)T, n_heads, hd, pos_h, pos_w,
                                               theta);
  emm::count_launch();
  EMM_CUDA_CHECK_LAUNCH("rope2d_kernel");
  return EMM_OK;
}
