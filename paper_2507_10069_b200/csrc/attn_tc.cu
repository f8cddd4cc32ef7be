// attn_tc.cu — prefill / encoder attention on tcgen05 for sm_100a (K4 / K5).
//
// Varlen flash attention over a batch of sequences: the uncached suffix's
// queries attend over [cached prefix KV | suffix KV] (causal, queries aligned
// to the end of the KV sequence), or bidirectionally inside an image / window
// (ViT).  GQA by head grouping.  This is the compute the reference models as
// prefill_time / encode_time (pkg/src/mmsim/costmodel.py:102-119).
//
// One CTA per (sequence, q-head, 128-query tile):
//   warp 0      TMA: Q tile once, K/V 128-row blocks into a 2-stage ring
//   warp 1      MMA: S_j = Q K_j^T   (M=128, N=128, K=HD)  into TMEM S[j%2]
//                    O  += P_j V_j   (M=128, N=HD,  K=128) into TMEM O
//               S is double buffered so S_{j+1} overlaps softmax of block j.
//   warps 4..7  softmax, one thread per query row: two passes over S_j in
//               TMEM (row max, then exp2 / row sum / bf16 P into swizzled
//               smem), exact O rescale in TMEM (tcgen05.ld/st) when the row
//               max moves, final 1/l normalisation and store.
// TMEM: S0 [0,128) S1 [128,256) O [256, 256+HD).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../../include/emm.h"
#include "ptx.cuh"
#include "runtime.h"

namespace emm {

constexpr int ATT_THREADS = 256;
constexpr int ATT_BM = 128;  // query rows per tile
constexpr int ATT_BN = 128;  // kv rows per block

struct AttnArgs {
  const int32_t* tiles;  // [n_tiles][3] = seq, q head, q tile
  const int32_t* q_start;
  const int32_t* q_len;
  const int32_t* kv_start;
  const int32_t* kv_len;
  __nv_bfloat16* out;
  int64_t out_tok_stride;  // elements
  int n_q_heads, group;    // group = n_q_heads / n_kv_heads
  float scale_log2;        // softmax scale * log2(e)
  int causal;
};

template <int HD>
struct AttnCfg {
  static constexpr int CH = HD / 64;                 // 64-element swizzle atoms per row
  static constexpr int TILE_BYTES = 128 * HD * 2;    // one 128-row bf16 tile
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = TILE_BYTES;           // 2 stages
  static constexpr int V_OFF = K_OFF + 2 * TILE_BYTES;
  static constexpr int P_OFF = V_OFF + 2 * TILE_BYTES;
  static constexpr int P_BYTES = 128 * 128 * 2;
  static constexpr int BAR_OFF = P_OFF + P_BYTES;
  static constexpr int N_BARS = 1 + 2 + 2 + 2 + 2 + 2 + 1 + 1;
  static constexpr int SMEM = BAR_OFF + N_BARS * 8 + 16 + 1024;
};

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ int attn_nblk(const AttnArgs& a, int seq, int qt) {
  const int ql = a.q_len[seq], kl = a.kv_len[seq];
  if (!a.causal) return (kl + ATT_BN - 1) / ATT_BN;
  const int last_q = min(ql, (qt + 1) * ATT_BM) - 1;  // last query row of the tile
  const int last_pos = kl - ql + last_q;              // its absolute KV position
  return last_pos / ATT_BN + 1;
}

template <int HD>
__global__ void __launch_bounds__(ATT_THREADS, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmQ,
                       const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV, const AttnArgs a) {
  using Cfg = AttnCfg<HD>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::BAR_OFF);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* v_full = bars + 3;
  uint64_t* kv_empty = bars + 5;
  uint64_t* s_full = bars + 7;
  uint64_t* s_free = bars + 9;
  uint64_t* p_full = bars + 11;
  uint64_t* o_done = bars + 12;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + Cfg::N_BARS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int seq = a.tiles[3 * blockIdx.x], head = a.tiles[3 * blockIdx.x + 1],
            qt = a.tiles[3 * blockIdx.x + 2];
  const int kvh = head / a.group;
  const int q_len = a.q_len[seq], kv_len = a.kv_len[seq];
  const int q0 = a.q_start[seq] + qt * ATT_BM;
  const int kv0 = a.kv_start[seq];
  const int nblk = attn_nblk(a, seq, qt);

  if (threadIdx.x == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 4);
    }
    mbar_init(p_full, 4);
    mbar_init(o_done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const uint32_t t_o = tbase + 256;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------- TMA
      mbar_arrive_expect_tx(q_full, Cfg::TILE_BYTES);
      for (int c = 0; c < Cfg::CH; ++c)
        tma_load_3d(smem + Cfg::Q_OFF + c * 16384, &tmQ, q_full, c * 64, head, q0);
      for (int j = 0; j < nblk; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&k_full[st], Cfg::TILE_BYTES);
        for (int c = 0; c < Cfg::CH; ++c)
          tma_load_3d(smem + Cfg::K_OFF + st * Cfg::TILE_BYTES + c * 16384, &tmK, &k_full[st],
                      c * 64, kvh, kv0 + j * ATT_BN);
        mbar_arrive_expect_tx(&v_full[st], Cfg::TILE_BYTES);
        for (int c = 0; c < Cfg::CH; ++c)
          tma_load_3d(smem + Cfg::V_OFF + st * Cfg::TILE_BYTES + c * 16384, &tmV, &v_full[st],
                      c * 64, kvh, kv0 + j * ATT_BN);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------- MMA
      constexpr uint32_t idesc_s = idesc_bf16_f32(128, ATT_BN, false, false);
      constexpr uint32_t idesc_o = idesc_bf16_f32(128, HD, false, true);
      const uint32_t q_addr = smem_u32(smem + Cfg::Q_OFF);
      const uint32_t p_addr = smem_u32(smem + Cfg::P_OFF);
      mbar_wait(q_full, 0);
      auto issue_pv = [&](int jj) {
        const int st = jj & 1;
        mbar_wait(p_full, jj & 1);
        mbar_wait(&v_full[st], (jj >> 1) & 1);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(smem + Cfg::V_OFF + st * Cfg::TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < ATT_BN / 16; ++kk) {
          const uint64_t adesc = desc_sw128_kmajor(p_addr + (kk >> 2) * 16384 + (kk & 3) * 32);
          const uint64_t bdesc = desc_sw128_mnmajor(v_addr + kk * 2048, 16384);
          mma_ss(t_o, adesc, bdesc, idesc_o, (jj | kk) != 0);
        }
        mma_commit(o_done);
        mma_commit(&kv_empty[st]);
      };
      for (int j = 0; j < nblk; ++j) {
        const int st = j & 1;
        mbar_wait(&k_full[st], (j >> 1) & 1);
        mbar_wait(&s_free[st], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(smem + Cfg::K_OFF + st * Cfg::TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          mma_ss(tbase + st * 128, desc_sw128_kmajor(q_addr + off),
                 desc_sw128_kmajor(k_addr + off), idesc_s, kk != 0);
        }
        mma_commit(&s_full[st]);
        if (j >= 1) issue_pv(j - 1);
      }
      issue_pv(nblk - 1);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------- softmax
    const int ew = warp & 3;
    const int r = ew * 32 + lane;                 // query row in the tile
    const int qrow = qt * ATT_BM + r;             // query index within the sequence
    const int qpos = kv_len - q_len + qrow;       // absolute KV position of the query
    const uint32_t lane_off = (uint32_t)(ew * 32) << 16;
    uint8_t* prow = smem + Cfg::P_OFF + r * 128;
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < nblk; ++j) {
      const int st = j & 1;
      mbar_wait(&s_full[st], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t t_s = tbase + lane_off + st * 128;
      const int kbase = j * ATT_BN;
      const int lim = a.causal ? min(qpos + 1, kv_len) : kv_len;  // visible keys: pos < lim
      // pass 1: row max
      float mx = -INFINITY;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld32(t_s + c * 32, v);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int kp = kbase + c * 32 + i;
          const float s = kp < lim ? __uint_as_float(v[i]) * a.scale_log2 : -INFINITY;
          mx = fmaxf(mx, s);
        }
      }
      const float m_new = fmaxf(m_run, mx);
      const float base = m_new == -INFINITY ? 0.f : m_new;
      const float alpha = fast_exp2(m_run - base);  // 0 when m_run = -inf
      // P buffer / O accumulator are free once PV_{j-1} has completed
      if (j > 0) {
        mbar_wait(o_done, (j - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll 1
          for (int c = 0; c < HD / 16; ++c) {
            uint32_t o[16];
            tmem_ld16(t_o + lane_off + c * 16, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st16(t_o + lane_off + c * 16, o);
          }
          tmem_wait_st();
        }
      }
      // pass 2: p = exp2(s - m), row sum, bf16 P into the SW128 K-major tile
      float rsum = 0.f;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld32(t_s + c * 32, v);
        tmem_wait_ld();
        float p[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int kp = kbase + c * 32 + i;
          p[i] = kp < lim ? fast_exp2(__uint_as_float(v[i]) * a.scale_log2 - base) : 0.f;
          rsum += p[i];
        }
        // 32 columns = 4 chunks of 16 B; atom = c/2, chunk index inside the row
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int chunk = (c & 1) * 4 + q;
          uint4 u;
          u.x = pack_bf16(p[8 * q + 0], p[8 * q + 1]);
          u.y = pack_bf16(p[8 * q + 2], p[8 * q + 3]);
          u.z = pack_bf16(p[8 * q + 4], p[8 * q + 5]);
          u.w = pack_bf16(p[8 * q + 6], p[8 * q + 7]);
          uint8_t* dst = prow + (c >> 1) * 16384 + ((chunk ^ (r & 7)) << 4);
          *reinterpret_cast<uint4*>(dst) = u;
        }
      }
      l_run = l_run * alpha + rsum;
      m_run = m_new;
      fence_async_smem();  // P (generic writes) -> visible to the tensor core
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&s_free[st]);
        mbar_arrive(p_full);
      }
    }
    // epilogue: O / l -> bf16
    mbar_wait(o_done, (nblk - 1) & 1);
    tc_fence_after();
    const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
    const bool ok = qrow < q_len;
    __nv_bfloat16* orow = a.out + (int64_t)(q0 + r) * a.out_tok_stride + (int64_t)head * HD;
#pragma unroll 1
    for (int c = 0; c < HD / 32; ++c) {
      uint32_t o[32];
      tmem_ld32(t_o + lane_off + c * 32, o);
      tmem_wait_ld();
      if (ok) {
        uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 u;
          u.x = pack_bf16(__uint_as_float(o[8 * q + 0]) * inv, __uint_as_float(o[8 * q + 1]) * inv);
          u.y = pack_bf16(__uint_as_float(o[8 * q + 2]) * inv, __uint_as_float(o[8 * q + 3]) * inv);
          u.z = pack_bf16(__uint_as_float(o[8 * q + 4]) * inv, __uint_as_float(o[8 * q + 5]) * inv);
          u.w = pack_bf16(__uint_as_float(o[8 * q + 6]) * inv, __uint_as_float(o[8 * q + 7]) * inv);
          dst[q] = u;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

template <int HD>
static int launch_attn(const void* q, int64_t q_tok_stride, const void* k, const void* v,
                       int64_t kv_tok_stride, int64_t n_q_tokens, int64_t n_kv_tokens,
                       int n_q_heads, int n_kv_heads, const AttnArgs& args, int n_tiles,
                       cudaStream_t stream) {
  using Cfg = AttnCfg<HD>;
  CUtensorMap tq, tk, tv;
  const CUtensorMapDataType bf = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  if (!make_tmap_3d(&tq, q, bf, 2, HD, n_q_heads, n_q_tokens, HD * 2, q_tok_stride * 2, 64, 1,
                    ATT_BM, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_tmap_3d(&tk, k, bf, 2, HD, n_kv_heads, n_kv_tokens, HD * 2, kv_tok_stride * 2, 64,
                    1, ATT_BN, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_tmap_3d(&tv, v, bf, 2, HD, n_kv_heads, n_kv_tokens, HD * 2, kv_tok_stride * 2, 64,
                    1, ATT_BN, CU_TENSOR_MAP_SWIZZLE_128B))
    return EMM_E_INVALID;
  static bool attr_done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_done[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_tc_kernel<HD>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return cuda_status(e, "attn smem attribute");
    attr_done[dev & 63] = true;
  }
  attn_fwd_tc_kernel<HD><<<n_tiles, ATT_THREADS, Cfg::SMEM, stream>>>(tq, tk, tv, args);
  count_launch();
  EMM_CUDA_CHECK_LAUNCH("attn_fwd_tc_kernel");
  return EMM_OK;
}

}  // namespace emm

extern "C" int emm_attention_bf16(const void* q, int64_t q_tok_stride, const void* k,
                                  const void* v, int64_t kv_tok_stride, void* out,
                                  int64_t out_tok_stride, int64_t n_q_tokens,
                                  int64_t n_kv_tokens, int n_q_heads, int n_kv_heads,
                                  int head_dim, const int32_t* tiles, int n_tiles,
                                  const int32_t* q_start, const int32_t* q_len,
                                  const int32_t* kv_start, const int32_t* kv_len, float scale,
                                  int causal, void* stream) {
  using namespace emm;
  if (n_tiles <= 0) return EMM_OK;
  if (!q || !k || !v || !out || n_kv_heads <= 0 || n_q_heads % n_kv_heads != 0 ||
      (head_dim != 64 && head_dim != 128) || (q_tok_stride % 8) || (kv_tok_stride % 8) ||
      (out_tok_stride % 8)) {
    emm_abi::set_error("emm_attention_bf16: head_dim 64/128, GQA divisibility, 16B pitches");
    return EMM_E_INVALID;
  }
  AttnArgs a;
  a.tiles = tiles;
  a.q_start = q_start;
  a.q_len = q_len;
  a.kv_start = kv_start;
  a.kv_len = kv_len;
  a.out = reinterpret_cast<__nv_bfloat16*>(out);
  a.out_tok_stride = out_tok_stride;
  a.n_q_heads = n_q_heads;
  a.group = n_q_heads / n_kv_heads;
  a.scale_log2 = scale * 1.4426950408889634f;
  a.causal = causal;
  cudaStream_t st = (cudaStream_t)stream;
  if (head_dim == 128)
    return launch_attn<128>(q, q_tok_stride, k, v, kv_tok_stride, n_q_tokens, n_kv_tokens,
                            n_q_heads, n_kv_heads, a, n_tiles, st);
  return launch_attn<64>(q, q_tok_stride, k, v, kv_tok_stride, n_q_tokens, n_kv_tokens,
                         n_q_heads, n_kv_heads, a, n_tiles, st);
}
