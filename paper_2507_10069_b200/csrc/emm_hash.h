// emm_hash.h — the block-hash function shared by the host control plane and
// the sm_100a kernels (K1).  Pure integer arithmetic, __host__ __device__.
//
// The reference keys its prefix tree by Python tuples (pkg/src/mmsim/engine.py:448-461)
// and never hashes anything; a GPU index needs fixed-width keys, so this file
// DEFINES the hash ("block hashes ... parity unpinned, the
// builder's own CPU restatement pins them").  The C restatement in
// oracle/hash_oracle.c implements the same definition independently.
//
//   symbol key  k  : uint64, injective encoding of a unified-sequence symbol
//                    (tag in bits 63..62, see paper_2507_10069_b200/keys.py)
//   weight      w  : KV-token weight of the symbol (image = token_count)
//   lane l in {0,1}, p = 2^61 - 1:
//     x_l(k,w) = red( mix(k ^ S_l) ^ mix(w + T_l) )
//     P_l(0)   = H_l ;  P_l(i) = P_l(i-1) * B_l + x_l(k_i, w_i)   (mod p)
//   block hash of position i = (P_0(i), P_1(i))  — 122 bits.
//
//   pixel digest of n bytes (8-byte little-endian words u_j, last zero-padded):
//     D_l = G_l ; D_l = D_l * C_l + red(mix(u_j ^ R_l)) for every word ;
//     D_l = D_l * C_l + red(mix(n ^ Q_l))                       (mod p)
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define EMM_HD __host__ __device__ __forceinline__
#else
#define EMM_HD static inline
#endif

#define EMM_M61 0x1FFFFFFFFFFFFFFFull

// prefix-hash constants (lane 0, lane 1)
#define EMM_B0 0x0F1E2D3C4B5A6978ull
#define EMM_B1 0x1A2B3C4D5E6F7081ull
#define EMM_S0 0x9E3779B97F4A7C15ull
#define EMM_S1 0xC2B2AE3D27D4EB4Full
#define EMM_T0 0x165667B19E3779F9ull
#define EMM_T1 0x27D4EB2F165667C5ull
#define EMM_H0 0x00123456789ABCDEull
#define EMM_H1 0x0FEDCBA987654321ull
// pixel-digest constants
#define EMM_C0 0x01234567890ABCDEull
#define EMM_C1 0x0DEADBEEFCAFEBABull
#define EMM_R0 0x5851F42D4C957F2Dull
#define EMM_R1 0x14057B7EF767814Full
#define EMM_Q0 0x2545F4914F6CDD1Dull
#define EMM_Q1 0x3C6EF372FE94F82Bull
#define EMM_G0 0x0A5A5A5A5A5A5A5Aull
#define EMM_G1 0x15A5A5A5A5A5A5A5ull

EMM_HD uint64_t emm_mix64(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27; z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

EMM_HD uint64_t emm_red61(uint64_t z) {
  uint64_t r = (z & EMM_M61) + (z >> 61);
  return r >= EMM_M61 ? r - EMM_M61 : r;
}

EMM_HD uint64_t emm_mulmod61(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
  uint64_t lo = a * b;
  uint64_t hi = __umul64hi(a, b);
#else
  unsigned __int128 p = (unsigned __int128)a * b;
  uint64_t lo = (uint64_t)p, hi = (uint64_t)(p >> 64);
#endif
  // p = hi*2^64 + lo ; 2^64 = 8 * 2^61 == 8 (mod M61)
  uint64_t r = (lo & EMM_M61) + (lo >> 61) + (hi << 3);
  r = (r & EMM_M61) + (r >> 61);
  return r >= EMM_M61 ? r - EMM_M61 : r;
}

EMM_HD uint64_t emm_addmod61(uint64_t a, uint64_t b) {
  uint64_t r = a + b;
  return r >= EMM_M61 ? r - EMM_M61 : r;
}

EMM_HD uint64_t emm_sym_term(uint64_t key, uint64_t w, int lane) {
  uint64_t s = lane ? EMM_S1 : EMM_S0, t = lane ? EMM_T1 : EMM_T0;
  return emm_red61(emm_mix64(key ^ s) ^ emm_mix64(w + t));
}

EMM_HD uint64_t emm_pix_term(uint64_t word, int lane) {
  return emm_red61(emm_mix64(word ^ (lane ? EMM_R1 : EMM_R0)));
}

// Sentinels for the device hash table: real hashes are < 2^61.
#define EMM_HT_EMPTY 0xFFFFFFFFFFFFFFFFull
#define EMM_HT_TOMB 0xFFFFFFFFFFFFFFFEull
