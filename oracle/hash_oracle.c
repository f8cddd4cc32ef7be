/* hash_oracle.c — TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * Independent, sequential CPU restatement of the block-hash and pixel-digest
 * definitions written down in paper_2507_10069_b200/csrc/emm_hash.h.  The
 * reference keys its radix tree by Python tuples (pkg/src/mmsim/engine.py:
 * 448-461) and hashes image identity strings (pkg/src/mmsim/workload.py:
 * 191-192), so these hashes have no reference counterpart: they are pinned by
 * this restatement plus the known-answer vectors in tests/golden/hash_kats.json
 * (parity of the hashes themselves is "builder-pinned").  What
 * the reference DOES pin — which symbols match, matched KV weight, eviction
 * order — is checked against its recorded call logs.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
 * this library (oracle/_build/liboracle.so).
 *
 * Arithmetic is done with plain 64x64->128 multiplication and % on the
 * Mersenne prime, deliberately not sharing code with the product.
 */
#include <stdint.h>
#include <string.h>

typedef unsigned __int128 u128;
static const uint64_t P61 = (1ull << 61) - 1;

static uint64_t mulp(uint64_t a, uint64_t b) { return (uint64_t)(((u128)a * b) % P61); }
static uint64_t addp(uint64_t a, uint64_t b) { return (uint64_t)(((u128)a + b) % P61); }

static uint64_t splitmix_fin(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static uint64_t modp(uint64_t z) { return z % P61; }

/* lane constants: base, key salt, weight salt, seed */
static const uint64_t BASE[2] = {0x0F1E2D3C4B5A6978ull, 0x1A2B3C4D5E6F7081ull};
static const uint64_t KSALT[2] = {0x9E3779B97F4A7C15ull, 0xC2B2AE3D27D4EB4Full};
static const uint64_t WSALT[2] = {0x165667B19E3779F9ull, 0x27D4EB2F165667C5ull};
static const uint64_t SEED[2] = {0x00123456789ABCDEull, 0x0FEDCBA987654321ull};
/* pixel digest */
static const uint64_t PBASE[2] = {0x01234567890ABCDEull, 0x0DEADBEEFCAFEBABull};
static const uint64_t PSALT[2] = {0x5851F42D4C957F2Dull, 0x14057B7EF767814Full};
static const uint64_t LSALT[2] = {0x2545F4914F6CDD1Dull, 0x3C6EF372FE94F82Bull};
static const uint64_t PSEED[2] = {0x0A5A5A5A5A5A5A5Aull, 0x15A5A5A5A5A5A5A5ull};

/* prefix hashes of one sequence: out0[i], out1[i] = lane values at symbol i */
void oracle_prefix_hashes(const uint64_t* keys, const int64_t* w, int64_t n, uint64_t* out0,
                          uint64_t* out1) {
  for (int lane = 0; lane < 2; ++lane) {
    uint64_t h = SEED[lane];
    uint64_t* out = lane ? out1 : out0;
    for (int64_t i = 0; i < n; ++i) {
      uint64_t x = splitmix_fin(keys[i] ^ KSALT[lane]) ^ splitmix_fin((uint64_t)w[i] + WSALT[lane]);
      h = addp(mulp(h, BASE[lane]), modp(x));
      out[i] = h;
    }
  }
}

/* digest of n bytes: 8-byte little-endian words, last one zero-padded */
void oracle_pixel_digest(const uint8_t* bytes, int64_t n, uint64_t out[2]) {
  for (int lane = 0; lane < 2; ++lane) {
    uint64_t h = PSEED[lane];
    for (int64_t off = 0; off < n; off += 8) {
      uint64_t word = 0;
      for (int b = 0; b < 8; ++b)
        if (off + b < n) word |= (uint64_t)bytes[off + b] << (8 * b);
      h = addp(mulp(h, PBASE[lane]), modp(splitmix_fin(word ^ PSALT[lane])));
    }
    h = addp(mulp(h, PBASE[lane]), modp(splitmix_fin((uint64_t)n ^ LSALT[lane])));
    out[lane] = h;
  }
}

/* KV-token block table of a request whose first `m` symbols are cached:
 * symbol j covers KV tokens [cum_{j-1}, cum_j).  Given the per-symbol first
 * pool slot lists (slot_of_token for each cached token, concatenated in
 * symbol order), the table is the first `want` entries — a restatement of
 * the device emission used by the gather tests. */
int64_t oracle_block_table(const int64_t* w, int64_t m, int64_t want, const int32_t* slots,
                           int32_t* out) {
  int64_t total = 0;
  for (int64_t j = 0; j < m; ++j) total += w[j];
  if (want > total) want = total;
  memcpy(out, slots, (size_t)want * sizeof(int32_t));
  return want;
}
