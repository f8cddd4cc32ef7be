// dataplane.cu — device mirror of one PrefixTree (K2) and its KV storage.
//
// The host tree (host_cache.cpp) stays the authority for every decision
// (pins, splits, LRU eviction).  Through the TreeHooks journal this index
// keeps, on the GPU:
//   * an open-addressing hash table  block-hash(symbol prefix) -> (vstart, w)
//     holding exactly the reachable cached symbol prefixes (prefix-closed,
//     so a request's longest cached prefix is its first probe miss);
//   * tok_slot[v]: virtual token record -> physical KV-pool slot.  A node's
//     tokens occupy one contiguous virtual range, so splits never move KV
//      and block tables are a gather through tok_slot;
//   * the paged KV pool itself lives in torch memory; this index only
//     allocates slots (free stack) and scatters inserted KV into them.
// Unreachable "ghost" tails are never published.
#include <cuda_runtime.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <unordered_map>
#include <vector>

#include "../../include/emm.h"
#include "emm_hash.h"
#include "abi_util.h"
#include "host_cache.h"
#include "ptx.cuh"
#include "runtime.h"

namespace emm {
int kv_copy_rows_launch(const void* src, int64_t src_stride, const int32_t* src_rows, void* dst,
                        int64_t dst_stride, const int32_t* dst_rows, int64_t n_rows,
                        int64_t row_bytes, int64_t n_layers, cudaStream_t stream);

struct HtEntry {
  uint64_t h0, h1;
  int64_t vstart, w;
};
static_assert(sizeof(HtEntry) == 32, "entry size");

// ------------------------------------------------------------------ kernels

__device__ __forceinline__ HtEntry ht_load(const HtEntry* t, uint64_t slot) {
  const uint4* p = reinterpret_cast<const uint4*>(t + slot);
  uint4 a = p[0], b = p[1];
  HtEntry e;
  e.h0 = ((uint64_t)a.y << 32) | a.x;
  e.h1 = ((uint64_t)a.w << 32) | a.z;
  e.vstart = (int64_t)(((uint64_t)b.y << 32) | b.x);
  e.w = (int64_t)(((uint64_t)b.w << 32) | b.z);
  return e;
}

__global__ void ht_erase_kernel(HtEntry* table, uint64_t mask, const uint64_t* __restrict__ keys,
                                int64_t n, int* err) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t k0 = keys[2 * i], k1 = keys[2 * i + 1];
  uint64_t slot = k0 & mask;
  for (uint64_t probe = 0; probe <= mask; ++probe) {
    const uint64_t h = table[slot].h0;
    if (h == EMM_HT_EMPTY) break;
    if (h == k0 && table[slot].h1 == k1) {
      table[slot].h0 = EMM_HT_TOMB;
      return;
    }
    slot = (slot + 1) & mask;
  }
  atomicExch(err, 1);
}

__global__ void ht_publish_kernel(HtEntry* table, uint64_t mask, const HtEntry* __restrict__ ops,
                                  int64_t n, int* err) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const HtEntry e = ops[i];
  uint64_t slot = e.h0 & mask;
  for (uint64_t probe = 0; probe <= mask; ++probe) {
    unsigned long long* hp = reinterpret_cast<unsigned long long*>(&table[slot].h0);
    unsigned long long cur = *((volatile unsigned long long*)hp);
    if (cur == EMM_HT_EMPTY || cur == EMM_HT_TOMB) {
      if (atomicCAS(hp, cur, (unsigned long long)e.h0) == cur) {
        table[slot].h1 = e.h1;
        table[slot].vstart = e.vstart;
        table[slot].w = e.w;
        return;
      }
      continue;  // lost the race: re-read this slot
    }
    slot = (slot + 1) & mask;
  }
  atomicExch(err, 2);
}

__global__ void tok_slot_set_kernel(int32_t* tok_slot, const int64_t* __restrict__ v,
                                    const int32_t* __restrict__ s, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) tok_slot[v[i]] = s[i];
}

constexpr int MATCH_THREADS = 256;

// K2: one CTA per request.  Probe every symbol's block hash; the first miss
// is the match length (the cached set is prefix-closed).  Then emit the
// token-granular block table for KV tokens [0, want_kv).
__global__ void __launch_bounds__(MATCH_THREADS) prefix_match_kernel(
    const HtEntry* __restrict__ table, uint64_t mask, const int32_t* __restrict__ tok_slot,
    const uint64_t* __restrict__ h0, const uint64_t* __restrict__ h1,
    const int64_t* __restrict__ cumw, const int64_t* __restrict__ seq_off,
    const int64_t* __restrict__ want_kv, const int64_t* __restrict__ bt_off,
    int64_t* __restrict__ matched_sym, int64_t* __restrict__ matched_kv,
    int64_t* __restrict__ sym_v, int32_t* __restrict__ bt) {
  __shared__ long long first_miss;
  const int s = blockIdx.x;
  const int64_t beg = seq_off[s], end = seq_off[s + 1];
  const int64_t n = end - beg;
  if (threadIdx.x == 0) first_miss = n;
  __syncthreads();
  for (int64_t base = 0; base < n; base += MATCH_THREADS) {
    if (base >= first_miss) break;  // uniform: read after the barrier
    const int64_t j = base + threadIdx.x;
    if (j < n) {
      const uint64_t k0 = h0[beg + j], k1 = h1[beg + j];
      uint64_t slot = k0 & mask;
      int64_t v = -1;
      for (uint64_t probe = 0; probe <= mask; ++probe) {
        const HtEntry e = ht_load(table, slot);
        if (e.h0 == EMM_HT_EMPTY) break;
        if (e.h0 == k0 && e.h1 == k1) {
          v = e.vstart;
          break;
        }
        slot = (slot + 1) & mask;
      }
      if (v < 0)
        atomicMin(&first_miss, (long long)j);
      else
        sym_v[beg + j] = v;
    }
    __syncthreads();
  }
  const int64_t m = first_miss;
  const int64_t mkv = m > 0 ? cumw[beg + m - 1] : 0;
  if (threadIdx.x == 0) {
    matched_sym[s] = m;
    matched_kv[s] = mkv;
  }
  const int64_t want = min(want_kv[s], mkv);
  int32_t* out = bt + bt_off[s];
  for (int64_t t = threadIdx.x; t < want; t += MATCH_THREADS) {
    // symbol j with cumw[j-1] <= t < cumw[j]
    int64_t lo = 0, hi = m - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (cumw[beg + mid] > t)
        hi = mid;
      else
        lo = mid + 1;
    }
    const int64_t start = lo > 0 ? cumw[beg + lo - 1] : 0;
    out[t] = tok_slot[sym_v[beg + lo] + (t - start)];
  }
}

}  // namespace emm

using emm::HtEntry;

// ----------------------------------------------------------------- DeviceIndex

struct emm_index : public emm::TreeHooks {
  struct emm_cache* cache = nullptr;
  emm::PrefixTree* tree = nullptr;
  int device = 0;
  cudaStream_t stream = nullptr;
  // device state
  HtEntry* table = nullptr;
  uint64_t cap = 0;
  int32_t* tok_slot = nullptr;
  int* err = nullptr;
  int64_t v_tokens = 0, n_slots = 0;
  // host mirrors / allocators
  std::vector<int32_t> tok_slot_host;
  std::map<int64_t, int64_t> vfree;  // start -> length (coalesced extents)
  std::vector<int32_t> slot_free;
  int64_t n_live = 0, n_tomb = 0;
  // pending device ops, in host order (coalesced at flush time)
  struct HtOp {
    HtEntry e;
    bool publish;
  };
  std::vector<HtOp> ht_ops;
  std::vector<std::pair<int64_t, int32_t>> tok_ops;  // v -> slot
  std::vector<std::pair<int32_t, int64_t>> sc_ops;   // dst slot <- (buffer << 40 | src row)
  bool need_rebuild = false;
  // flush outputs (coalesced)
  std::vector<uint64_t> erase_ops;  // pairs
  std::vector<HtEntry> pub_ops;
  std::vector<int64_t> tok_v;
  std::vector<int32_t> tok_s;
  std::vector<int64_t> sc_src;  // buffer << 40 | row
  std::vector<int32_t> sc_dst;
  // KV sources and geometry
  std::map<std::pair<uint64_t, uint64_t>, int64_t> kv_src;
  void* pool = nullptr;
  int64_t pool_kv_stride = 0;
  // request KV buffers the scatter reads (buffer 0 = the set_kv_geometry one;
  // more are added for prefill batches split across GPUs, read peer-to-peer)
  std::vector<void*> reqs;
  std::vector<int64_t> req_strides;
  int64_t row_bytes = 0, n_layers = 0;
  // staging
  uint8_t* dev_stage = nullptr;
  size_t dev_stage_cap = 0;
  static constexpr int RING = 32;
  uint8_t* pinned[RING] = {nullptr};
  size_t pinned_cap[RING] = {0};
  cudaEvent_t ev[RING] = {nullptr};
  int ring_head = 0;
  // scratch for hashes of the sequence being inserted
  std::vector<uint64_t> hh0, hh1;

  ~emm_index() {
    cudaFree(table);
    cudaFree(tok_slot);
    cudaFree(err);
    cudaFree(dev_stage);
    for (int i = 0; i < RING; ++i) {
      if (pinned[i]) cudaFreeHost(pinned[i]);
      if (ev[i]) cudaEventDestroy(ev[i]);
    }
  }

  int64_t valloc(int64_t n) {
    for (auto it = vfree.begin(); it != vfree.end(); ++it) {
      if (it->second >= n) {
        const int64_t start = it->first, len = it->second;
        vfree.erase(it);
        if (len > n) vfree[start + n] = len - n;
        return start;
      }
    }
    throw emm::CacheError{EMM_E_OOM, "virtual token space exhausted (fragmentation)"};
  }
  void vrelease(int64_t start, int64_t n) {
    if (n <= 0) return;
    auto next = vfree.lower_bound(start);
    if (next != vfree.end() && next->first == start + n) {
      n += next->second;
      next = vfree.erase(next);
    }
    if (next != vfree.begin()) {
      auto prev = std::prev(next);
      if (prev->first + prev->second == start) {
        prev->second += n;
        return;
      }
    }
    vfree[start] = n;
  }

  void on_new_node(emm::Node* node, const uint64_t* keys, const int64_t* w, int64_t n_total,
                   int64_t pos) override {
    hh0.resize(n_total);
    hh1.resize(n_total);
    uint64_t a = EMM_H0, b = EMM_H1;
    int64_t kv_before = 0;
    for (int64_t i = 0; i < n_total; ++i) {
      a = emm_addmod61(emm_mulmod61(a, EMM_B0), emm_sym_term(keys[i], (uint64_t)w[i], 0));
      b = emm_addmod61(emm_mulmod61(b, EMM_B1), emm_sym_term(keys[i], (uint64_t)w[i], 1));
      hh0[i] = a;
      hh1[i] = b;
      if (i < pos) kv_before += w[i];
    }
    const int64_t len = (int64_t)node->span.size();
    if (node->kv > (int64_t)slot_free.size())
      throw emm::CacheError{EMM_E_OOM, "KV pool has no free slots for the insert"};
    const int64_t vstart = valloc(node->kv);
    node->recs.resize(len);
    int64_t v = vstart;
    for (int64_t i = 0; i < len; ++i) {
      node->recs[i] = emm::SymRec{hh0[pos + i], hh1[pos + i], v, w[pos + i]};
      ht_ops.push_back(HtOp{HtEntry{hh0[pos + i], hh1[pos + i], v, w[pos + i]}, true});
      v += w[pos + i];
    }
    n_live += len;
    // KV source registered for this sequence?
    auto it = kv_src.find({hh0[n_total - 1], hh1[n_total - 1]});
    for (int64_t t = 0; t < node->kv; ++t) {
      const int32_t slot = slot_free.back();
      slot_free.pop_back();
      tok_slot_host[vstart + t] = slot;
      tok_ops.push_back({vstart + t, slot});
      if (it != kv_src.end()) sc_ops.push_back({slot, it->second + kv_before + t});
    }
    if ((double)(n_live + n_tomb) > 0.7 * (double)cap) need_rebuild = true;
  }

  void on_evict(emm::Node* node) override {
    if (node->recs.empty()) return;
    for (auto& r : node->recs) {
      ht_ops.push_back(HtOp{HtEntry{r.h0, r.h1, r.vstart, r.w}, false});
      for (int64_t t = 0; t < r.w; ++t) slot_free.push_back(tok_slot_host[r.vstart + t]);
    }
    vrelease(node->recs[0].vstart, node->kv);
    n_live -= (int64_t)node->recs.size();
    n_tomb += (int64_t)node->recs.size();
    if ((double)(n_live + n_tomb) > 0.7 * (double)cap) need_rebuild = true;
  }

  // pinned staging slot for `bytes`, waiting for its previous copy to finish
  uint8_t* stage_host(size_t bytes, int& slot) {
    slot = ring_head;
    ring_head = (ring_head + 1) % RING;
    if (ev[slot]) cudaEventSynchronize(ev[slot]);
    if (pinned_cap[slot] < bytes) {
      if (pinned[slot]) cudaFreeHost(pinned[slot]);
      size_t c = bytes < (1u << 20) ? (1u << 20) : bytes * 2;
      if (cudaMallocHost(&pinned[slot], c) != cudaSuccess)
        throw emm::CacheError{EMM_E_OOM, "pinned staging allocation failed"};
      pinned_cap[slot] = c;
    }
    return pinned[slot];
  }
  uint8_t* stage_dev(size_t bytes) {
    if (dev_stage_cap < bytes) {
      cudaStreamSynchronize(stream);
      cudaFree(dev_stage);
      dev_stage = nullptr;
      dev_stage_cap = 0;
      size_t c = bytes * 2 < (16u << 20) ? (16u << 20) : bytes * 2;
      if (cudaMalloc(&dev_stage, c) != cudaSuccess) {
        cudaGetLastError();  // clear the sticky-free OOM status
        dev_stage = nullptr;  // the caller may free memory and retry (dataplane.py)
        throw emm::CacheError{EMM_E_OOM, "device staging allocation failed"};
      }
      dev_stage_cap = c;
    }
    return dev_stage;
  }

  void rebuild_table() {
    // drop pending table ops: rebuild from the authoritative host tree
    ht_ops.clear();
    erase_ops.clear();
    pub_ops.clear();
    std::vector<const emm::Node*> nodes;
    tree->collect_nodes(nodes);
    for (const emm::Node* nd : nodes)
      for (auto& r : nd->recs) pub_ops.push_back(HtEntry{r.h0, r.h1, r.vstart, r.w});
    cudaMemsetAsync(table, 0xFF, cap * sizeof(HtEntry), stream);
    n_live = (int64_t)pub_ops.size();
    n_tomb = 0;
    need_rebuild = false;
  }

  // Coalesce the journal: per key the first op tells presence before the
  // window (an erase implies present, a publish implies absent) and the last
  // op presence after it; tok_slot / scatter writes are last-writer-wins
  // (a slot freed and re-allocated inside the window keeps only its final
  // contents), which makes one batched launch equal the sequential result.
  void coalesce() {
    erase_ops.clear();
    pub_ops.clear();
    tok_v.clear();
    tok_s.clear();
    sc_src.clear();
    sc_dst.clear();
    struct KeyState {
      bool first_publish;
      bool last_publish;
      HtEntry last;
    };
    std::unordered_map<uint64_t, std::vector<std::pair<uint64_t, KeyState>>> ks;
    std::vector<std::pair<uint64_t, uint64_t>> order;
    for (auto& op : ht_ops) {
      auto& bucket = ks[op.e.h0];
      KeyState* st = nullptr;
      for (auto& kv : bucket)
        if (kv.first == op.e.h1) st = &kv.second;
      if (!st) {
        bucket.push_back({op.e.h1, KeyState{op.publish, op.publish, op.e}});
        order.push_back({op.e.h0, op.e.h1});
      } else {
        st->last_publish = op.publish;
        st->last = op.e;
      }
    }
    for (auto& k : order) {
      KeyState* st = nullptr;
      for (auto& kv : ks[k.first])
        if (kv.first == k.second) st = &kv.second;
      const bool present_before = !st->first_publish, present_after = st->last_publish;
      if (present_before) {
        erase_ops.push_back(k.first);
        erase_ops.push_back(k.second);
      }
      if (present_after) pub_ops.push_back(st->last);
    }
    ht_ops.clear();
    std::unordered_map<int64_t, size_t> tv;
    for (auto& o : tok_ops) {
      auto it = tv.find(o.first);
      if (it == tv.end()) {
        tv[o.first] = tok_v.size();
        tok_v.push_back(o.first);
        tok_s.push_back(o.second);
      } else {
        tok_s[it->second] = o.second;
      }
    }
    tok_ops.clear();
    std::unordered_map<int32_t, size_t> sd;
    for (auto& o : sc_ops) {
      auto it = sd.find(o.first);
      if (it == sd.end()) {
        sd[o.first] = sc_dst.size();
        sc_dst.push_back(o.first);
        sc_src.push_back(o.second);
      } else {
        sc_src[it->second] = o.second;
      }
    }
    sc_ops.clear();
  }

  // coalesced ops of a flush that failed before launching (staging OOM):
  // the retry uploads them as they are
  bool pending_coalesced() const {
    return !erase_ops.empty() || !pub_ops.empty() || !tok_v.empty() || !sc_src.empty();
  }

  bool dirty() const {
    return need_rebuild || !ht_ops.empty() || !tok_ops.empty() || !sc_ops.empty() ||
           pending_coalesced();
  }

  int flush() {
    if (!dirty()) return EMM_OK;
    if (!pending_coalesced()) {
      coalesce();
      if (need_rebuild) rebuild_table();
    }
    if (erase_ops.empty() && pub_ops.empty() && tok_v.empty() && sc_src.empty()) return EMM_OK;
    const size_t n_er = erase_ops.size() / 2, n_pub = pub_ops.size(), n_tok = tok_v.size(),
                 n_sc = sc_src.size();
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t o_er = 0, o_pub = al(o_er + n_er * 16), o_tv = al(o_pub + n_pub * 32),
                 o_ts = al(o_tv + n_tok * 8), o_ss = al(o_ts + n_tok * 4),
                 o_sd = al(o_ss + n_sc * 4), total = al(o_sd + n_sc * 4);
    int slot;
    uint8_t* h = stage_host(total, slot);
    memcpy(h + o_er, erase_ops.data(), n_er * 16);
    memcpy(h + o_pub, pub_ops.data(), n_pub * 32);
    memcpy(h + o_tv, tok_v.data(), n_tok * 8);
    memcpy(h + o_ts, tok_s.data(), n_tok * 4);
    // scatter entries grouped by source buffer: rows (int32) and slots
    std::vector<size_t> ord(n_sc);
    for (size_t i = 0; i < n_sc; ++i) ord[i] = i;
    std::stable_sort(ord.begin(), ord.end(),
                     [&](size_t a, size_t b) { return (sc_src[a] >> 40) < (sc_src[b] >> 40); });
    std::vector<std::pair<int64_t, size_t>> seg;  // (buffer, first index)
    {
      int32_t* hs = reinterpret_cast<int32_t*>(h + o_ss);
      int32_t* hd = reinterpret_cast<int32_t*>(h + o_sd);
      for (size_t i = 0; i < n_sc; ++i) {
        const int64_t src = sc_src[ord[i]], buf = src >> 40;
        if (seg.empty() || seg.back().first != buf) seg.push_back({buf, i});
        hs[i] = (int32_t)(src & ((int64_t(1) << 40) - 1));
        hd[i] = sc_dst[ord[i]];
      }
    }
    uint8_t* d = stage_dev(total);
    cudaError_t e = cudaMemcpyAsync(d, h, total, cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return emm::cuda_status(e, "index staging upload");
    if (!ev[slot]) cudaEventCreateWithFlags(&ev[slot], cudaEventDisableTiming);
    cudaEventRecord(ev[slot], stream);
    const uint64_t mask = cap - 1;
    if (n_er) {
      emm::ht_erase_kernel<<<(unsigned)((n_er + 255) / 256), 256, 0, stream>>>(
          table, mask, reinterpret_cast<uint64_t*>(d + o_er), (int64_t)n_er, err);
      emm::count_launch();
    }
    if (n_pub) {
      emm::ht_publish_kernel<<<(unsigned)((n_pub + 255) / 256), 256, 0, stream>>>(
          table, mask, reinterpret_cast<HtEntry*>(d + o_pub), (int64_t)n_pub, err);
      emm::count_launch();
    }
    if (n_tok) {
      emm::tok_slot_set_kernel<<<(unsigned)((n_tok + 255) / 256), 256, 0, stream>>>(
          tok_slot, reinterpret_cast<int64_t*>(d + o_tv), reinterpret_cast<int32_t*>(d + o_ts),
          (int64_t)n_tok);
      emm::count_launch();
    }
    EMM_CUDA_CHECK_LAUNCH("index update kernels");
    for (size_t g = 0; g < seg.size(); ++g) {
      const int64_t buf = seg[g].first;
      const size_t i0 = seg[g].second, i1 = g + 1 < seg.size() ? seg[g + 1].second : n_sc;
      if (!pool || buf >= (int64_t)reqs.size() || !reqs[buf]) {
        emm_abi::set_error("KV source registered but KV geometry / request buffer not set");
        return EMM_E_INVALID;
      }
      int rc = emm::kv_copy_rows_launch(
          reqs[buf], req_strides[buf], reinterpret_cast<int32_t*>(d + o_ss) + i0, pool,
          pool_kv_stride, reinterpret_cast<int32_t*>(d + o_sd) + i0, (int64_t)(i1 - i0),
          row_bytes, n_layers, stream);
      if (rc != EMM_OK) return rc;
    }
    erase_ops.clear();
    pub_ops.clear();
    tok_v.clear();
    tok_s.clear();
    sc_src.clear();
    sc_dst.clear();
    return EMM_OK;
  }
};

// emm_cache internals (abi_host.cpp) — only the pieces needed here
struct emm_cache_view {
  emm::UnifiedCache uc;
};

extern "C" int emm_cache_parts(emm_cache* c, emm_pool** images, emm_tree** prefixes);
extern "C" int emm_cache_set_index_(emm_cache* c, emm_index* ix);

extern "C" int emm_index_attach(emm_cache* c, int device, int64_t max_syms, int64_t v_tokens,
                                int64_t n_slots, emm_index** out) {
  if (!c || !out || max_syms <= 0 || v_tokens <= 0 || n_slots <= 0 || n_slots > (1ll << 31)) {
    emm_abi::set_error("emm_index_attach: bad arguments");
    return EMM_E_INVALID;
  }
  emm_tree* t = nullptr;
  emm_cache_parts(c, nullptr, &t);
  emm::PrefixTree* tree = reinterpret_cast<emm::PrefixTree*>(t);
  if (tree->total_tokens() != 0) {
    emm_abi::set_error("emm_index_attach: attach before the first insert");
    return EMM_E_INVALID;
  }
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  auto* ix = new emm_index();
  ix->cache = c;
  ix->tree = tree;
  ix->device = device;
  uint64_t cap = 1024;
  while (cap < (uint64_t)max_syms * 2) cap <<= 1;
  ix->cap = cap;
  ix->v_tokens = v_tokens;
  ix->n_slots = n_slots;
  cudaError_t e = cudaMalloc(&ix->table, cap * sizeof(HtEntry));
  if (e == cudaSuccess) e = cudaMalloc(&ix->tok_slot, v_tokens * sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMalloc(&ix->err, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(ix->table, 0xFF, cap * sizeof(HtEntry));
  if (e == cudaSuccess) e = cudaMemset(ix->tok_slot, 0xFF, v_tokens * sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMemset(ix->err, 0, sizeof(int));
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    delete ix;
    return emm::cuda_status(e, "emm_index_attach allocation");
  }
  ix->tok_slot_host.assign(v_tokens, -1);
  ix->vfree[0] = v_tokens;
  ix->slot_free.resize(n_slots);
  for (int64_t i = 0; i < n_slots; ++i) ix->slot_free[i] = (int32_t)(n_slots - 1 - i);
  tree->set_hooks(ix);
  emm_cache_set_index_(c, ix);
  *out = ix;
  return EMM_OK;
}

extern "C" int emm_index_detach_(emm_index* ix) {
  if (!ix) return EMM_OK;
  ix->tree->set_hooks(nullptr);
  delete ix;
  return EMM_OK;
}

extern "C" int emm_index_set_stream(emm_index* ix, void* stream) {
  if (!ix) return EMM_E_INVALID;
  ix->stream = (cudaStream_t)stream;
  return EMM_OK;
}

extern "C" int emm_index_set_kv_source(emm_index* ix, uint64_t h0, uint64_t h1,
                                       int64_t src_row0) {
  if (!ix) return EMM_E_INVALID;
  ix->kv_src[{h0, h1}] = src_row0;
  return EMM_OK;
}

extern "C" int emm_index_set_kv_source_buf(emm_index* ix, uint64_t h0, uint64_t h1, int buffer,
                                           int64_t src_row0) {
  if (!ix || buffer < 0 || buffer >= (int)ix->reqs.size() || src_row0 < 0 ||
      src_row0 >= (int64_t(1) << 31))
    return EMM_E_INVALID;
  ix->kv_src[{h0, h1}] = (int64_t(buffer) << 40) | src_row0;
  return EMM_OK;
}

extern "C" int emm_index_add_request_buffer(emm_index* ix, void* req, int64_t req_kv_stride,
                                            int* buffer) {
  if (!ix || !req || !buffer || !ix->pool) return EMM_E_INVALID;
  ix->reqs.push_back(req);
  ix->req_strides.push_back(req_kv_stride);
  *buffer = (int)ix->reqs.size() - 1;
  return EMM_OK;
}

extern "C" int emm_index_clear_kv_sources(emm_index* ix) {
  if (!ix) return EMM_E_INVALID;
  ix->kv_src.clear();
  return EMM_OK;
}

extern "C" int emm_index_set_kv_geometry(emm_index* ix, void* pool, int64_t pool_kv_stride,
                                         void* req, int64_t req_kv_stride, int64_t row_bytes,
                                         int64_t n_layers) {
  if (!ix) return EMM_E_INVALID;
  if (ix->dirty()) {  // pending scatters refer to the previous request buffer
    try {
      int rc = ix->flush();
      if (rc != EMM_OK) return rc;
    } catch (const emm::CacheError& e) {
      emm_abi::set_error(e.msg);
      return e.code;
    }
  }
  ix->pool = pool;
  ix->pool_kv_stride = pool_kv_stride;
  ix->reqs.assign(1, req);
  ix->req_strides.assign(1, req_kv_stride);
  ix->row_bytes = row_bytes;
  ix->n_layers = n_layers;
  return EMM_OK;
}

extern "C" int emm_index_flush(emm_index* ix, void* stream) {
  if (!ix) return EMM_E_INVALID;
  if (stream) ix->stream = (cudaStream_t)stream;
  try {
    return ix->flush();
  } catch (const emm::CacheError& e) {
    emm_abi::set_error(e.msg);
    return e.code;
  }
}

extern "C" int emm_index_match(emm_index* ix, const uint64_t* h0, const uint64_t* h1,
                               const int64_t* cumw, const int64_t* seq_off, int64_t n_seqs,
                               const int64_t* want_kv, const int64_t* bt_off,
                               int64_t* matched_sym, int64_t* matched_kv, int64_t* sym_v,
                               int32_t* bt, void* stream) {
  if (!ix) return EMM_E_INVALID;
  if (n_seqs <= 0) return EMM_OK;
  cudaStream_t st = stream ? (cudaStream_t)stream : ix->stream;
  if (ix->dirty()) {  // the device mirror must reflect every host decision so far
    ix->stream = st;
    try {
      int rc = ix->flush();
      if (rc != EMM_OK) return rc;
    } catch (const emm::CacheError& e) {
      emm_abi::set_error(e.msg);
      return e.code;
    }
  }
  emm::prefix_match_kernel<<<(unsigned)n_seqs, emm::MATCH_THREADS, 0, st>>>(
      ix->table, ix->cap - 1, ix->tok_slot, h0, h1, cumw, seq_off, want_kv, bt_off, matched_sym,
      matched_kv, sym_v, bt);
  emm::count_launch();
  EMM_CUDA_CHECK_LAUNCH("prefix_match_kernel");
  return EMM_OK;
}

extern "C" int emm_index_info(emm_index* ix, int64_t out6[6]) {
  if (!ix) return EMM_E_INVALID;
  out6[0] = ix->n_live;
  out6[1] = ix->n_tomb;
  out6[2] = (int64_t)ix->cap;
  out6[3] = (int64_t)ix->slot_free.size();
  int herr = 0;
  cudaMemcpy(&herr, ix->err, sizeof(int), cudaMemcpyDeviceToHost);  // synchronous (debug)
  out6[4] = herr;
  int64_t vfree_total = 0;
  for (auto& kv : ix->vfree) vfree_total += kv.second;
  out6[5] = vfree_total;
  return EMM_OK;
}

// host copy of tok_slot for a virtual range (tests)
extern "C" int emm_index_tok_slots_host(emm_index* ix, int64_t v0, int64_t n, int32_t* out) {
  if (!ix || v0 < 0 || v0 + n > ix->v_tokens) return EMM_E_INVALID;
  memcpy(out, ix->tok_slot_host.data() + v0, n * sizeof(int32_t));
  return EMM_OK;
}
