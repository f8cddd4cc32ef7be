// abi_host.cpp — extern "C" entry points of the host control plane
// (include/emm.h, section "Host control plane").
#include <string.h>
#include <unordered_map>

#include <exception>
#include <string>

#include "../../include/emm.h"
#include "emm_hash.h"
#include "host_cache.h"
#include "abi_util.h"

struct emm_pool {
  emm::ImagePool pool;
  explicit emm_pool(int64_t c) : pool(c) {}
};
struct emm_tree {
  emm::PrefixTree tree;
  explicit emm_tree(int64_t c) : tree(c) {}
};
// UnifiedCache façade; `images`/`prefixes` views alias the embedded objects.
struct emm_cache {
  emm::UnifiedCache uc;
  emm_pool* images_view;  // non-owning wrappers pointing into uc
  emm_tree* prefixes_view;
  struct emm_index* index = nullptr;
  emm_cache(int64_t b, double f) : uc(b, f) {
    images_view = reinterpret_cast<emm_pool*>(&uc.images);
    prefixes_view = reinterpret_cast<emm_tree*>(&uc.prefixes);
  }
};
static_assert(sizeof(emm_pool) == sizeof(emm::ImagePool), "view aliasing");
static_assert(sizeof(emm_tree) == sizeof(emm::PrefixTree), "view aliasing");

namespace emm_abi {
thread_local std::string g_err;
void set_error(const std::string& s) { g_err = s; }
}  // namespace emm_abi

extern "C" const char* emm_last_error(void) { return emm_abi::g_err.c_str(); }
extern "C" int emm_version(void) { return 1; }

#define CHECK_ARG(cond, msg)                  \
  do {                                        \
    if (!(cond)) {                            \
      emm_abi::set_error(msg);                \
      return EMM_E_INVALID;                   \
    }                                         \
  } while (0)

// ------------------------------------------------------------------ ImagePool
extern "C" int emm_pool_create(int64_t capacity_tokens, emm_pool** out) {
  CHECK_ARG(out, "null out");
  EMM_GUARD({ *out = new emm_pool(capacity_tokens); });
}
static std::unordered_map<emm_pool*, std::string>& staged_map();
extern "C" int emm_pool_destroy(emm_pool* p) {
  staged_map().erase(p);
  delete p;
  return EMM_OK;
}
extern "C" int emm_pool_lookup(emm_pool* p, const char* h, double now, int64_t* out) {
  CHECK_ARG(p && h && out, "null argument");
  EMM_GUARD({ *out = p->pool.lookup(std::string(h), now); });
}
extern "C" int emm_pool_insert(emm_pool* p, const char* h, int64_t tokens, double now,
                               int64_t bytes, int32_t* ok) {
  CHECK_ARG(p && h && ok, "null argument");
  EMM_GUARD({ *ok = p->pool.insert(std::string(h), tokens, now, bytes) ? 1 : 0; });
}
extern "C" int emm_pool_info(emm_pool* p, int64_t out4[4]) {
  CHECK_ARG(p && out4, "null argument");
  out4[0] = p->pool.total_tokens();
  out4[1] = p->pool.evictions();
  out4[2] = p->pool.capacity();
  out4[3] = p->pool.size();
  return EMM_OK;
}

// evicted hashes staged per pool until the caller's buffer is large enough
#include <unordered_map>
static std::unordered_map<emm_pool*, std::string> g_staged;
static std::unordered_map<emm_pool*, std::string>& staged_map() { return g_staged; }

extern "C" int emm_pool_take_evicted(emm_pool* p, char* buf, int64_t cap, int64_t* needed) {
  CHECK_ARG(p && needed, "null argument");
  std::string& st = g_staged[p];
  for (auto& s : p->pool.take_evicted()) {
    st += s;
    st += '\n';
  }
  *needed = (int64_t)st.size();
  if (buf && cap >= (int64_t)st.size()) {
    memcpy(buf, st.data(), st.size());
    st.clear();
  }
  return EMM_OK;
}

// ----------------------------------------------------------------- PrefixTree
extern "C" int emm_tree_create(int64_t capacity_tokens, emm_tree** out) {
  CHECK_ARG(out, "null out");
  EMM_GUARD({ *out = new emm_tree(capacity_tokens); });
}
extern "C" int emm_tree_destroy(emm_tree* t) {
  delete t;
  return EMM_OK;
}
extern "C" int emm_tree_match(emm_tree* t, const uint64_t* keys, const int64_t* w, int64_t n,
                              double now, int64_t* matched, uint64_t* handle) {
  CHECK_ARG(t && matched && handle && (n == 0 || (keys && w)), "null argument");
  EMM_GUARD({ *matched = t->tree.match_prefix(keys, w, n, now, handle); });
}
extern "C" int emm_tree_release(emm_tree* t, uint64_t handle) {
  CHECK_ARG(t, "null tree");
  EMM_GUARD({ t->tree.release(handle); });
}
extern "C" int emm_tree_insert(emm_tree* t, const uint64_t* keys, const int64_t* w, int64_t n,
                               double now, int64_t* added) {
  CHECK_ARG(t && added && (n == 0 || (keys && w)), "null argument");
  EMM_GUARD({ *added = t->tree.insert_prefix(keys, w, n, now); });
}
extern "C" int emm_tree_evict(emm_tree* t, int64_t needed, double now, int64_t* freed) {
  CHECK_ARG(t && freed, "null argument");
  EMM_GUARD({ *freed = t->tree.evict(needed, now); });
}
extern "C" int emm_tree_info(emm_tree* t, int64_t out8[8]) {
  CHECK_ARG(t && out8, "null argument");
  out8[0] = t->tree.capacity();
  out8[1] = t->tree.total_tokens();
  out8[2] = t->tree.evictions();
  out8[3] = t->tree.increments();
  out8[4] = t->tree.decrements();
  out8[5] = t->tree.live_handle_count();
  out8[6] = (int64_t)t->tree.eviction_log().size();
  std::vector<const emm::Node*> nodes;
  t->tree.collect_nodes(nodes);
  out8[7] = (int64_t)nodes.size();
  return EMM_OK;
}
extern "C" int emm_tree_eviction_log(emm_tree* t, int64_t i0, int64_t n, int64_t* ids,
                                     int64_t* kvs, double* lu) {
  CHECK_ARG(t && ids && kvs && lu, "null argument");
  const auto& log = t->tree.eviction_log();
  CHECK_ARG(i0 >= 0 && i0 + n <= (int64_t)log.size(), "eviction_log range");
  for (int64_t i = 0; i < n; ++i) {
    ids[i] = std::get<0>(log[i0 + i]);
    kvs[i] = std::get<1>(log[i0 + i]);
    lu[i] = std::get<2>(log[i0 + i]);
  }
  return EMM_OK;
}
extern "C" int emm_tree_nodes(emm_tree* t, int64_t max_nodes, int64_t max_syms,
                              int64_t* n_nodes, int64_t* n_syms, int64_t* ids,
                              int64_t* parents, int64_t* kvs, int64_t* ucs, double* lu,
                              int64_t* span_off, uint64_t* span_keys, int64_t* span_w) {
  CHECK_ARG(t && n_nodes && n_syms, "null argument");
  std::vector<const emm::Node*> nodes;
  t->tree.collect_nodes(nodes);
  int64_t syms = 0;
  for (auto* nd : nodes) syms += (int64_t)nd->span.size();
  *n_nodes = (int64_t)nodes.size();
  *n_syms = syms;
  if (!ids || !span_off || (int64_t)nodes.size() > max_nodes || syms > max_syms)
    return EMM_OK;  // size query
  int64_t off = 0;
  for (size_t i = 0; i < nodes.size(); ++i) {
    const emm::Node* nd = nodes[i];
    ids[i] = nd->id;
    parents[i] = nd->parent ? nd->parent->id : -1;
    kvs[i] = nd->kv;
    ucs[i] = nd->user_count;
    lu[i] = nd->last_used;
    span_off[i] = off;
    for (size_t j = 0; j < nd->span.size(); ++j) {
      span_keys[off + j] = nd->span[j];
      span_w[off + j] = nd->weights[j];
    }
    off += (int64_t)nd->span.size();
  }
  span_off[nodes.size()] = off;
  return EMM_OK;
}
extern "C" int emm_tree_handle_entries(emm_tree* t, uint64_t handle, int64_t* n) {
  CHECK_ARG(t && n, "null argument");
  *n = t->tree.handle_entry_count(handle);
  return EMM_OK;
}

// --------------------------------------------------------------- UnifiedCache
extern "C" int emm_cache_create(int64_t budget, double fraction, emm_cache** out) {
  CHECK_ARG(out, "null out");
  EMM_GUARD({ *out = new emm_cache(budget, fraction); });
}
extern "C" int emm_index_detach_(emm_index* ix);
extern "C" int emm_index_flush(emm_index* ix, void* stream);

extern "C" int emm_cache_set_index_(emm_cache* c, emm_index* ix) {
  c->index = ix;
  return EMM_OK;
}

extern "C" int emm_cache_destroy(emm_cache* c) {
  if (c && c->index) {
    emm_index_detach_(c->index);
    c->index = nullptr;
  }
  if (c) g_staged.erase(c->images_view);
  delete c;
  return EMM_OK;
}
extern "C" int emm_cache_parts(emm_cache* c, emm_pool** images, emm_tree** prefixes) {
  CHECK_ARG(c, "null cache");
  if (images) *images = c->images_view;
  if (prefixes) *prefixes = c->prefixes_view;
  return EMM_OK;
}
extern "C" int emm_cache_image_lookup(emm_cache* c, const char* h, double now, int64_t* out) {
  CHECK_ARG(c && h && out, "null argument");
  EMM_GUARD({
    int64_t found = c->uc.images.lookup(std::string(h), now);  // cache.py:372-379
    if (found < 0) {
      c->uc.stats.image_misses += 1;
    } else {
      c->uc.stats.image_hits += 1;
      c->uc.stats.image_tokens_saved += found;
    }
    *out = found;
  });
}
extern "C" int emm_cache_image_insert(emm_cache* c, const char* h, int64_t tokens, double now,
                                      int64_t bytes, int32_t* ok) {
  CHECK_ARG(c && h && ok, "null argument");
  EMM_GUARD({ *ok = c->uc.images.insert(std::string(h), tokens, now, bytes) ? 1 : 0; });
}
extern "C" int emm_cache_match_prefix(emm_cache* c, const uint64_t* keys, const int64_t* w,
                                      int64_t n, double now, int64_t* matched,
                                      uint64_t* handle) {
  CHECK_ARG(c && matched && handle && (n == 0 || (keys && w)), "null argument");
  EMM_GUARD({
    int64_t m = c->uc.prefixes.match_prefix(keys, w, n, now, handle);  // cache.py:385-392
    c->uc.stats.prefix_lookups += 1;
    if (m > 0) {
      c->uc.stats.prefix_hits += 1;
      c->uc.stats.prefix_tokens_saved += m;
    }
    *matched = m;
  });
}
extern "C" int emm_cache_match_prefix_lazy(emm_cache* c, const uint64_t* keys, int64_t n_avail,
                                           int64_t n_total, double now, int64_t* matched,
                                           uint64_t* handle, int32_t* need_more) {
  CHECK_ARG(c && matched && handle && need_more && (n_avail == 0 || keys) &&
                n_avail <= n_total,
            "bad argument");
  EMM_GUARD({
    *need_more = 0;
    if (n_avail < n_total && c->uc.prefixes.match_extent(keys, n_avail) == n_avail) {
      *need_more = 1;
      *matched = 0;
      *handle = 0;
    } else {
      int64_t m = c->uc.prefixes.match_prefix(keys, nullptr, n_avail, now, handle);
      c->uc.stats.prefix_lookups += 1;  // cache.py:385-392
      if (m > 0) {
        c->uc.stats.prefix_hits += 1;
        c->uc.stats.prefix_tokens_saved += m;
      }
      *matched = m;
    }
  });
}
extern "C" int emm_cache_insert_prefix(emm_cache* c, const uint64_t* keys, const int64_t* w,
                                       int64_t n, double now, int64_t* added) {
  CHECK_ARG(c && added && (n == 0 || (keys && w)), "null argument");
  // device updates are journaled by the index hooks and flushed, coalesced,
  // before the next device match / KV-source change / explicit flush
  EMM_GUARD({ *added = c->uc.prefixes.insert_prefix(keys, w, n, now); });
}
extern "C" int emm_cache_release(emm_cache* c, uint64_t handle) {
  CHECK_ARG(c, "null cache");
  EMM_GUARD({ c->uc.prefixes.release(handle); });
}
extern "C" int emm_cache_stats(emm_cache* c, int64_t out9[9]) {
  CHECK_ARG(c && out9, "null argument");
  const auto& s = c->uc.stats;
  out9[0] = s.image_hits;
  out9[1] = s.image_misses;
  out9[2] = s.image_tokens_saved;
  out9[3] = s.prefix_lookups;
  out9[4] = s.prefix_hits;
  out9[5] = s.prefix_tokens_saved;
  out9[6] = c->uc.images.evictions() + c->uc.prefixes.evictions();  // cache.py:403
  out9[7] = c->uc.images.total_tokens();
  out9[8] = c->uc.prefixes.total_tokens();
  return EMM_OK;
}

extern "C" int emm_prefix_hashes_host(const uint64_t* keys, const int64_t* w, int64_t n,
                                      uint64_t* h0, uint64_t* h1) {
  CHECK_ARG(n == 0 || (keys && w && h0 && h1), "null argument");
  uint64_t a = EMM_H0, b = EMM_H1;
  for (int64_t i = 0; i < n; ++i) {
    a = emm_addmod61(emm_mulmod61(a, EMM_B0), emm_sym_term(keys[i], (uint64_t)w[i], 0));
    b = emm_addmod61(emm_mulmod61(b, EMM_B1), emm_sym_term(keys[i], (uint64_t)w[i], 1));
    h0[i] = a;
    h1[i] = b;
  }
  return EMM_OK;
}
