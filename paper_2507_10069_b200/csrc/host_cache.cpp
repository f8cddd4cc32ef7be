// host_cache.cpp — see host_cache.h.  Every function cites the reference
// lines it restates; quirks are reproduced on purpose.
#include "host_cache.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>

namespace emm {

static std::atomic<uint64_t> g_next_handle{1};

// ---------------------------------------------------------------- PrefixTree

PrefixTree::PrefixTree(int64_t capacity) : capacity_(capacity) {
  // cache.py:108-117 — root has id 0, ids start at 1
  auto r = std::make_unique<Node>();
  r->id = 0;
  root_ = r.get();
  owned_[root_] = std::move(r);
}

PrefixTree::~PrefixTree() {}

Node* PrefixTree::new_node() {
  auto n = std::make_unique<Node>();
  Node* p = n.get();
  owned_[p] = std::move(n);
  return p;
}

void PrefixTree::unindex(Node* n) {
  if (n->in_idle) {
    idle_.erase({n->idle_key, n});
    n->in_idle = false;
  }
}

// An evictable candidate is a reachable, unpinned leaf (cache.py:286-301).
void PrefixTree::reindex(Node* n) {
  unindex(n);
  if (n != root_ && n->alive && n->children.empty() && n->user_count <= 0) {
    n->idle_key = {n->last_used, n->id};
    idle_.insert({n->idle_key, n});
    n->in_idle = true;
  }
}

// length of the common prefix of a[0..lim) and b[0..lim): the edge compare of
// the reference walk (cache.py:135-140, 204-206) over raw keys; memcmp settles
// the common full-edge case with vector loads, the scan only runs on a mismatch
static inline int64_t common_prefix(const uint64_t* a, const uint64_t* b, int64_t lim) {
  if (lim <= 0) return 0;
  if (std::memcmp(a, b, (size_t)lim * sizeof(uint64_t)) == 0) return lim;
  int64_t i = 0;
  while (a[i] == b[i]) ++i;
  return i;
}

int64_t PrefixTree::match_extent(const uint64_t* keys, int64_t n_avail) const {
  // the read-only walk of match_prefix below; returns the index of the first
  // key that decides the match (a mismatch), or n_avail if none does yet
  const Node* node = root_;
  int64_t pos = 0;
  while (pos < n_avail) {
    auto it = node->children.find(keys[pos]);
    if (it == node->children.end()) return pos;
    const Node* child = it->second;
    const int64_t slen = (int64_t)child->span.size();
    const int64_t common =
        common_prefix(child->span.data(), keys + pos, std::min(slen, n_avail - pos));
    if (pos + common == n_avail) return n_avail;
    if (common < slen) return pos + common;
    pos += common;
    node = child;
  }
  return n_avail;
}

int64_t PrefixTree::match_prefix(const uint64_t* keys, const int64_t* w, int64_t n,
                                 double now, uint64_t* handle_out) {
  (void)w;  // matched weight comes from the stored span (cache.py:145)
  int64_t matched_kv = 0;
  std::unique_ptr<Handle> h;
  if (spare_.empty()) {
    h = std::make_unique<Handle>();
  } else {
    h = std::move(spare_.back());
    spare_.pop_back();
    h->entries.clear();
  }
  Node* node = root_;
  int64_t pos = 0;
  while (pos < n) {
    auto it = node->children.find(keys[pos]);
    if (it == node->children.end()) break;
    Node* child = it->second;
    const int64_t slen = (int64_t)child->span.size();
    const int64_t common = common_prefix(child->span.data(), keys + pos, std::min(slen, n - pos));
    if (common == 0) break;
    if (common == slen) {
      matched_kv += child->kv;  // kv == sum(weights) (cache.py:88-90)
    } else {
      for (int64_t i = 0; i < common; ++i) matched_kv += child->weights[i];
    }
    child->user_count += 1;
    child->last_used = now;
    increments_ += 1;
    reindex(child);
    h->entries.push_back({child, common});
    if (common < slen) break;
    pos += common;
    node = child;
  }
  h->id = g_next_handle.fetch_add(1);
  *handle_out = h->id;
  h->prev = live_tail_;
  h->next = nullptr;
  (live_tail_ ? live_tail_->next : live_head_) = h.get();
  live_tail_ = h.get();
  live_count_ += 1;
  live_.emplace(h->id, std::move(h));
  return matched_kv;
}

void PrefixTree::release(uint64_t handle) {
  auto it = live_.find(handle);
  if (it == live_.end())  // cache.py:159-160
    throw CacheError{EMM_E_RELEASE_WITHOUT_MATCH, "handle already released or unknown"};
  Handle* h = it->second.get();
  for (auto& e : h->entries) {
    Node* node = e.first;
    if (node->user_count <= 0)  // cache.py:162-163
      throw CacheError{EMM_E_RELEASE_WITHOUT_MATCH, "user_count underflow"};
    node->user_count -= 1;
    decrements_ += 1;
    reindex(node);
  }
  (h->prev ? h->prev->next : live_head_) = h->next;
  (h->next ? h->next->prev : live_tail_) = h->prev;
  live_count_ -= 1;
  if (spare_.size() < 1024) spare_.push_back(std::move(it->second));
  live_.erase(it);
}

int64_t PrefixTree::handle_entry_count(uint64_t handle) const {
  auto it = live_.find(handle);
  return it == live_.end() ? -1 : (int64_t)it->second->entries.size();
}

int64_t PrefixTree::insert_prefix(const uint64_t* keys, const int64_t* w, int64_t n,
                                  double now) {
  last_insert_ = InsertInfo();
  Node* node = root_;
  int64_t pos = 0, added = 0, kv_pos = 0;
  int64_t result = 0;
  bool done = false;
  while (pos < n && !done) {
    auto it = node->children.find(keys[pos]);
    if (it == node->children.end()) {
      // new tail (cache.py:187-202)
      int64_t keep = n - pos;
      int64_t kv = 0;
      for (int64_t i = pos; i < n; ++i) kv += w[i];
      if (!make_room(kv, now)) {
        // _trim_to_budget (cache.py:246-255): whole symbols that fit
        const int64_t free_tok = capacity_ - total_tokens_;
        keep = 0;
        kv = 0;
        for (int64_t i = pos; i < n; ++i) {
          if (kv + w[i] > free_tok) break;
          kv += w[i];
          ++keep;
        }
        if (keep == 0) {
          result = added;
          done = true;
          break;
        }
      }
      Node* nn = new_node();
      nn->id = next_id_++;
      nn->span.assign(keys + pos, keys + pos + keep);
      nn->weights.assign(w + pos, w + pos + keep);
      nn->kv = kv;
      nn->last_used = now;
      nn->parent = node;
      nn->alive = node->alive;
      node->children[nn->span[0]] = nn;
      total_tokens_ += kv;
      added += kv;
      last_insert_.tail_pos = pos;
      last_insert_.tail_len = keep;
      last_insert_.tail_kv = kv;
      last_insert_.tail_kv_start = kv_pos;
      last_insert_.ghost = !nn->alive;
      if (nn->alive) {
        reindex(node);
        reindex(nn);
        if (hooks_) hooks_->on_new_node(nn, keys, w, n, pos);
      } else {
        graveyard_.push_back(nn);  // unreachable ghost: counted, never served
      }
      result = added;
      done = true;
      break;
    }
    Node* child = it->second;
    const int64_t slen = (int64_t)child->span.size();
    const int64_t common = common_prefix(child->span.data(), keys + pos, std::min(slen, n - pos));
    child->last_used = now;  // cache.py:207
    reindex(child);
    for (int64_t i = 0; i < common; ++i) kv_pos += w[pos + i];
    if (common == slen) {
      pos += common;
      node = child;
      continue;
    }
    split(child, common);  // cache.py:212-216
    child->last_used = now;
    reindex(child);
    pos += common;
    node = child;
  }
  if (!done) result = added;
  flush_graveyard();
  return result;
}

// Free evicted and ghost nodes.  No live handle can reference them (an
// evicted leaf had user_count == 0; a ghost is unreachable).
void PrefixTree::flush_graveyard() {
  std::vector<Node*> doomed;
  for (Node* g : graveyard_) {
    doomed.push_back(g);
    for (auto& kvp : g->children) doomed.push_back(kvp.second);
  }
  graveyard_.clear();
  for (Node* d : doomed) owned_.erase(d);
}

void PrefixTree::split(Node* node, int64_t at) {
  Node* bottom = new_node();
  bottom->id = next_id_++;
  bottom->span.assign(node->span.begin() + at, node->span.end());
  bottom->weights.assign(node->weights.begin() + at, node->weights.end());
  if (!node->recs.empty()) {
    bottom->recs.assign(node->recs.begin() + at, node->recs.end());
    node->recs.resize(at);
  }
  bottom->children.swap(node->children);
  for (auto& kvp : bottom->children) kvp.second->parent = bottom;
  bottom->user_count = node->user_count;
  bottom->last_used = node->last_used;
  bottom->parent = node;
  bottom->alive = node->alive;
  node->children[bottom->span[0]] = bottom;
  node->span.resize(at);
  node->weights.resize(at);
  int64_t kv_top = 0;
  for (int64_t x : node->weights) kv_top += x;
  bottom->kv = node->kv - kv_top;
  node->kv = kv_top;
  // rewrite outstanding pins that extend past the top half (cache.py:229-237)
  for (Handle* h = live_head_; h; h = h->next) {
    const size_t ne = h->entries.size();
    for (size_t i = 0; i < ne; ++i) {
      if (h->entries[i].first == node && h->entries[i].second > at) {
        int64_t extra = h->entries[i].second - at;
        h->entries[i].second = at;
        h->entries.push_back({bottom, extra});
        increments_ += 1;
        break;
      }
    }
  }
  // recompute pins from the live handles (cache.py:238-244)
  int64_t pb = 0, pt = 0;
  for (const Handle* h = live_head_; h; h = h->next) {
    for (auto& e : h->entries) {
      if (e.first == bottom) ++pb;
      if (e.first == node) ++pt;
    }
  }
  bottom->user_count = pb;
  node->user_count = pt;
  reindex(bottom);
  reindex(node);
}

bool PrefixTree::make_room(int64_t needed, double now) {  // cache.py:257-263
  if (needed > capacity_) return false;
  int64_t shortfall = needed - (capacity_ - total_tokens_);
  if (shortfall > 0) evict_impl(shortfall, now);
  return needed <= capacity_ - total_tokens_;
}

Node* PrefixTree::lru_idle_leaf() {
  if (idle_.empty()) return nullptr;
  return idle_.begin()->second;  // min (last_used, node_id)  (cache.py:296)
}

int64_t PrefixTree::evict(int64_t needed, double now) {
  int64_t freed = evict_impl(needed, now);
  flush_graveyard();
  return freed;
}

int64_t PrefixTree::evict_impl(int64_t needed, double now) {  // cache.py:267-284
  (void)now;
  int64_t freed = 0;
  while (freed < needed) {
    Node* leaf = lru_idle_leaf();
    if (!leaf) break;
    Node* parent = leaf->parent;
    parent->children.erase(leaf->span[0]);
    total_tokens_ -= leaf->kv;
    freed += leaf->kv;
    evictions_ += 1;
    eviction_log_.emplace_back(leaf->id, leaf->kv, leaf->last_used);
    leaf->alive = false;
    unindex(leaf);
    reindex(parent);
    if (hooks_) hooks_->on_evict(leaf);
    graveyard_.push_back(leaf);
  }
  return freed;
}

void PrefixTree::collect_nodes(std::vector<const Node*>& out) const {
  std::vector<const Node*> stack;
  for (auto& kv : root_->children) stack.push_back(kv.second);
  while (!stack.empty()) {
    const Node* n = stack.back();
    stack.pop_back();
    out.push_back(n);
    for (auto& kv : n->children) stack.push_back(kv.second);
  }
}

// ----------------------------------------------------------------- ImagePool

void ImagePool::touch(const std::string& h, Entry& e, double now) {
  lru_.erase({e.last_used, h});
  e.last_used = now;
  lru_.insert({e.last_used, h});
}

int64_t ImagePool::lookup(const std::string& h, double now) {  // cache.py:40-46
  auto it = entries_.find(h);
  if (it == entries_.end()) return -1;
  touch(h, it->second, now);
  return it->second.tokens;
}

bool ImagePool::insert(const std::string& h, int64_t tokens, double now, int64_t bytes) {
  auto it = entries_.find(h);  // cache.py:51-53
  if (it != entries_.end()) {
    touch(h, it->second, now);
    return true;
  }
  if (tokens > capacity_) return false;  // :54-55
  evict(tokens - (capacity_ - total_tokens_));  // :56
  if (tokens > capacity_ - total_tokens_) return false;  // :57-58
  entries_[h] = Entry{tokens, now, bytes};
  lru_.insert({now, h});
  total_tokens_ += tokens;
  return true;
}

int64_t ImagePool::evict(int64_t needed) {  // cache.py:63-71, key (last_used, hash)
  int64_t freed = 0;
  while (freed < needed && !entries_.empty()) {
    auto victim = *lru_.begin();
    lru_.erase(lru_.begin());
    auto it = entries_.find(victim.second);
    freed += it->second.tokens;
    total_tokens_ -= it->second.tokens;
    evicted_.push_back(victim.second);
    entries_.erase(it);
    evictions_ += 1;
  }
  return freed;
}

// -------------------------------------------------------------- UnifiedCache

static int64_t image_budget_of(int64_t budget, double fraction) {
  return (int64_t)((double)budget * fraction);  // int(budget * fraction), cache.py:367
}

UnifiedCache::UnifiedCache(int64_t budget_tokens, double image_fraction)
    : images(image_budget_of(budget_tokens, image_fraction)),
      prefixes(budget_tokens - image_budget_of(budget_tokens, image_fraction)) {}

}  // namespace emm
