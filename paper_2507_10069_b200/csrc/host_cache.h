// host_cache.h — host control plane of the unified multimodal prefix cache.
//
// A bit-exact C++ restatement of the reference's decision logic:
//   ImagePool    pkg/src/mmsim/cache.py:31-74   (LRU by (last_used, hash))
//   PrefixTree   pkg/src/mmsim/cache.py:105-336 (span-compressed weighted radix,
//                pins, split pin-rewrite, trim, LRU idle-leaf eviction)
//   UnifiedCache pkg/src/mmsim/cache.py:341-406 (budget split + CacheStats)
// Symbols are uint64 keys (injective encoding done by the Python boundary,
// paper_2507_10069_b200/keys.py).  The tree is the authority for every cache
// decision; the device index (dataplane.cu) mirrors it through the journal
// hooks below.
#pragma once
#include <stdint.h>

#include <map>
#include <memory>
#include <list>
#include <set>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "../../include/emm.h"

namespace emm {

struct CacheError {
  int code;
  std::string msg;
};

// Per-symbol data-plane record: the symbol's block hash (prefix hash at its
// position) and the start of its token records in the virtual token space.
struct SymRec {
  uint64_t h0, h1;
  int64_t vstart;  // first virtual token record, -1 when no data plane
  int64_t w;
};

struct Node {
  int64_t id = 0;
  std::vector<uint64_t> span;
  std::vector<int64_t> weights;
  std::vector<SymRec> recs;  // parallel to span when the data plane is attached
  std::unordered_map<uint64_t, Node*> children;
  Node* parent = nullptr;
  int64_t user_count = 0;
  double last_used = 0.0;
  int64_t kv = 0;  // sum(weights)  (cache.py:88-90)
  bool alive = true;  // reachable from the root
  bool in_idle = false;
  std::pair<double, int64_t> idle_key{0.0, 0};
};

struct Handle {
  uint64_t id = 0;
  std::vector<std::pair<Node*, int64_t>> entries;  // [node, covered] (cache.py:93-103)
  Handle* prev = nullptr;  // intrusive live list in _live_handles order (O(1) release)
  Handle* next = nullptr;
};

// Journal consumed by the data plane after every mutating call.
struct TreeHooks {
  virtual ~TreeHooks() {}
  // a new reachable node was created from symbols [pos, pos+len) of the
  // sequence being inserted; the hook fills node->recs.
  virtual void on_new_node(Node* node, const uint64_t* keys, const int64_t* w,
                           int64_t n_total, int64_t pos) = 0;
  // a reachable leaf was evicted; its recs are released by the hook.
  virtual void on_evict(Node* node) = 0;
};

class PrefixTree {
 public:
  explicit PrefixTree(int64_t capacity);
  ~PrefixTree();

  // Symbols match_prefix would read for keys[0, n_avail): n_avail means the walk
  // ran off the end of what is available (more keys could extend the match).
  int64_t match_extent(const uint64_t* keys, int64_t n_avail) const;
  int64_t match_prefix(const uint64_t* keys, const int64_t* w, int64_t n, double now,
                       uint64_t* handle_out);                      // cache.py:121-156
  void release(uint64_t handle);                                   // cache.py:158-167
  int64_t insert_prefix(const uint64_t* keys, const int64_t* w, int64_t n,
                        double now);                               // cache.py:171-217
  int64_t evict(int64_t needed, double now);                       // cache.py:267-284

  // introspection (cache.py:303-336)
  int64_t capacity() const { return capacity_; }
  int64_t total_tokens() const { return total_tokens_; }
  int64_t evictions() const { return evictions_; }
  int64_t increments() const { return increments_; }
  int64_t decrements() const { return decrements_; }
  int64_t live_handle_count() const { return live_count_; }
  const std::vector<std::tuple<int64_t, int64_t, double>>& eviction_log() const {
    return eviction_log_;
  }
  int64_t handle_entry_count(uint64_t handle) const;
  bool handle_live(uint64_t handle) const { return live_.count(handle) != 0; }
  void collect_nodes(std::vector<const Node*>& out) const;  // pre-order, reachable
  const Node* root() const { return root_; }

  // information about the last insert_prefix, for the data plane
  struct InsertInfo {
    int64_t tail_pos = -1;  // first symbol of the stored tail, -1 if none
    int64_t tail_len = 0;   // symbols stored
    int64_t tail_kv = 0;
    int64_t tail_kv_start = 0;  // KV-token offset of the tail in the sequence
    bool ghost = false;         // tail attached to an evicted node (SURVEY App.A H1)
  };
  const InsertInfo& last_insert() const { return last_insert_; }

  void set_hooks(TreeHooks* hooks) { hooks_ = hooks; }

 private:
  Node* new_node();
  void reindex(Node* n);
  void unindex(Node* n);
  void split(Node* node, int64_t at);                       // cache.py:219-244
  bool make_room(int64_t needed, double now);                // cache.py:257-263
  Node* lru_idle_leaf();                                      // cache.py:286-301
  int64_t evict_impl(int64_t needed, double now);
  void flush_graveyard();

  int64_t capacity_;
  int64_t next_id_ = 1;
  Node* root_;
  int64_t total_tokens_ = 0;
  int64_t evictions_ = 0;
  int64_t increments_ = 0, decrements_ = 0;
  std::vector<std::tuple<int64_t, int64_t, double>> eviction_log_;
  std::unordered_map<uint64_t, std::unique_ptr<Handle>> live_;
  Handle* live_head_ = nullptr;  // _live_handles list order, oldest first
  Handle* live_tail_ = nullptr;
  int64_t live_count_ = 0;
  std::vector<std::unique_ptr<Handle>> spare_;  // released handles, reused (no malloc per match)
  std::set<std::pair<std::pair<double, int64_t>, Node*>> idle_;
  std::vector<Node*> graveyard_;
  std::unordered_map<Node*, std::unique_ptr<Node>> owned_;
  TreeHooks* hooks_ = nullptr;
  InsertInfo last_insert_;
};

class ImagePool {
 public:
  explicit ImagePool(int64_t capacity) : capacity_(capacity) {}
  // returns token count or -1 (cache.py:40-46)
  int64_t lookup(const std::string& h, double now);
  bool insert(const std::string& h, int64_t tokens, double now, int64_t bytes);  // :48-61
  int64_t capacity() const { return capacity_; }
  int64_t total_tokens() const { return total_tokens_; }
  int64_t evictions() const { return evictions_; }
  int64_t size() const { return (int64_t)entries_.size(); }
  // hashes evicted since the last call (the data plane drops their slabs)
  std::vector<std::string> take_evicted() {
    std::vector<std::string> out;
    out.swap(evicted_);
    return out;
  }
  bool contains(const std::string& h) const { return entries_.count(h) != 0; }

 private:
  struct Entry {
    int64_t tokens;
    double last_used;
    int64_t bytes;
  };
  int64_t evict(int64_t needed);  // :63-71
  void touch(const std::string& h, Entry& e, double now);
  int64_t capacity_;
  int64_t total_tokens_ = 0;
  int64_t evictions_ = 0;
  std::unordered_map<std::string, Entry> entries_;
  std::set<std::pair<double, std::string>> lru_;
  std::vector<std::string> evicted_;
};

struct CacheStats {  // cache.py:341-360
  int64_t image_hits = 0, image_misses = 0, image_tokens_saved = 0;
  int64_t prefix_lookups = 0, prefix_hits = 0, prefix_tokens_saved = 0;
};

class UnifiedCache {  // cache.py:363-406
 public:
  UnifiedCache(int64_t budget_tokens, double image_fraction);
  ImagePool images;
  PrefixTree prefixes;
  CacheStats stats;
};

}  // namespace emm
