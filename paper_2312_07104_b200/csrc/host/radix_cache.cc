// Host radix tree + token-slot pool behind the rx_cache_* / rx_match_prefix /
// rx_insert / rx_inc_ref / rx_dec_ref / rx_evict / rx_alloc calls (include/rx.h).
//
// PAPER.md §3: the tree maps token sequences to KV slots "in a
// non-contiguous, paged layout, where the size of each page is equivalent to
// one token"; LRU leaf-first eviction; per-node reference counters; cache and
// running requests share one pool; the tree lives on the CPU.  Alg. 1
// names the operations.  Readings R1-R10 fix every
// tie-break so the result is deterministic.
//
// Data layout choices (host performance; the tree is on the scheduling path):
//  * free slots: two-level bitmap (bit per slot + bit per 64-slot word) with a
//    low-water hint, so alloc(n) of the n smallest free slots costs
//    O(n + words skipped) and free(k) O(k);
//  * nodes: token/slot runs in std::vector<int32_t>, children in a hash map
//    keyed by first token, id -> node map for handles;
//  * evictable / cached token counts maintained incrementally, and so is the set of eviction
//    candidates (non-root childless nodes with ref 0, ordered by (last_access, id), R2): every
//    stamp, ref change, insert and eviction updates it, so evict(k) costs O(evicted leaves x log)
//    instead of a walk over the whole tree.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <new>
#include <queue>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../../include/rx.h"

namespace {

struct Node {
  int64_t id;
  std::vector<int32_t> tokens;
  std::vector<int32_t> slots;
  Node* parent;
  std::unordered_map<int32_t, Node*> children;
  int64_t ref;
  uint64_t last_access;
};

class SlotBitmap {
 public:
  explicit SlotBitmap(int64_t n) : n_(n) {
    words_.assign((n + 63) / 64, 0);
    summary_.assign((words_.size() + 63) / 64, 0);
    lo_ = words_.size();
  }
  int64_t count() const { return count_; }
  bool test(int64_t s) const { return (words_[s >> 6] >> (s & 63)) & 1; }
  void set(int64_t s) {  // mark free
    size_t w = s >> 6;
    if (!words_[w]) summary_[w >> 6] |= 1ull << (w & 63);
    words_[w] |= 1ull << (s & 63);
    if (w < lo_) lo_ = w;
    ++count_;
  }
  // Pop the n smallest free slots (caller checked count() >= n).
  void take_smallest(int64_t n, int32_t* out) {
    size_t w = lo_;
    int64_t got = 0;
    while (got < n) {
      // skip empty words via the summary
      while (!words_[w]) {
        size_t sw = w >> 6;
        uint64_t m = summary_[sw] & (~0ull << (w & 63));
        while (!m) m = summary_[++sw];
        w = (sw << 6) + __builtin_ctzll(m);
      }
      uint64_t bits = words_[w];
      while (bits && got < n) {
        int b = __builtin_ctzll(bits);
        out[got++] = static_cast<int32_t>((w << 6) + b);
        bits &= bits - 1;
      }
      words_[w] = bits;
      if (!bits) {
        summary_[w >> 6] &= ~(1ull << (w & 63));
        ++w;
      }
    }
    count_ -= n;
    lo_ = w < words_.size() ? w : words_.size();
  }

 private:
  int64_t n_;
  std::vector<uint64_t> words_, summary_;
  size_t lo_;
  int64_t count_ = 0;
};

}  // namespace

struct rx_cache {
  int64_t num_slots;
  SlotBitmap free_slots;
  Node root;
  int64_t next_id = 1;
  uint64_t clock = 0;
  int64_t evictable = 0;
  int64_t cached = 0;
  std::unordered_map<int64_t, Node*> by_id;
  using CandKey = std::pair<std::pair<uint64_t, int64_t>, Node*>;
  std::set<CandKey> cands;                 // eviction candidates, smallest (last_access, id) first

  static CandKey key(Node* n) { return {{n->last_access, n->id}, n}; }
  bool candidate(const Node* n) const { return n != &root && n->children.empty() && n->ref == 0; }
  // every change of a node's stamp / ref / children goes through these two
  void before_change(Node* n) {
    if (candidate(n)) cands.erase(key(n));
  }
  void after_change(Node* n) {
    if (candidate(n)) cands.insert(key(n));
  }
  void stamp(Node* n, uint64_t now) {
    before_change(n);
    n->last_access = now;
    after_change(n);
  }

  explicit rx_cache(int64_t n) : num_slots(n), free_slots(n) {
    for (int64_t s = 1; s < n; ++s) free_slots.set(s);
    root.id = 0;
    root.parent = nullptr;
    root.ref = 0;
    root.last_access = 0;
    by_id[0] = &root;
  }
  ~rx_cache() {
    std::vector<Node*> stack;
    for (auto& kv : root.children) stack.push_back(kv.second);
    while (!stack.empty()) {
      Node* n = stack.back();
      stack.pop_back();
      for (auto& kv : n->children) stack.push_back(kv.second);
      delete n;
    }
  }

  Node* lookup(rx_node h) const {
    auto it = by_id.find(h);
    return it == by_id.end() ? nullptr : it->second;
  }

  // R4: the upper half is a new node (fresh id) that copies ref and stamp;
  // the lower half keeps its id, stamp and children.
  Node* split(Node* child, size_t k) {
    Node* up = new Node();
    up->id = next_id++;
    up->tokens.assign(child->tokens.begin(), child->tokens.begin() + k);
    up->slots.assign(child->slots.begin(), child->slots.begin() + k);
    up->parent = child->parent;
    up->ref = child->ref;
    up->last_access = child->last_access;
    child->parent->children[up->tokens[0]] = up;
    child->tokens.erase(child->tokens.begin(), child->tokens.begin() + k);
    child->slots.erase(child->slots.begin(), child->slots.begin() + k);
    child->parent = up;
    up->children[child->tokens[0]] = child;
    by_id[up->id] = up;
    return up;
  }

  void release(const int32_t* s, int64_t n) {
    for (int64_t i = 0; i < n; ++i) free_slots.set(s[i]);
  }
};

namespace {

// Length of the common prefix: 64-token blocks by memcmp (vectorised by libc; long shared
// prefixes such as an 8 k-token RAG context are walked at memory speed), then token by token.
inline size_t common_len(const int32_t* a, size_t na, const int32_t* b, size_t nb) {
  size_t n = na < nb ? na : nb, k = 0;
  constexpr size_t kBlk = 64;
  while (k + kBlk <= n && std::memcmp(a + k, b + k, kBlk * sizeof(int32_t)) == 0) k += kBlk;
  while (k < n && a[k] == b[k]) ++k;
  return k;
}

void json_ints(std::string& o, const std::vector<int32_t>& v) {
  o += '[';
  char buf[16];
  for (size_t i = 0; i < v.size(); ++i) {
    if (i) o += ',';
    int len = snprintf(buf, sizeof buf, "%d", v[i]);
    o.append(buf, len);
  }
  o += ']';
}

void dump_node(const Node* n, std::string& o) {
  char buf[96];
  snprintf(buf, sizeof buf, "{\"id\":%lld,\"tokens\":", (long long)n->id);
  o += buf;
  json_ints(o, n->tokens);
  o += ",\"slots\":";
  json_ints(o, n->slots);
  snprintf(buf, sizeof buf, ",\"ref\":%lld,\"last_access\":%llu,\"children\":[", (long long)n->ref,
           (unsigned long long)n->last_access);
  o += buf;
  std::vector<int32_t> keys;
  keys.reserve(n->children.size());
  for (auto& kv : n->children) keys.push_back(kv.first);
  std::sort(keys.begin(), keys.end());
  for (size_t i = 0; i < keys.size(); ++i) {
    if (i) o += ',';
    dump_node(n->children.at(keys[i]), o);
  }
  o += "]}";
}

}  // namespace

extern "C" {

rx_status rx_cache_create(int64_t num_slots, rx_cache** out) {
  if (!out || num_slots < 1 || num_slots > (int64_t(1) << 31)) return RX_E_INVALID;
  rx_cache* c = new (std::nothrow) rx_cache(num_slots);
  if (!c) return RX_E_NOMEM;
  *out = c;
  return RX_OK;
}

void rx_cache_destroy(rx_cache* c) { delete c; }

rx_status rx_match_prefix(rx_cache* c, const int32_t* tokens, int64_t n, rx_node* node,
                          int64_t* matched_len, int32_t* slots_out) {
  if (!c || n < 0 || (n > 0 && !tokens) || !node || !matched_len) return RX_E_INVALID;
  uint64_t now = ++c->clock;  // R1
  Node* cur = &c->root;
  int64_t i = 0;
  while (i < n) {
    auto it = cur->children.find(tokens[i]);
    if (it == cur->children.end()) break;
    Node* ch = it->second;
    size_t k = common_len(ch->tokens.data(), ch->tokens.size(), tokens + i, size_t(n - i));
    if (k < ch->tokens.size()) ch = c->split(ch, k);  // R3: eager split
    c->stamp(ch, now);
    if (slots_out) std::memcpy(slots_out + i, ch->slots.data(), k * sizeof(int32_t));
    i += int64_t(k);
    cur = ch;
  }
  *node = cur->id;
  *matched_len = i;
  return RX_OK;
}

rx_status rx_insert(rx_cache* c, const int32_t* tokens, const int32_t* slots, int64_t n,
                    int64_t* new_cached, int64_t* dup_freed) {
  if (!c || n < 0 || (n > 0 && (!tokens || !slots)) || !new_cached) return RX_E_INVALID;
  for (int64_t i = 0; i < n; ++i)
    if (slots[i] < 1 || slots[i] >= c->num_slots) return RX_E_INVALID;
  uint64_t now = ++c->clock;  // R1, R9
  Node* cur = &c->root;
  int64_t i = 0;
  std::vector<int32_t> dup;
  while (i < n) {
    auto it = cur->children.find(tokens[i]);
    if (it == cur->children.end()) break;
    Node* ch = it->second;
    size_t k = common_len(ch->tokens.data(), ch->tokens.size(), tokens + i, size_t(n - i));
    if (k < ch->tokens.size()) ch = c->split(ch, k);
    c->stamp(ch, now);
    if (std::memcmp(slots + i, ch->slots.data(), k * sizeof(int32_t)) != 0)   // R10 (usually equal)
      for (size_t j = 0; j < k; ++j)
        if (slots[i + j] != ch->slots[j]) dup.push_back(slots[i + j]);
    i += int64_t(k);
    cur = ch;
  }
  int64_t added = n - i;
  if (added > 0) {
    Node* leaf = new Node();
    leaf->id = c->next_id++;
    leaf->tokens.assign(tokens + i, tokens + n);
    leaf->slots.assign(slots + i, slots + n);
    leaf->parent = cur;
    leaf->ref = 0;
    leaf->last_access = now;
    c->before_change(cur);                 // cur gains a child: no longer a candidate
    cur->children[tokens[i]] = leaf;
    c->after_change(leaf);
    c->by_id[leaf->id] = leaf;
    c->evictable += added;
    c->cached += added;
  }
  c->release(dup.data(), int64_t(dup.size()));
  *new_cached = added;
  if (dup_freed) *dup_freed = int64_t(dup.size());
  return RX_OK;
}

rx_status rx_inc_ref(rx_cache* c, rx_node h, int64_t* d_evictable) {
  if (!c) return RX_E_INVALID;
  Node* n = c->lookup(h);
  if (!n) return RX_E_STALE;
  int64_t d = 0;
  for (; n != &c->root; n = n->parent) {
    if (n->ref == 0) d -= int64_t(n->tokens.size());
    c->before_change(n);
    ++n->ref;
  }
  c->evictable += d;
  if (d_evictable) *d_evictable = d;
  return RX_OK;
}

rx_status rx_dec_ref(rx_cache* c, rx_node h, int64_t* d_evictable) {
  if (!c) return RX_E_INVALID;
  Node* n = c->lookup(h);
  if (!n) return RX_E_STALE;
  for (Node* m = n; m != &c->root; m = m->parent)
    if (m->ref < 1) return RX_E_UNDERFLOW;
  int64_t d = 0;
  for (; n != &c->root; n = n->parent) {
    if (--n->ref == 0) d += int64_t(n->tokens.size());
    c->after_change(n);
  }
  c->evictable += d;
  if (d_evictable) *d_evictable = d;
  return RX_OK;
}

static rx_status evict_impl(rx_cache* c, int64_t needed, int64_t* evicted, rx_evict_cb cb, rx_evict_path_cb pcb,
                            void* user) {
  if (!c || !evicted) return RX_E_INVALID;
  *evicted = 0;
  if (needed <= 0) return RX_OK;
  int64_t got = 0;
  // candidates: non-root leaves with ref 0, min-ordered by (last_access, id) (R2), kept
  // incrementally in c->cands
  while (got < needed && !c->cands.empty()) {
    Node* n = c->cands.begin()->second;
    c->cands.erase(c->cands.begin());
    Node* p = n->parent;
    p->children.erase(n->tokens[0]);
    int64_t len = int64_t(n->tokens.size());
    c->release(n->slots.data(), len);
    if (cb) cb(user, n->slots.data(), len);
    if (pcb) {
      std::vector<const Node*> chain;                 // root-exclusive path p ... n
      for (const Node* a = p; a != &c->root; a = a->parent) chain.push_back(a);
      std::vector<int32_t> path;
      for (auto it = chain.rbegin(); it != chain.rend(); ++it)
        path.insert(path.end(), (*it)->tokens.begin(), (*it)->tokens.end());
      const int64_t leaf_start = int64_t(path.size());
      path.insert(path.end(), n->tokens.begin(), n->tokens.end());
      pcb(user, path.data(), int64_t(path.size()), leaf_start, n->slots.data(), len);
    }
    got += len;
    c->evictable -= len;
    c->cached -= len;
    c->by_id.erase(n->id);
    delete n;
    c->after_change(p);                    // a parent left childless with ref 0 becomes a candidate
  }
  *evicted = got;
  return RX_OK;
}

rx_status rx_evict(rx_cache* c, int64_t needed, int64_t* evicted, rx_evict_cb cb, void* user) {
  return evict_impl(c, needed, evicted, cb, nullptr, user);
}

rx_status rx_evict_paths(rx_cache* c, int64_t needed, int64_t* evicted, rx_evict_path_cb cb, void* user) {
  return evict_impl(c, needed, evicted, nullptr, cb, user);
}

rx_status rx_alloc(rx_cache* c, int64_t n, int32_t* out) {
  if (!c || n < 0 || (n > 0 && !out)) return RX_E_INVALID;
  if (n > c->free_slots.count()) return RX_E_NOMEM;
  if (n) c->free_slots.take_smallest(n, out);
  return RX_OK;
}

rx_status rx_free(rx_cache* c, const int32_t* slots, int64_t n) {
  if (!c || n < 0 || (n > 0 && !slots)) return RX_E_INVALID;
  for (int64_t i = 0; i < n; ++i) {
    if (slots[i] < 1 || slots[i] >= c->num_slots || c->free_slots.test(slots[i])) return RX_E_INVALID;
    for (int64_t j = 0; j < i; ++j)
      if (slots[j] == slots[i]) return RX_E_INVALID;
  }
  c->release(slots, n);
  return RX_OK;
}

rx_status rx_alloc_evict(rx_cache* c, int64_t n, int32_t* out, int64_t* evicted, rx_evict_cb cb,
                         void* user) {
  if (evicted) *evicted = 0;
  rx_status st = rx_alloc(c, n, out);
  if (st != RX_E_NOMEM) return st;
  int64_t got = 0;
  st = rx_evict(c, n - c->free_slots.count(), &got, cb, user);  // R6: the shortfall
  if (st != RX_OK) return st;
  if (evicted) *evicted = got;
  return rx_alloc(c, n, out);
}

rx_status rx_match_prefix_batch(rx_cache* c, int32_t batch, const int32_t* tokens, const int64_t* offsets,
                                rx_node* nodes, int64_t* matched, int32_t* slots_out) {
  if (!c || batch < 0 || (batch > 0 && (!tokens || !offsets || !nodes || !matched))) return RX_E_INVALID;
  for (int32_t b = 0; b < batch; ++b) {
    const int64_t o = offsets[b], n = offsets[b + 1] - o;
    rx_status st = rx_match_prefix(c, tokens + o, n, nodes + b, matched + b, slots_out ? slots_out + o : nullptr);
    if (st != RX_OK) return st;
  }
  return RX_OK;
}

rx_status rx_inc_ref_batch(rx_cache* c, int32_t batch, const rx_node* nodes, int64_t* deltas) {
  if (!c || batch < 0 || (batch > 0 && !nodes)) return RX_E_INVALID;
  for (int32_t b = 0; b < batch; ++b) {
    int64_t d = 0;
    rx_status st = rx_inc_ref(c, nodes[b], &d);
    if (st != RX_OK) return st;
    if (deltas) deltas[b] = d;
  }
  return RX_OK;
}

rx_status rx_finish_batch(rx_cache* c, int32_t batch, const rx_node* nodes, const int32_t* tokens,
                          const int64_t* offsets, const int32_t* slots, int64_t* d_evict, int64_t* new_cached,
                          int64_t* dup_freed) {
  if (!c || batch < 0 || (batch > 0 && (!nodes || !tokens || !offsets || !slots))) return RX_E_INVALID;
  for (int32_t b = 0; b < batch; ++b) {
    int64_t d = 0, nc = 0, nd = 0;
    rx_status st = rx_dec_ref(c, nodes[b], &d);
    if (st != RX_OK) return st;
    const int64_t o = offsets[b];
    st = rx_insert(c, tokens + o, slots + o, offsets[b + 1] - o, &nc, &nd);
    if (st != RX_OK) return st;
    if (d_evict) d_evict[b] = d;
    if (new_cached) new_cached[b] = nc;
    if (dup_freed) dup_freed[b] = nd;
  }
  return RX_OK;
}

int64_t rx_evictable_size(const rx_cache* c) { return c ? c->evictable : -1; }
int64_t rx_total_cached(const rx_cache* c) { return c ? c->cached : -1; }
int64_t rx_available(const rx_cache* c) { return c ? c->free_slots.count() : -1; }
int64_t rx_num_slots(const rx_cache* c) { return c ? c->num_slots : -1; }
int64_t rx_clock(const rx_cache* c) { return c ? int64_t(c->clock) : -1; }

int64_t rx_dump_json(const rx_cache* c, char* buf, int64_t cap) {
  if (!c) return -1;
  std::string o;
  dump_node(&c->root, o);
  if (buf && cap > 0) {
    int64_t m = std::min<int64_t>(cap - 1, int64_t(o.size()));
    std::memcpy(buf, o.data(), size_t(m));
    buf[m] = 0;
  }
  return int64_t(o.size());
}

}  // extern "C"
