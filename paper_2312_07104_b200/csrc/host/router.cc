// Data-parallel RadixAttention router (rx_router_*, include/rx.h) — SURVEY §8(f)
// NEXT-3, App. A.4: "each worker maintains its own
// sub-tree, while the router oversees a meta-tree ... a trie that tracks all
// sub-trees and their associated devices"; dispatch by "each request's
// affinity—measured by the length of the shared prefix with specific workers
// and other requests in the same group"; "should an eviction occur at a worker
// node, it commits this eviction to a queue, which the router then processes to
// update the meta-tree during periods of low activity" (weakly consistent).
//
// Meta-tree: a compressed trie over token sequences whose nodes carry a bitmask
// of the workers believed to cache that edge (<= 64 workers).  Readings
// (R24): affinity[w] = tokens matched along the path while w is in
// every node's mask from the root; score = affinity - load_weight * load;
// argmax score, ties -> least load -> smallest worker id; the chosen worker is
// credited with the request's prompt at once (group affinity within a batch);
// load[w] grows by the request's uncached prompt tokens.
#include <algorithm>
#include <cstdint>
#include <deque>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../../include/rx.h"

namespace {

struct MNode {
  std::vector<int32_t> tokens;
  uint64_t mask = 0;
  std::vector<uint64_t> stamp;   // per worker: router clock of its latest insert over this edge
  MNode* parent = nullptr;
  std::unordered_map<int32_t, MNode*> children;
};

struct EvictRec {
  int32_t worker;
  std::vector<int32_t> path;
  int64_t leaf_start;
  uint64_t stamp;                // router clock when the eviction was queued
};

size_t common(const int32_t* a, size_t na, const int32_t* b, size_t nb) {
  size_t n = na < nb ? na : nb, k = 0;
  while (k < n && a[k] == b[k]) ++k;
  return k;
}

}  // namespace

struct rx_router {
  int32_t workers;
  MNode root;
  std::deque<EvictRec> queue;
  uint64_t clock = 0;

  ~rx_router() {
    std::vector<MNode*> st;
    for (auto& kv : root.children) st.push_back(kv.second);
    while (!st.empty()) {
      MNode* n = st.back();
      st.pop_back();
      for (auto& kv : n->children) st.push_back(kv.second);
      delete n;
    }
  }

  MNode* split(MNode* ch, size_t k) {
    MNode* up = new MNode();
    up->tokens.assign(ch->tokens.begin(), ch->tokens.begin() + k);
    up->mask = ch->mask;
    up->stamp = ch->stamp;
    up->parent = ch->parent;
    ch->parent->children[up->tokens[0]] = up;
    ch->tokens.erase(ch->tokens.begin(), ch->tokens.begin() + k);
    ch->parent = up;
    up->children[ch->tokens[0]] = ch;
    return up;
  }

  // worker w caches tokens[0..n): mark every edge of the path
  void insert(int32_t w, const int32_t* t, int64_t n) {
    const uint64_t bit = 1ull << w;
    const uint64_t now = ++clock;
    MNode* cur = &root;
    int64_t i = 0;
    while (i < n) {
      auto it = cur->children.find(t[i]);
      if (it == cur->children.end()) {
        MNode* leaf = new MNode();
        leaf->tokens.assign(t + i, t + n);
        leaf->mask = bit;
        leaf->stamp.assign(size_t(workers), 0);
        leaf->stamp[size_t(w)] = now;
        leaf->parent = cur;
        cur->children[t[i]] = leaf;
        return;
      }
      MNode* ch = it->second;
      size_t k = common(ch->tokens.data(), ch->tokens.size(), t + i, size_t(n - i));
      if (k < ch->tokens.size()) ch = split(ch, k);
      ch->mask |= bit;
      ch->stamp[size_t(w)] = now;
      i += int64_t(k);
      cur = ch;
    }
  }

  void affinity(const int32_t* t, int64_t n, int64_t* aff) const {
    for (int32_t w = 0; w < workers; ++w) aff[w] = 0;
    uint64_t alive = workers >= 64 ? ~0ull : ((1ull << workers) - 1);
    const MNode* cur = &root;
    int64_t i = 0;
    while (i < n && alive) {
      auto it = cur->children.find(t[i]);
      if (it == cur->children.end()) break;
      const MNode* ch = it->second;
      size_t k = common(ch->tokens.data(), ch->tokens.size(), t + i, size_t(n - i));
      alive &= ch->mask;
      for (int32_t w = 0; w < workers; ++w)
        if (alive >> w & 1) aff[w] += int64_t(k);
      if (k < ch->tokens.size()) break;
      i += int64_t(k);
      cur = ch;
    }
  }

  // remove w from positions [leaf_start, path_len) of the path
  void apply(const EvictRec& r) {
    const uint64_t bit = 1ull << r.worker;
    const int32_t* t = r.path.data();
    const int64_t n = int64_t(r.path.size());
    MNode* cur = &root;
    int64_t i = 0;
    std::vector<MNode*> touched;
    while (i < n) {
      auto it = cur->children.find(t[i]);
      if (it == cur->children.end()) break;  // already gone (stale record)
      MNode* ch = it->second;
      size_t k = common(ch->tokens.data(), ch->tokens.size(), t + i, size_t(n - i));
      if (k < ch->tokens.size()) ch = split(ch, k);
      if (i < r.leaf_start && i + int64_t(k) > r.leaf_start) {
        // straddles the evicted leaf's start: split so only the leaf part loses w
        ch = split(ch, size_t(r.leaf_start - i));
        i = r.leaf_start;
        cur = ch;
        continue;
      }
      if (i >= r.leaf_start && ch->stamp[size_t(r.worker)] < r.stamp) {
        // only annotations older than the eviction: a later re-insert of the
        // same path by that worker survives (staleness may only over-approximate)
        ch->mask &= ~bit;
        touched.push_back(ch);
      }
      i += int64_t(k);
      cur = ch;
    }
    // prune childless nodes no worker claims, bottom-up from the deepest node
    // of the path (the touched nodes form one chain, so this covers them all)
    MNode* m = cur;
    while (m != &root && m->mask == 0 && m->children.empty()) {
      MNode* p = m->parent;
      p->children.erase(m->tokens[0]);
      delete m;
      m = p;
    }
    (void)touched;
  }
};

namespace {

void dump(const MNode* n, std::string& o) {
  o += "{\"tokens\":[";
  for (size_t i = 0; i < n->tokens.size(); ++i) {
    if (i) o += ',';
    o += std::to_string(n->tokens[i]);
  }
  o += "],\"mask\":" + std::to_string(n->mask) + ",\"children\":[";
  std::vector<int32_t> keys;
  for (auto& kv : n->children) keys.push_back(kv.first);
  std::sort(keys.begin(), keys.end());
  for (size_t i = 0; i < keys.size(); ++i) {
    if (i) o += ',';
    dump(n->children.at(keys[i]), o);
  }
  o += "]}";
}

}  // namespace

extern "C" {

rx_status rx_router_create(int32_t num_workers, rx_router** out) {
  if (!out || num_workers < 1 || num_workers > 64) return RX_E_INVALID;
  rx_router* r = new rx_router();
  r->workers = num_workers;
  *out = r;
  return RX_OK;
}

void rx_router_destroy(rx_router* r) { delete r; }

rx_status rx_router_affinity(const rx_router* r, const int32_t* tokens, int64_t n, int64_t* aff) {
  if (!r || n < 0 || (n > 0 && !tokens) || !aff) return RX_E_INVALID;
  r->affinity(tokens, n, aff);
  return RX_OK;
}

rx_status rx_router_dispatch(rx_router* r, int32_t batch, const int32_t* tokens, const int64_t* offsets,
                             int64_t* loads, double load_weight, int32_t* worker_out, int64_t* affinity_out) {
  if (!r || batch < 0 || (batch > 0 && (!tokens || !offsets || !loads || !worker_out)) || load_weight < 0)
    return RX_E_INVALID;
  std::vector<int64_t> aff(size_t(r->workers));
  for (int32_t b = 0; b < batch; ++b) {
    const int32_t* t = tokens + offsets[b];
    const int64_t n = offsets[b + 1] - offsets[b];
    r->affinity(t, n, aff.data());
    int32_t best = 0;
    for (int32_t w = 1; w < r->workers; ++w) {
      const double sw = double(aff[w]) - load_weight * double(loads[w]);
      const double sb = double(aff[best]) - load_weight * double(loads[best]);
      if (sw > sb || (sw == sb && loads[w] < loads[best])) best = w;
    }
    worker_out[b] = best;
    if (affinity_out) affinity_out[b] = aff[best];
    loads[best] += n - aff[best];
    r->insert(best, t, n);  // group affinity: later requests of the batch see it
  }
  return RX_OK;
}

rx_status rx_router_insert(rx_router* r, int32_t worker, const int32_t* tokens, int64_t n) {
  if (!r || worker < 0 || worker >= r->workers || n < 0 || (n > 0 && !tokens)) return RX_E_INVALID;
  r->insert(worker, tokens, n);
  return RX_OK;
}

rx_status rx_router_queue_evict(rx_router* r, int32_t worker, const int32_t* path, int64_t path_len,
                                int64_t leaf_start) {
  if (!r || worker < 0 || worker >= r->workers || path_len < 0 || leaf_start < 0 || leaf_start > path_len ||
      (path_len > 0 && !path))
    return RX_E_INVALID;
  r->queue.push_back({worker, std::vector<int32_t>(path, path + path_len), leaf_start, ++r->clock});
  return RX_OK;
}

int64_t rx_router_sync(rx_router* r) {
  if (!r) return -1;
  int64_t n = 0;
  while (!r->queue.empty()) {
    r->apply(r->queue.front());
    r->queue.pop_front();
    ++n;
  }
  return n;
}

int64_t rx_router_queue_len(const rx_router* r) { return r ? int64_t(r->queue.size()) : -1; }

int64_t rx_router_dump_json(const rx_router* r, char* buf, int64_t cap) {
  if (!r) return -1;
  std::string o;
  dump(&r->root, o);
  if (buf && cap > 0) {
    int64_t m = std::min<int64_t>(cap - 1, int64_t(o.size()));
    o.copy(buf, size_t(m));
    buf[m] = 0;
  }
  return int64_t(o.size());
}

}  // extern "C"
