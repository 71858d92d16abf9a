// scheduler.cc — cache-aware admission (Alg. 1 lines P:522-547, §3 "Cache-aware scheduling"
// P:214-219) as one host C call per scheduling step: match every waiting request, order the queue
// by the policy, admit under the memory fit check, pin the admitted requests' prefix nodes.
//
// Policies (P:432 ablation "FCFS Schedule" / "Random Schedule" vs the paper's order):
//   RX_SCHED_LSPF   longest matched prefix first, arrival order breaks ties (Theorem 1)
//   RX_SCHED_FCFS   arrival order
//   RX_SCHED_RANDOM ascending caller-supplied keys[b], arrival order breaks ties (the random draw is an
//                   input, so the oracle and this library produce the same order)
// Fit check (readings R7, R25): admit while size + current < available + delta, available =
// evictable + free updated by each inc_ref delta, delta = the candidate's own
// pin delta, current += size after each admission, size = (prompt - usable prefix) + max_new
// (R11: usable prefix = min(matched, n - 1)).
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <vector>

#include "rx.h"

extern "C" {

rx_status rx_schedule(rx_cache* c, int32_t batch, const int32_t* tokens, const int64_t* offsets,
                      const int64_t* max_new, int32_t policy, const uint64_t* keys, rx_node* nodes,
                      int64_t* matched, int32_t* slots_out, int32_t* admitted, int32_t* n_admitted,
                      int64_t* deltas) {
  if (!c || batch < 0 || !n_admitted) return RX_E_INVALID;
  *n_admitted = 0;
  if (batch == 0) return RX_OK;
  if (!tokens || !offsets || !max_new || !nodes || !matched || !admitted) return RX_E_INVALID;
  if (policy != RX_SCHED_LSPF && policy != RX_SCHED_FCFS && policy != RX_SCHED_RANDOM) return RX_E_INVALID;
  if (policy == RX_SCHED_RANDOM && !keys) return RX_E_INVALID;
  for (int32_t b = 0; b < batch; ++b) {
    if (offsets[b + 1] - offsets[b] < 1 || max_new[b] < 0) return RX_E_INVALID;
  }
  // Alg. 1: T.match_prefix for every waiting request (in arrival order: clock ticks)
  rx_status st = rx_match_prefix_batch(c, batch, tokens, offsets, nodes, matched, slots_out);
  if (st != RX_OK) return st;
  // requests.sort()
  std::vector<int32_t> order(static_cast<size_t>(batch));
  std::iota(order.begin(), order.end(), 0);
  if (policy == RX_SCHED_LSPF) {
    std::stable_sort(order.begin(), order.end(),
                     [&](int32_t a, int32_t b) { return matched[a] > matched[b]; });
  } else if (policy == RX_SCHED_RANDOM) {
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return keys[a] < keys[b]; });
  }
  // select requests for the next batch
  int64_t available = rx_evictable_size(c) + rx_available(c);
  int64_t current = 0;
  int32_t k = 0;
  for (int32_t b : order) {
    const int64_t n = offsets[b + 1] - offsets[b];
    const int64_t usable = std::min<int64_t>(matched[b], n - 1);
    const int64_t size = (n - usable) + max_new[b];
    // reading R25: the candidate's own pin delta counts in its fit check (pin, test, unpin on
    // failure), so sum(size) < evictable + free holds after every admission
    int64_t d = 0;
    st = rx_inc_ref(c, nodes[b], &d);
    if (st != RX_OK) return st;
    if (size + current < available + d) {
      available += d;
      current += size;
      if (deltas) deltas[k] = d;
      admitted[k++] = b;
    } else {
      st = rx_dec_ref(c, nodes[b], nullptr);
      if (st != RX_OK) return st;
    }
  }
  *n_admitted = k;
  return RX_OK;
}

}  // extern "C"
