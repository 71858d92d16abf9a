// decode_steps.cc — Alg. 1's output loop (§3 / App. A.2) for plain decoding, planned on
// the host in one C call per run of iterations: per iteration, alloc one slot per running request
// (evict the shortfall and retry once, R6; batch order, R23), write the slots into the host mirror
// of req_to_token, emit the device staging record of the step, and finish every request that
// produced its last token (decrease_ref_counter then insert(prompt + outputs)).  The
// mock-model tokens are known in advance, so nothing here waits for the device.
#include <algorithm>
#include <cstdint>
#include <vector>

#include "rx.h"

namespace {
struct EvictRelay {
  rx_step_event_cb cb;
  void* user;
};
void relay_run(void* u, const int32_t* slots, int64_t n) {
  auto* r = static_cast<EvictRelay*>(u);
  r->cb(r->user, RX_EV_EVICT_RUN, nullptr, slots, n);
}
}  // namespace

extern "C" {

rx_status rx_decode_steps(rx_cache* c, int32_t batch, int32_t* table, int64_t stride, int32_t* cur,
                          const int32_t* end, const int32_t* stable, const rx_node* nodes, const int32_t* tokens,
                          const int64_t* offsets, int32_t* running, int32_t* n_running, int32_t max_steps,
                          int32_t* out, int64_t out_cap, int64_t* step_meta, int32_t* n_steps,
                          rx_step_event_cb cb, void* user) {
  if (!c || !n_running || !n_steps || batch < 0 || stride < 1 || max_steps < 0 || out_cap < 0) return RX_E_INVALID;
  *n_steps = 0;
  if (*n_running < 0 || *n_running > batch) return RX_E_INVALID;
  if (*n_running == 0 || max_steps == 0) return RX_OK;
  if (!table || !cur || !end || !stable || !nodes || !tokens || !offsets || !running || !out || !step_meta)
    return RX_E_INVALID;
  for (int32_t k = 0; k < *n_running; ++k) {
    const int32_t b = running[k];
    if (b < 0 || b >= batch || (k > 0 && b <= running[k - 1])) return RX_E_INVALID;
    if (cur[b] >= end[b] || end[b] > stride || end[b] > offsets[b + 1] - offsets[b]) return RX_E_INVALID;
  }
  std::vector<int32_t> slots;
  int64_t used = 0;
  int32_t steps = 0;
  while (steps < max_steps && *n_running > 0) {
    const int32_t B = *n_running;
    if (used + 4 * int64_t(B) > out_cap) break;          // the caller launches these and calls again
    // Alg. 1 P:551-556 with R6: alloc, on shortfall evict (n - free) and retry once
    slots.resize(size_t(B));
    rx_status st = rx_alloc(c, B, slots.data());
    if (st == RX_E_NOMEM) {
      const int64_t short_by = B - rx_available(c);
      int64_t ev = 0;
      EvictRelay relay{cb, user};
      st = rx_evict(c, short_by, &ev, cb ? relay_run : nullptr, cb ? &relay : nullptr);
      if (st != RX_OK) return st;
      if (cb) {
        const int64_t v[2] = {short_by, ev};
        cb(user, RX_EV_EVICT, v, nullptr, 0);
      }
      st = rx_alloc(c, B, slots.data());
    }
    if (st != RX_OK) return st;                          // RX_E_NOMEM: this step is not planned
    if (cb) {
      const int64_t v[1] = {B};
      cb(user, RX_EV_ALLOC, v, slots.data(), B);
    }
    // the step's device record [new slots | seq_lens | table rows | stable lens], and the table
    int32_t* rec = out + used;
    int32_t max_seq = 0;
    for (int32_t k = 0; k < B; ++k) {
      const int32_t b = running[k];
      table[int64_t(b) * stride + cur[b]] = slots[size_t(k)];
      rec[k] = slots[size_t(k)];
      rec[B + k] = cur[b] + 1;                           // seq_len counts the new token
      rec[2 * B + k] = b;
      rec[3 * B + k] = stable[b];
      max_seq = std::max(max_seq, cur[b] + 1);
      cur[b] += 1;
    }
    step_meta[3 * steps] = B;
    step_meta[3 * steps + 1] = used;
    step_meta[3 * steps + 2] = max_seq;
    used += 4 * int64_t(B);
    ++steps;
    *n_steps = steps;
    // finished requests, in batch order
    int32_t keep = 0;
    for (int32_t k = 0; k < B; ++k) {
      const int32_t b = running[k];
      if (cur[b] < end[b]) {
        running[keep++] = b;
        continue;
      }
      int64_t d = 0, nc = 0, nd = 0;
      st = rx_dec_ref(c, nodes[b], &d);
      if (st != RX_OK) return st;
      st = rx_insert(c, tokens + offsets[b], table + int64_t(b) * stride, end[b], &nc, &nd);
      if (st != RX_OK) return st;
      if (cb) {
        const int64_t v[4] = {b, d, nc, nd};
        cb(user, RX_EV_FINISH, v, nullptr, 0);
      }
    }
    *n_running = keep;
  }
  return RX_OK;
}

}  // extern "C"
