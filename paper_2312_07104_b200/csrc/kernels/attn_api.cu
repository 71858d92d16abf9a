// C-ABI entry points for the device half of include/rx.h: argument checks,
// planning, and the launches of store.cu / extend.cu / decode.cu.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "../../../include/rx.h"

#include "params.cuh"

namespace {
thread_local int32_t g_last_launches = 0;

rx_status check_cfg(const rx_attn_cfg* c) {
  if (!c || c->h_q <= 0 || c->h_kv <= 0) return RX_E_INVALID;
  if (c->h_q % c->h_kv) return RX_E_UNSUPPORTED;
  const int G = c->h_q / c->h_kv;
  if (!(c->head_dim == 64 || c->head_dim == 128)) return RX_E_UNSUPPORTED;
  if (!(G == 1 || G == 2 || G == 4 || G == 8)) return RX_E_UNSUPPORTED;
  return RX_OK;
}
// rx_extend kernel choice: the multi-query decode kernel when every request's segment is at most
// 32 (row, head) columns (<= 4 column tiles of 8) and (request, kv head) pairs alone fill the SMs
// (it runs one split per request); the tcgen05 extend kernel otherwise.  RX_EXTEND_MULTI=0 turns
// the multi-query path off (A/B knob).
bool use_multi_query(int G, int batch, int h_kv, int max_ext) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("RX_EXTEND_MULTI");
    env = e ? atoi(e) : 1;
  }
  return env != 0 && max_ext * G <= 32 && int64_t(batch) * h_kv >= 148;
}
}  // namespace

extern "C" {

const char* rx_status_str(int s) {
  switch (s) {
    case RX_OK: return "RX_OK";
    case RX_E_INVALID: return "RX_E_INVALID";
    case RX_E_NOMEM: return "RX_E_NOMEM";
    case RX_E_UNDERFLOW: return "RX_E_UNDERFLOW";
    case RX_E_STALE: return "RX_E_STALE";
    case RX_E_UNSUPPORTED: return "RX_E_UNSUPPORTED";
    case RX_E_CUDA: return "RX_E_CUDA";
    case RX_E_WORKSPACE: return "RX_E_WORKSPACE";
    case RX_E_CAPACITY: return "RX_E_CAPACITY";
    default: return "RX_E_UNKNOWN";
  }
}

const char* rx_version(void) { return "rx 0.1 sm_100a (tcgen05 extend, mma.sync decode)"; }

int32_t rx_last_launch_count(void) { return g_last_launches; }

rx_status rx_store_kv(const rx_attn_cfg* cfg, int64_t n, const int32_t* d_slots, const void* d_k, const void* d_v,
                      void* d_k_pool, void* d_v_pool, int64_t num_slots, int32_t* d_rtt,
                      const int64_t* d_rtt_index, void* stream) {
  rx_status s = check_cfg(cfg);
  if (s != RX_OK) return s;
  if (n < 0 || num_slots < 1) return RX_E_INVALID;
  const bool table_only = !d_k && !d_v && d_rtt_index;      // append table entries only
  if (n > 0 && (!d_slots || (!table_only && (!d_k || !d_v || !d_k_pool || !d_v_pool)))) return RX_E_INVALID;
  if (d_rtt_index && !d_rtt) return RX_E_INVALID;
  g_last_launches = 0;
  if (n == 0) return RX_OK;
  cudaError_t e = rx::launch_store_kv(n, cfg->h_kv * cfg->head_dim * 2, d_slots, d_k, d_v, d_k_pool, d_v_pool,
                                      d_rtt, d_rtt_index, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return RX_E_CUDA;
  g_last_launches = 1;
  return RX_OK;
}

rx_status rx_copy_h2d(void* d_dst, const void* h_src, int64_t bytes, void* stream) {
  if (bytes < 0 || (bytes > 0 && (!d_dst || !h_src))) return RX_E_INVALID;
  g_last_launches = 0;
  if (bytes == 0) return RX_OK;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, h_src) != cudaSuccess || a.type != cudaMemoryTypeHost) return RX_E_INVALID;
  if (rx::launch_copy_h2d(d_dst, a.devicePointer ? a.devicePointer : h_src, bytes,
                          static_cast<cudaStream_t>(stream)) != cudaSuccess)
    return RX_E_CUDA;
  g_last_launches = 1;
  return RX_OK;
}

size_t rx_decode_workspace_bytes(const rx_attn_cfg* cfg, int32_t batch, int32_t max_seq_len) {
  if (check_cfg(cfg) != RX_OK || batch <= 0 || max_seq_len <= 0) return 0;
  return rx::decode_ws_bytes(cfg->h_q, cfg->head_dim, batch, max_seq_len, cfg->h_kv);
}

static rx_status decode_impl(const rx_attn_cfg* cfg, int32_t batch, const int32_t* d_rtt, int64_t rtt_stride,
                             const int32_t* d_rows, const int32_t* d_seq_lens, int32_t max_seq_len, const void* d_q,
                             const void* d_k_pool, const void* d_v_pool, int64_t num_slots, void* d_o, void* d_ws,
                             size_t ws_bytes, void* stream, const void* d_k_new, const void* d_v_new,
                             const int32_t* d_new_slots, int32_t* d_rtt_w, const int32_t* d_stable_lens,
                             const rx::OutSpec* os = nullptr) {
  rx_status s = check_cfg(cfg);
  if (s != RX_OK) return s;
  if (batch < 0 || max_seq_len < 0 || num_slots < 1) return RX_E_INVALID;
  g_last_launches = 0;
  if (batch == 0) return RX_OK;
  if (max_seq_len < 1 || !d_rtt || !d_seq_lens || !d_q || !d_k_pool || !d_v_pool || (!d_o && !os))
    return RX_E_INVALID;
  if (rtt_stride < max_seq_len) return RX_E_INVALID;
  const size_t need = rx::decode_ws_bytes(cfg->h_q, cfg->head_dim, batch, max_seq_len, cfg->h_kv);
  if (need > 0 && (!d_ws || ws_bytes < need)) return RX_E_WORKSPACE;
  rx::DecodePlan pl = rx::plan_decode(batch, cfg->h_kv, max_seq_len);
  rx::DecodeParams p{};
  p.q = static_cast<const __nv_bfloat16*>(d_q);
  p.kpool = static_cast<const __nv_bfloat16*>(d_k_pool);
  p.vpool = static_cast<const __nv_bfloat16*>(d_v_pool);
  p.o = static_cast<__nv_bfloat16*>(d_o);
  p.rtt = d_rtt;
  p.rtt_stride = rtt_stride;
  p.rows = d_rows;
  p.seq_lens = d_seq_lens;
  const size_t n = size_t(batch) * cfg->h_q * pl.max_splits;
  char* part = need ? static_cast<char*>(d_ws) + rx::kWsHeader : nullptr;   // partials follow the header
  p.ws_o = reinterpret_cast<float*>(part);
  p.ws_lse = need ? reinterpret_cast<float*>(part + n * cfg->head_dim * sizeof(float)) : nullptr;
  p.h_q = cfg->h_q;
  p.h_kv = cfg->h_kv;
  p.chunk = pl.chunk;
  p.max_splits = pl.max_splits;
  p.scale_log2 = cfg->sm_scale * 1.4426950408889634f;
  p.k_new = static_cast<const __nv_bfloat16*>(d_k_new);
  p.v_new = static_cast<const __nv_bfloat16*>(d_v_new);
  p.new_slots = d_new_slots;
  p.rtt_w = d_rtt_w;
  p.stable_lens = d_stable_lens;
  if (os) p.out = *os;
  int launches = 0;
  cudaError_t e = rx::launch_decode(cfg->head_dim, cfg->h_q / cfg->h_kv, p, batch,
                                    static_cast<cudaStream_t>(stream), &launches);
  if (e != cudaSuccess) return RX_E_CUDA;
  g_last_launches = launches;
  return RX_OK;
}

rx_status rx_decode(const rx_attn_cfg* cfg, int32_t batch, const int32_t* d_rtt, int64_t rtt_stride,
                    const int32_t* d_rows, const int32_t* d_seq_lens, int32_t max_seq_len, const void* d_q,
                    const void* d_k_pool, const void* d_v_pool, int64_t num_slots, void* d_o, void* d_ws,
                    size_t ws_bytes, void* stream) {
  return decode_impl(cfg, batch, d_rtt, rtt_stride, d_rows, d_seq_lens, max_seq_len, d_q, d_k_pool, d_v_pool,
                     num_slots, d_o, d_ws, ws_bytes, stream, nullptr, nullptr, nullptr, nullptr, nullptr);
}

rx_status rx_decode_append(const rx_attn_cfg* cfg, int32_t batch, int32_t* d_rtt, int64_t rtt_stride,
                           const int32_t* d_rows, const int32_t* d_seq_lens, const int32_t* d_stable_lens,
                           int32_t max_seq_len, const void* d_q, const void* d_k_new, const void* d_v_new,
                           const int32_t* d_new_slots, void* d_k_pool, void* d_v_pool, int64_t num_slots, void* d_o,
                           void* d_ws, size_t ws_bytes, void* stream) {
  if (!d_k_new || !d_v_new || !d_new_slots) return RX_E_INVALID;
  return decode_impl(cfg, batch, d_rtt, rtt_stride, d_rows, d_seq_lens, max_seq_len, d_q, d_k_pool, d_v_pool,
                     num_slots, d_o, d_ws, ws_bytes, stream, d_k_new, d_v_new, d_new_slots, d_rtt, d_stable_lens);
}

size_t rx_decode_cascade_workspace_bytes(const rx_attn_cfg* cfg, int32_t batch, int32_t max_seq_len,
                                         int32_t shared_len) {
  if (check_cfg(cfg) != RX_OK || batch <= 0 || shared_len <= 0 || max_seq_len <= shared_len) return 0;
  return rx::cascade_ws_bytes(cfg->h_q, cfg->head_dim, batch, cfg->h_kv, max_seq_len, shared_len);
}

static rx_status cascade_impl(const rx_attn_cfg* cfg, int32_t batch, int32_t* d_rtt, int64_t rtt_stride,
                              const int32_t* d_rows, const int32_t* d_seq_lens, const int32_t* d_stable_lens,
                              int32_t max_seq_len, int32_t shared_len, const void* d_q, const void* d_k_new,
                              const void* d_v_new, const int32_t* d_new_slots, void* d_k_pool, void* d_v_pool,
                              int64_t num_slots, void* d_o, void* d_ws, size_t ws_bytes, void* stream,
                              const rx::OutSpec* os) {
  rx_status s = check_cfg(cfg);
  if (s != RX_OK) return s;
  if (batch < 0 || num_slots < 1 || shared_len < 0) return RX_E_INVALID;
  g_last_launches = 0;
  if (batch == 0) return RX_OK;
  if (shared_len == 0) {  // nothing shared: the ordinary fused path
    if (!d_k_new || !d_v_new || !d_new_slots) return RX_E_INVALID;
    return decode_impl(cfg, batch, d_rtt, rtt_stride, d_rows, d_seq_lens, max_seq_len, d_q, d_k_pool, d_v_pool,
                       num_slots, d_o, d_ws, ws_bytes, stream, d_k_new, d_v_new, d_new_slots, d_rtt, d_stable_lens,
                       os);
  }
  if (max_seq_len <= shared_len || !d_rtt || !d_seq_lens || !d_q || !d_k_new || !d_v_new || !d_new_slots ||
      !d_k_pool || !d_v_pool || (!d_o && !os) || rtt_stride < max_seq_len)
    return RX_E_INVALID;
  const int G = cfg->h_q / cfg->h_kv;
  const size_t need = rx::cascade_ws_bytes(cfg->h_q, cfg->head_dim, batch, cfg->h_kv, max_seq_len, shared_len);
  if (!d_ws || ws_bytes < need) return RX_E_WORKSPACE;
  const rx::CascadePlan pl = rx::plan_cascade(batch, cfg->h_kv, G, max_seq_len, shared_len);
  const size_t n = size_t(batch) * cfg->h_q * pl.total_splits;
  char* part = static_cast<char*>(d_ws) + rx::kWsHeader;
  float* ws_o = reinterpret_cast<float*>(part);
  float* ws_lse = reinterpret_cast<float*>(part + n * cfg->head_dim * sizeof(float));
  const float scale_log2 = cfg->sm_scale * 1.4426950408889634f;
  cudaStream_t st = static_cast<cudaStream_t>(stream);

  // (1) suffix [shared_len, seq_len) + the step's KV append: partials at split >= n_sh
  rx::DecodeParams dp{};
  dp.q = static_cast<const __nv_bfloat16*>(d_q);
  dp.kpool = static_cast<const __nv_bfloat16*>(d_k_pool);
  dp.vpool = static_cast<const __nv_bfloat16*>(d_v_pool);
  dp.o = static_cast<__nv_bfloat16*>(d_o);
  dp.rtt = d_rtt;
  dp.rtt_stride = rtt_stride;
  dp.rows = d_rows;
  dp.seq_lens = d_seq_lens;
  dp.ws_o = ws_o;
  dp.ws_lse = ws_lse;
  dp.h_q = cfg->h_q;
  dp.h_kv = cfg->h_kv;
  dp.chunk = pl.suffix.chunk;
  dp.max_splits = pl.total_splits;
  dp.scale_log2 = scale_log2;
  dp.k_new = static_cast<const __nv_bfloat16*>(d_k_new);
  dp.v_new = static_cast<const __nv_bfloat16*>(d_v_new);
  dp.new_slots = d_new_slots;
  dp.rtt_w = d_rtt;
  dp.kv_start = shared_len;
  dp.split_base = pl.n_sh;
  dp.stable_lens = d_stable_lens;
  // the shared pass launched next needs whole SMs: release it after the suffix streaming
  // (RX_CASCADE_EARLY=1: as soon as every suffix CTA has started — A/B knob)
  static int early = -1;
  if (early < 0) {
    const char* ev = getenv("RX_CASCADE_EARLY");
    early = ev ? atoi(ev) : 0;
  }
  dp.late_trigger = early ? 0 : 1;
  int launches = 0;
  cudaError_t e = rx::launch_decode(cfg->head_dim, G, dp, batch, st, &launches);
  if (e != cudaSuccess) return RX_E_CUDA;
  // (2) shared prefix [0, shared_len), attended ONCE for all requests on the tensor cores (rows =
  //     requests x GQA heads), stream-K over the SMs: partials at [0, n_sh); (3) the log-sum-exp
  //     merge with (1)'s suffix partials into o
  rx::ExtendParams ep{};
  ep.rtt = d_rtt;
  ep.rtt_stride = rtt_stride;
  ep.rows = d_rows;
  ep.kpool = static_cast<__nv_bfloat16*>(d_k_pool);
  ep.vpool = static_cast<__nv_bfloat16*>(d_v_pool);
  ep.o = static_cast<__nv_bfloat16*>(d_o);
  ep.h_q = cfg->h_q;
  ep.h_kv = cfg->h_kv;
  ep.num_slots = num_slots;
  ep.scale_log2 = scale_log2;
  ep.cascade = 1;
  ep.cas_ctas = pl.ctas;
  ep.cas_tiles = pl.tiles;
  ep.n_sh = pl.n_sh;
  ep.part_o = ws_o;
  ep.part_lse = ws_lse;
  ep.part_splits = pl.total_splits;
  ep.cas_prefix = shared_len;
  ep.cas_seq_lens = d_seq_lens;
  ep.cas_kv_start = shared_len;
  ep.cas_chunk = pl.suffix.chunk;
  ep.pdl = rx::pdl_on();
  ep.sched = static_cast<int*>(d_ws);
  if (os) ep.out = *os;
  e = rx::launch_extend_cascade(cfg->head_dim, G, ep, d_q, batch, st);
  if (e != cudaSuccess) return RX_E_CUDA;
  g_last_launches = launches + 2;
  return RX_OK;
}

rx_status rx_decode_cascade_append(const rx_attn_cfg* cfg, int32_t batch, int32_t* d_rtt, int64_t rtt_stride,
                                   const int32_t* d_rows, const int32_t* d_seq_lens, const int32_t* d_stable_lens,
                                   int32_t max_seq_len,
                                   int32_t shared_len, const void* d_q, const void* d_k_new, const void* d_v_new,
                                   const int32_t* d_new_slots, void* d_k_pool, void* d_v_pool, int64_t num_slots,
                                   void* d_o, void* d_ws, size_t ws_bytes, void* stream) {
  if (!d_o) return RX_E_INVALID;
  return cascade_impl(cfg, batch, d_rtt, rtt_stride, d_rows, d_seq_lens, d_stable_lens, max_seq_len, shared_len,
                      d_q, d_k_new, d_v_new, d_new_slots, d_k_pool, d_v_pool, num_slots, d_o, d_ws, ws_bytes, stream,
                      nullptr);
}

rx_status rx_decode_run(const rx_attn_cfg* cfg, int32_t n_steps, const int32_t* h_batch, const int32_t* h_max_seq,
                        int32_t shared_len, int32_t* d_rtt, int64_t rtt_stride, const int32_t* d_rec,
                        const int64_t* h_rec_off, int32_t with_stable, void* const* h_q, void* const* h_k_new,
                        void* const* h_v_new, void* d_k_pool, void* d_v_pool, int64_t num_slots, void* const* h_o,
                        int32_t tp_world, int32_t tp_h_q_total, int32_t tp_head_offset, void* d_ws,
                        size_t ws_bytes, void* stream) {
  if (n_steps < 0 || (n_steps > 0 && (!h_batch || !h_max_seq || !d_rec || !h_rec_off || !h_q || !h_k_new ||
                                      !h_v_new || !h_o)))
    return RX_E_INVALID;
  if (tp_world < 0 || tp_world > rx::kTpMaxRanks || !cfg ||
      (tp_world > 0 && (tp_head_offset < 0 || tp_h_q_total < tp_head_offset + cfg->h_q)))
    return RX_E_INVALID;
  const int32_t W = tp_world > 0 ? tp_world : 1;
  int32_t total = 0;
  for (int32_t k = 0; k < n_steps; ++k) {
    const int32_t B = h_batch[k];
    if (B < 0 || h_rec_off[k] < 0) return RX_E_INVALID;
    const int32_t* r = d_rec + h_rec_off[k];   // [new slots | seq_lens | rows | stable lens], B each
    rx::OutSpec os{};
    if (tp_world > 0) {                        // step k's gathered block on every rank (fused gather)
      for (int32_t p = 0; p < tp_world; ++p) {
        if (!h_o[int64_t(k) * W + p]) return RX_E_INVALID;
        os.ptr[p] = static_cast<__nv_bfloat16*>(h_o[int64_t(k) * W + p]);
      }
      os.n = tp_world;
      os.head_off = tp_head_offset;
      os.row_stride = int64_t(tp_h_q_total) * cfg->head_dim;
    }
    const rx_status st =
        cascade_impl(cfg, B, d_rtt, rtt_stride, r + 2 * B, r + B, with_stable ? r + 3 * B : nullptr, h_max_seq[k],
                     shared_len, h_q[k], h_k_new[k], h_v_new[k], r, d_k_pool, d_v_pool, num_slots,
                     tp_world > 0 ? nullptr : h_o[k], d_ws, ws_bytes, stream, tp_world > 0 ? &os : nullptr);
    if (st != RX_OK) return st;
    total += g_last_launches;
  }
  g_last_launches = total;
  return RX_OK;
}

rx_status rx_decode_append_tp(const rx_attn_cfg* cfg, int32_t batch, int32_t* d_rtt, int64_t rtt_stride,
                              const int32_t* d_rows, const int32_t* d_seq_lens, const int32_t* d_stable_lens,
                              int32_t max_seq_len, int32_t shared_len, const void* d_q, const void* d_k_new,
                              const void* d_v_new, const int32_t* d_new_slots, void* d_k_pool, void* d_v_pool,
                              int64_t num_slots, const rx_tp_out* out, void* d_ws, size_t ws_bytes, void* stream) {
  if (!out || out->world < 1 || out->world > rx::kTpMaxRanks || !cfg || out->head_offset < 0 ||
      out->h_q_total < out->head_offset + cfg->h_q)
    return RX_E_INVALID;
  rx::OutSpec os{};
  for (int i = 0; i < out->world; ++i) {
    if (!out->d_o[i]) return RX_E_INVALID;
    os.ptr[i] = static_cast<__nv_bfloat16*>(out->d_o[i]);
  }
  os.n = out->world;
  os.head_off = out->head_offset;
  os.row_stride = int64_t(out->h_q_total) * cfg->head_dim;
  return cascade_impl(cfg, batch, d_rtt, rtt_stride, d_rows, d_seq_lens, d_stable_lens, max_seq_len, shared_len,
                      d_q, d_k_new, d_v_new, d_new_slots, d_k_pool, d_v_pool, num_slots, nullptr, d_ws, ws_bytes,
                      stream, &os);
}

// Multi-query cascade (rx_extend_cascade): rows = every new token of the batch.
static rx::CascadePlan plan_extend_cascade(const rx_attn_cfg* cfg, int64_t total_new, int32_t shared_len) {
  rx::CascadePlan pl = rx::plan_cascade(int(total_new), cfg->h_kv, cfg->h_q / cfg->h_kv, shared_len + 1, shared_len);
  pl.total_splits = pl.n_sh + 1;
  return pl;
}

size_t rx_extend_cascade_workspace_bytes(const rx_attn_cfg* cfg, int64_t total_new, int32_t shared_len) {
  if (check_cfg(cfg) != RX_OK || total_new <= 0 || shared_len <= 0) return 0;
  const rx::CascadePlan pl = plan_extend_cascade(cfg, total_new, shared_len);
  const size_t n = size_t(total_new) * cfg->h_q * pl.total_splits;
  return rx::kWsHeader + n * cfg->head_dim * sizeof(float) + n * sizeof(float) + 256;
}

rx_status rx_extend_cascade(const rx_attn_cfg* cfg, int32_t batch, const int32_t* d_rtt, int64_t rtt_stride,
                            const int32_t* d_rows, const int32_t* d_prefix_lens, const int32_t* d_extend_lens,
                            const int32_t* d_qo_indptr, int64_t total_new, int32_t max_extend_len,
                            int32_t max_prefix_len, int32_t shared_len, const void* d_q, const void* d_k_new,
                            const void* d_v_new, void* d_k_pool, void* d_v_pool, int64_t num_slots, void* d_o,
                            void* d_ws, size_t ws_bytes, void* stream) {
  rx_status s = check_cfg(cfg);
  if (s != RX_OK) return s;
  if (shared_len < 0 || total_new < 0 || batch < 0) return RX_E_INVALID;
  const int G = cfg->h_q / cfg->h_kv;
  if (shared_len == 0 || batch == 0 || total_new == 0 || !use_multi_query(G, batch, cfg->h_kv, max_extend_len))
    return rx_extend(cfg, batch, d_rtt, rtt_stride, d_rows, d_prefix_lens, d_extend_lens, d_qo_indptr, total_new,
                     max_extend_len, max_prefix_len, d_q, d_k_new, d_v_new, d_k_pool, d_v_pool, num_slots, d_o,
                     d_ws, ws_bytes, stream);
  if (!d_rtt || !d_prefix_lens || !d_extend_lens || !d_qo_indptr || !d_q || !d_k_new || !d_v_new || !d_k_pool ||
      !d_v_pool || !d_o || num_slots < 1 || max_extend_len < 1)
    return RX_E_INVALID;
  if (rtt_stride < max_prefix_len || rtt_stride < max_extend_len || shared_len > max_prefix_len)
    return RX_E_INVALID;
  const size_t need = rx_extend_cascade_workspace_bytes(cfg, total_new, shared_len);
  if (!d_ws || ws_bytes < need) return RX_E_WORKSPACE;
  g_last_launches = 0;
  const rx::CascadePlan pl = plan_extend_cascade(cfg, total_new, shared_len);
  const size_t n = size_t(total_new) * cfg->h_q * pl.total_splits;
  char* part = static_cast<char*>(d_ws) + rx::kWsHeader;
  float* ws_o = reinterpret_cast<float*>(part);
  float* ws_lse = reinterpret_cast<float*>(part + n * cfg->head_dim * sizeof(float));
  const float scale_log2 = cfg->sm_scale * 1.4426950408889634f;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // A5: the new rows into their slots
  cudaError_t e = rx::launch_extend_store(total_new, batch, cfg->h_kv * cfg->head_dim * 2, d_qo_indptr, d_extend_lens,
                                          d_prefix_lens, d_rows, d_rtt, rtt_stride, d_k_new, d_v_new, d_k_pool,
                                          d_v_pool, st);
  if (e != cudaSuccess) return RX_E_CUDA;
  // (1) each request's own positions [shared_len, prefix + j] on the multi-query decode kernel:
  //     partial at split n_sh of every row
  rx::DecodeParams dp{};
  dp.q = static_cast<const __nv_bfloat16*>(d_q);
  dp.kpool = static_cast<const __nv_bfloat16*>(d_k_pool);
  dp.vpool = static_cast<const __nv_bfloat16*>(d_v_pool);
  dp.o = static_cast<__nv_bfloat16*>(d_o);
  dp.rtt = d_rtt;
  dp.rtt_stride = rtt_stride;
  dp.rows = d_rows;
  dp.ws_o = ws_o;
  dp.ws_lse = ws_lse;
  dp.h_q = cfg->h_q;
  dp.h_kv = cfg->h_kv;
  dp.chunk = (max_prefix_len + max_extend_len + 15) / 16 * 16;
  dp.max_splits = pl.total_splits;
  dp.scale_log2 = scale_log2;
  dp.qo_indptr = d_qo_indptr;
  dp.prefix_lens = d_prefix_lens;
  dp.col_tiles = (max_extend_len * G + 7) / 8;
  dp.kv_start = shared_len;
  dp.split_base = pl.n_sh;
  e = rx::launch_decode_multi(cfg->head_dim, G, dp, batch, st);
  if (e != cudaSuccess) return RX_E_CUDA;
  // (2) the shared prefix [0, shared_len) once for every row of the batch on tcgen05 (the rows are
  //     one virtual request, no mask: every row's position is >= shared_len), stream-K; (3) the
  //     log-sum-exp merge with (1)'s partial into o
  rx::ExtendParams ep{};
  ep.rtt = d_rtt;
  ep.rtt_stride = rtt_stride;
  ep.rows = d_rows;
  ep.kpool = static_cast<__nv_bfloat16*>(d_k_pool);
  ep.vpool = static_cast<__nv_bfloat16*>(d_v_pool);
  ep.o = static_cast<__nv_bfloat16*>(d_o);
  ep.h_q = cfg->h_q;
  ep.h_kv = cfg->h_kv;
  ep.num_slots = num_slots;
  ep.scale_log2 = scale_log2;
  ep.cascade = 1;
  ep.cas_ctas = pl.ctas;
  ep.cas_tiles = pl.tiles;
  ep.n_sh = pl.n_sh;
  ep.part_o = ws_o;
  ep.part_lse = ws_lse;
  ep.part_splits = pl.total_splits;
  ep.cas_prefix = shared_len;
  ep.cas_fixed_suffix = 1;
  ep.sched = static_cast<int*>(d_ws);
  e = rx::launch_extend_cascade(cfg->head_dim, G, ep, d_q, int(total_new), st);
  if (e != cudaSuccess) return RX_E_CUDA;
  g_last_launches = 4;
  return RX_OK;
}

size_t rx_extend_workspace_bytes(const rx_attn_cfg* cfg, int32_t batch, int32_t max_extend_len) {
  // the persistent kernel's work counters (the workspace header); the short-segment path uses none
  if (check_cfg(cfg) != RX_OK || batch <= 0 || max_extend_len <= 0) return 0;
  return rx::kWsHeader;
}

rx_status rx_extend(const rx_attn_cfg* cfg, int32_t batch, const int32_t* d_rtt, int64_t rtt_stride,
                    const int32_t* d_rows, const int32_t* d_prefix_lens, const int32_t* d_extend_lens,
                    const int32_t* d_qo_indptr, int64_t total_new, int32_t max_extend_len, int32_t max_prefix_len,
                    const void* d_q, const void* d_k_new, const void* d_v_new, void* d_k_pool, void* d_v_pool,
                    int64_t num_slots, void* d_o, void* d_ws, size_t ws_bytes, void* stream) {
  rx_status s = check_cfg(cfg);
  if (s != RX_OK) return s;
  if (batch < 0 || total_new < 0 || max_extend_len < 0 || max_prefix_len < 0 || num_slots < 1)
    return RX_E_INVALID;
  g_last_launches = 0;
  if (batch == 0 || total_new == 0 || max_extend_len == 0) return RX_OK;
  if (!d_rtt || !d_prefix_lens || !d_extend_lens || !d_qo_indptr || !d_q || !d_k_new || !d_v_new || !d_k_pool ||
      !d_v_pool || !d_o)
    return RX_E_INVALID;
  if (rtt_stride < max_prefix_len || rtt_stride < max_extend_len) return RX_E_INVALID;
  const int G = cfg->h_q / cfg->h_kv;
  const bool multi = use_multi_query(G, batch, cfg->h_kv, max_extend_len);
  if (!multi && (!d_ws || ws_bytes < rx::kWsHeader)) return RX_E_WORKSPACE;
  rx::ExtendParams p{};
  p.rtt = d_rtt;
  p.rtt_stride = rtt_stride;
  p.rows = d_rows;
  p.prefix_lens = d_prefix_lens;
  p.extend_lens = d_extend_lens;
  p.qo_indptr = d_qo_indptr;
  p.k_new = static_cast<const __nv_bfloat16*>(d_k_new);
  p.v_new = static_cast<const __nv_bfloat16*>(d_v_new);
  p.kpool = static_cast<__nv_bfloat16*>(d_k_pool);
  p.vpool = static_cast<__nv_bfloat16*>(d_v_pool);
  p.o = static_cast<__nv_bfloat16*>(d_o);
  p.h_q = cfg->h_q;
  p.h_kv = cfg->h_kv;
  p.num_slots = num_slots;
  p.scale_log2 = cfg->sm_scale * 1.4426950408889634f;
  p.sched = static_cast<int*>(d_ws);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // A5: new K/V rows into their slots (independent of the attention reads:
  // new slots are never prefix slots, and the attention reads k_new/v_new)
  cudaError_t e = rx::launch_extend_store(total_new, batch, cfg->h_kv * cfg->head_dim * 2, d_qo_indptr, d_extend_lens,
                                          d_prefix_lens, d_rows, d_rtt, rtt_stride, d_k_new, d_v_new, d_k_pool,
                                          d_v_pool, st);
  if (e != cudaSuccess) return RX_E_CUDA;
  if (multi) {
    // short segments (jump-forward edges, §4): (row, head) columns of the decode kernel's
    // mma.sync tile instead of 128-row tcgen05 tiles that would be almost all padding
    rx::DecodeParams dp{};
    dp.q = static_cast<const __nv_bfloat16*>(d_q);
    dp.kpool = static_cast<const __nv_bfloat16*>(d_k_pool);
    dp.vpool = static_cast<const __nv_bfloat16*>(d_v_pool);
    dp.o = static_cast<__nv_bfloat16*>(d_o);
    dp.rtt = d_rtt;
    dp.rtt_stride = rtt_stride;
    dp.rows = d_rows;
    dp.h_q = cfg->h_q;
    dp.h_kv = cfg->h_kv;
    dp.chunk = (max_prefix_len + max_extend_len + 15) / 16 * 16;   // one split per request
    dp.max_splits = 1;
    dp.scale_log2 = p.scale_log2;
    dp.qo_indptr = d_qo_indptr;
    dp.prefix_lens = d_prefix_lens;
    dp.col_tiles = (max_extend_len * G + 7) / 8;
    e = rx::launch_decode_multi(cfg->head_dim, G, dp, batch, st);
  } else {
    e = rx::launch_extend(cfg->head_dim, G, p, d_q, total_new, batch, max_extend_len, st);
  }
  if (e != cudaSuccess) return RX_E_CUDA;
  g_last_launches = 2;
  return RX_OK;
}

}  // extern "C"
