// Kernel parameter blocks and launcher prototypes shared by the rx kernels
// and their C-ABI wrappers (attn_api.cu).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <cstdlib>

namespace rx {

// Every workspace a call takes (include/rx.h "Workspaces") starts with a 256-byte header that
// holds the persistent extend kernel's work counters ([0] next work index, [1] CTAs finished).
// It must be zero before the workspace is first used; every call leaves it zero again (the last
// CTA of an extend grid resets it).  Partial buffers follow the header.  Keeping the counters in
// the caller's workspace (not in a __device__ global) makes calls on different streams with
// different workspaces independent.
constexpr size_t kWsHeader = 256;

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device): the attribute is
// per device context, so a process that drives several GPUs sets it on each.  Keyed by the kernel's
// address (every instantiation of a kernel template has the same function TYPE).
cudaError_t ensure_smem_attr_ptr(const void* kern, int bytes);   // decode.cu
template <typename Kern>
inline cudaError_t ensure_smem_attr(Kern* kern, int bytes) {
  return ensure_smem_attr_ptr(reinterpret_cast<const void*>(kern), bytes);
}

// SM count of the current device (cached per device)
inline int device_sms() {
  static int sms[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  int& v = sms[dev & 63];
  if (!v) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    v = n > 0 ? n : 148;
  }
  return v;
}

struct DecodeParams {
  const __nv_bfloat16* q;       // [B, h_q, HD]
  const __nv_bfloat16* kpool;   // [S, h_kv, HD]
  const __nv_bfloat16* vpool;
  __nv_bfloat16* o;             // [B, h_q, HD]
  const int32_t* rtt;
  int64_t rtt_stride;
  const int32_t* rows;          // nullable
  const int32_t* seq_lens;      // [B]
  float* ws_o;                  // [B, h_q, max_splits, HD]
  float* ws_lse;                // [B, h_q, max_splits]
  int h_q, h_kv;
  int chunk;                    // tokens per split (multiple of 16)
  int max_splits;
  float scale_log2;             // sm_scale * log2(e)
  // decode-append (nullable): newest token's K/V [B, h_kv, HD] and slot [B];
  // rtt_w is the writable view of rtt for the append
  const __nv_bfloat16* k_new;
  const __nv_bfloat16* v_new;
  const int32_t* new_slots;
  int32_t* rtt_w;
  // cascade: positions [0, kv_start) are attended elsewhere (shared prefix);
  // this kernel covers [kv_start, seq_len) and always writes partials at split
  // index split_base + s of a [B, h_q, max_splits] layout (max_splits includes
  // the split_base shared partials); the merge combines split_base + nsplit_b.
  int kv_start;
  int split_base;
  // nullable: positions < stable_lens[b] were written before the decode phase (by plain-launched
  // kernels) and may be read before the programmatic-dependency wait
  const int32_t* stable_lens;
  // multi-query mode (rx_extend with short segments, decode_kernel<..., MULTI>): request b owns
  // query rows qo_indptr[b] .. qo_indptr[b+1] (q / o ragged [N, h_q, HD]) at positions
  // prefix_lens[b] + j; causal inside the segment; CTA z = b * col_tiles + tile of 8 columns
  // (column = row j x GQA head); one split per request (chunk >= every sequence)
  const int32_t* qo_indptr;
  const int32_t* prefix_lens;
  int col_tiles;
  // merge: when > 0, every row has exactly this many partials (multi-query cascade:
  // n_sh shared chunks + 1 suffix split) and seq_lens is not read
  int fixed_splits;
};

struct ExtendParams {
  const int32_t* rtt;
  int64_t rtt_stride;
  const int32_t* rows;
  const int32_t* prefix_lens;
  const int32_t* extend_lens;
  const int32_t* qo_indptr;
  const __nv_bfloat16* k_new;   // [N, h_kv, HD]
  const __nv_bfloat16* v_new;
  __nv_bfloat16* kpool;         // [S, h_kv, HD]
  __nv_bfloat16* vpool;
  __nv_bfloat16* o;             // [N, h_q, HD]
  int h_q, h_kv;
  int64_t num_slots;
  float scale_log2;
  int batch;                    // set by the launcher
  int max_qtiles;               // set by the launcher
  // Cascade (shared-prefix) mode: the `batch` rows are decode queries of B requests
  // that share cached prefix positions [0, prefix_lens[0]) (slots of table row
  // rows[0]); no new tiles, no causal mask.  The prefix is cut into n_kv_splits
  // chunks of kv_split_tiles tiles; each (q tile, kv head, chunk) item writes a
  // normalized fp32 partial o and its log2-domain lse at split index
  // part_base + chunk of the [B, h_q, part_splits] partial arrays.
  int cascade;
  int kv_split_tiles;
  int n_kv_splits;
  float* part_o;                // [B, h_q, part_splits, HD]
  float* part_lse;              // [B, h_q, part_splits]
  int part_splits;
  int part_base;
  int cas_prefix;               // shared prefix length (cascade mode; prefix_lens unused)
  // cascade partials launched as a programmatic dependent of the suffix decode: the grid may
  // start before that decode completes (it reads only the shared prefix); its epilogue waits for
  // the decode (hence the previous step's merge) before writing partials, and one thread per CTA
  // waits before exiting, so the merge that waits on this grid also sees the decode's partials
  int pdl;
  int* sched;                   // [2] work counters: the caller's workspace header (kWsHeader)
};

struct DecodePlan {
  int chunk;
  int max_splits;
};

// Split-KV plan: a fixed function of (batch, h_kv, max_seq_len) only — NOT of
// the device's SM count — so a P-GPU run and the same shards run one after
// another on one GPU partition identically (SURVEY §8(e) "fake TP").
inline DecodePlan plan_decode(int batch, int h_kv, int max_seq_len) {
  const int64_t units = int64_t(batch) * h_kv;
  const int64_t target_ctas = 8 * 148;
  int64_t chunk = (units * max_seq_len + target_ctas - 1) / target_ctas;
  chunk = chunk < 256 ? 256 : chunk;
  chunk = (chunk + 63) / 64 * 64;
  if (chunk > max_seq_len) chunk = (int64_t(max_seq_len) + 15) / 16 * 16;
  if (chunk < 16) chunk = 16;
  const int max_splits = int((max_seq_len + chunk - 1) / chunk);
  return {int(chunk), max_splits};
}

inline size_t decode_ws_bytes(int h_q, int head_dim, int batch, int max_seq_len, int h_kv) {
  DecodePlan pl = plan_decode(batch, h_kv, max_seq_len);
  if (pl.max_splits <= 1) return 0;
  const size_t n = size_t(batch) * h_q * pl.max_splits;
  return kWsHeader + n * head_dim * sizeof(float) + n * sizeof(float) + 256;
}

// Cascade plan (shared-prefix decode): the shared prefix [0, shared_len) is cut
// into n_sh chunks of kv_split_tiles 128-token tiles so that (q tiles x kv heads
// x chunks) gives ~2 items per SM of a 148-SM part (a constant, not the device's
// count); the suffix [shared_len, seq_len) follows the ordinary split plan.
struct CascadePlan {
  int n_sh;
  int kv_split_tiles;
  DecodePlan suffix;
  int total_splits;
};

// Items per SM the shared-prefix split aims at (extend items are handed out dynamically, so more,
// smaller items trade per-item overhead for a shorter tail).  RX_CASCADE_IPS overrides (A/B knob).
inline int cascade_items_per_sm() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RX_CASCADE_IPS");
    v = e ? atoi(e) : 2;
    if (v < 1 || v > 32) v = 2;
  }
  return v;
}

inline CascadePlan plan_cascade(int batch, int h_kv, int group, int max_seq_len, int shared_len) {
  CascadePlan c{};
  const int tok = 128 / group;
  const int qt = (batch + tok - 1) / tok;
  const int tiles = (shared_len + 127) / 128;
  const int per_chunk = qt * h_kv;
  int n = (cascade_items_per_sm() * 148 + per_chunk - 1) / per_chunk;
  n = n < 1 ? 1 : (n > tiles ? tiles : n);
  c.kv_split_tiles = (tiles + n - 1) / n;
  c.n_sh = (tiles + c.kv_split_tiles - 1) / c.kv_split_tiles;
  c.suffix = plan_decode(batch, h_kv, max_seq_len - shared_len);
  c.total_splits = c.n_sh + c.suffix.max_splits;
  return c;
}

inline size_t cascade_ws_bytes(int h_q, int head_dim, int batch, int h_kv, int max_seq_len, int shared_len) {
  CascadePlan c = plan_cascade(batch, h_kv, h_q / h_kv, max_seq_len, shared_len);
  const size_t n = size_t(batch) * h_q * c.total_splits;
  return kWsHeader + n * head_dim * sizeof(float) + n * sizeof(float) + 256;
}

cudaError_t launch_store_kv(int64_t n, int row_bytes, const int32_t* slots, const void* k, const void* v,
                            void* kpool, void* vpool, int32_t* rtt, const int64_t* rtt_idx, cudaStream_t st);
cudaError_t launch_extend_store(int64_t n, int batch, int row_bytes, const int32_t* qo, const int32_t* ext,
                                const int32_t* prefix, const int32_t* rows, const int32_t* rtt, int64_t rtt_stride,
                                const void* k, const void* v, void* kpool, void* vpool, cudaStream_t st);
cudaError_t launch_decode_merge(int head_dim, const DecodeParams& p, int batch, cudaStream_t st);
int pdl_on();   // RX_PDL knob (decode.cu)
cudaError_t launch_extend_cascade(int head_dim, int G, const ExtendParams& p, const void* q, int batch,
                                  cudaStream_t st);
cudaError_t launch_decode(int head_dim, int G, const DecodeParams& p, int batch, cudaStream_t st, int* launches);
cudaError_t launch_decode_multi(int head_dim, int G, const DecodeParams& p, int batch, cudaStream_t st);
cudaError_t launch_extend(int head_dim, int G, const ExtendParams& p, const void* q, int64_t total_new, int batch,
                          int max_ext, cudaStream_t st);

}  // namespace rx
