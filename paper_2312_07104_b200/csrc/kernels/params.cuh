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

// Stream-K partition of the cascade work: W = units x tiles pair-tiles over
// `ctas` virtual CTAs; virtual CTA c owns the pair-tiles [cut(c), cut(c+1)), cut(c) = c W / ctas,
// split at unit boundaries into segments; a unit's segments are numbered by the virtual CTA that
// owns them, from the CTA that holds its first tile.  Shared by the host plan and the kernel.
__host__ __device__ inline int64_t cas_cut(int64_t c, int64_t W, int64_t ctas) { return c * W / ctas; }
__host__ __device__ inline int cas_cta_of(int64_t x, int64_t W, int64_t ctas) {
  return int(((x + 1) * ctas - 1) / W);     // the virtual CTA whose range holds pair-tile x
}
__host__ __device__ inline int cas_parts(int u, int tiles, int64_t W, int64_t ctas) {
  return cas_cta_of(int64_t(u + 1) * tiles - 1, W, ctas) - cas_cta_of(int64_t(u) * tiles, W, ctas) + 1;
}

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

// TP peer-memory all-gather (tp.cu): buffer header = int64 flags [kTpMaxRanks] + an int32 CTA
// counter, padded to kTpHeader bytes; two slots of world x cap bytes follow.
constexpr int kTpMaxRanks = 8;
constexpr int64_t kTpHeader = 256;

// Where a call's final bf16 output rows go (rx_decode_append_tp, include/rx.h section 3): n == 0
// -> the call's own o [rows, h_q, HD]; n > 0 -> row b, local head h of EVERY destination ptr[i]
// (each rank's gathered buffer, peer-mapped) at b * row_stride + (head_off + h) * HD: the TP
// all-gather done by the epilogue's stores.
struct OutSpec {
  __nv_bfloat16* ptr[kTpMaxRanks];
  int n;
  int head_off;
  int64_t row_stride;     // elements per gathered row (h_q_total * HD)
};

// Store a value of type T (bf16, or a packed pair) at head dim d of output row b, local head hq.
template <typename T>
__device__ __forceinline__ void out_put(const OutSpec& os, __nv_bfloat16* o, int h_q, int hd, int64_t b, int hq,
                                        int d, T v) {
  if (os.n == 0) {
    *reinterpret_cast<T*>(o + (b * h_q + hq) * hd + d) = v;
    return;
  }
  const int64_t off = b * os.row_stride + int64_t(os.head_off + hq) * hd + d;
#pragma unroll 1
  for (int i = 0; i < os.n; ++i) *reinterpret_cast<T*>(os.ptr[i] + off) = v;
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
  // with stable_lens: release the dependent grid only after this CTA's streaming (the cascade
  // chain, whose next kernel needs whole SMs), not as soon as every CTA has started
  int late_trigger;
  // multi-query mode (rx_extend with short segments, decode_kernel<..., MULTI>): request b owns
  // query rows qo_indptr[b] .. qo_indptr[b+1] (q / o ragged [N, h_q, HD]) at positions
  // prefix_lens[b] + j; causal inside the segment; CTA z = b * col_tiles + tile of 8 columns
  // (column = row j x GQA head); one split per request (chunk >= every sequence)
  const int32_t* qo_indptr;
  const int32_t* prefix_lens;
  int col_tiles;
  OutSpec out;                  // final output rows (non-MULTI); n == 0: o
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
  // Cascade (shared-prefix) mode: the `batch` rows (decode queries, or every new token of a
  // jump-forward step) share cached prefix positions [0, cas_prefix) (slots of table row rows[0]);
  // no new tiles, no causal mask.  Work = units (q-tile pair, kv head), kv head major, x tiles of
  // the prefix, partitioned stream-K over cas_ctas virtual CTAs (cas_cut above); each segment
  // writes a normalized fp32 partial o and its log2-domain lse at part index `segment number` of
  // the [batch, h_q, part_splits] partial arrays; the merge kernel that follows combines a row's
  // cas_parts segment partials with its suffix partials at part indices n_sh .. n_sh + suffix
  // splits (written by the kernel launched before the shared pass) into bf16 o.
  int cascade;
  int cas_ctas;
  int cas_tiles;
  int n_sh;                     // max segments of a unit = first suffix part index
  float* part_o;                // [B, h_q, part_splits, HD]
  float* part_lse;              // [B, h_q, part_splits]
  int part_splits;
  int cas_prefix;               // shared prefix length (cascade mode; prefix_lens unused)
  // suffix partials per row: cas_fixed_suffix if > 0, else ceil((cas_seq_lens[row] - cas_kv_start)
  // / cas_chunk) (the decode split plan)
  int cas_fixed_suffix;
  const int32_t* cas_seq_lens;
  int cas_kv_start;
  int cas_chunk;
  // cascade launched as a programmatic dependent of the suffix decode: the grid may start before
  // that decode completes (it reads only the shared prefix); its epilogue waits for the decode
  // (hence the previous step, whose reads of the workspace are done) before writing partials
  int pdl;
  int* sched;                   // [2] work counters: the caller's workspace header (kWsHeader)
  OutSpec out;                  // cascade merge output rows (decode steps); n == 0: o
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

// Cascade plan (shared-prefix decode / jump-forward extend): the shared prefix [0, shared_len) of
// every (q-tile pair, kv head) unit is attended stream-K over `ctas` virtual CTAs (a constant
// multiple of a 148-SM part, not the device's count, so TP shards reproduce on one GPU); the suffix
// [shared_len, seq_len) follows the ordinary decode split plan.
struct CascadePlan {
  int n_sh;            // max segments of a unit (first suffix part index)
  int ctas;
  int tiles;
  int units;
  DecodePlan suffix;
  int total_splits;
};

// Virtual CTAs per SM of the shared-prefix pass (RX_CASCADE_IPS, A/B knob; 1 = one segment range
// per SM of a 148-SM part, every SM busy for the same number of pair-tiles).
inline int cascade_items_per_sm() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RX_CASCADE_IPS");
    v = e ? atoi(e) : 1;
    if (v < 1 || v > 32) v = 1;
  }
  return v;
}

inline CascadePlan plan_cascade(int batch, int h_kv, int group, int max_seq_len, int shared_len) {
  CascadePlan c{};
  const int tok = 128 / group;
  const int qt = (batch + tok - 1) / tok;
  const int qp = (qt + 1) / 2;
  c.units = qp * h_kv;
  c.tiles = (shared_len + 127) / 128;
  const int64_t W = int64_t(c.units) * c.tiles;
  const int64_t want = int64_t(cascade_items_per_sm()) * 148;
  const int64_t most = (W + 1) / 2;            // segments of >= 2 tiles: bounded partial counts
  c.ctas = int(most < want ? most : want);
  // When the units fit the SMs, every CTA gets ONE segment of one unit (ctas = units x k): a
  // second segment per CTA costs another pipeline fill and partial write (C5 step 93 -> 81 us,
  // profiles/r2_kbench_cascade_aligned.txt); RX_CASCADE_ALIGN=0 keeps the plain stream-K cut.
  static int align = -1;
  if (align < 0) {
    const char* e = getenv("RX_CASCADE_ALIGN");
    align = e ? atoi(e) : 1;
  }
  if (align && c.units <= want) {
    const int per = int(want / c.units);
    const int k = per < c.tiles ? per : c.tiles;
    c.ctas = c.units * (k > 0 ? k : 1);
  }
  c.n_sh = 1;
  for (int u = 0; u < c.units; ++u) {
    const int n = cas_parts(u, c.tiles, W, c.ctas);
    c.n_sh = n > c.n_sh ? n : c.n_sh;
  }
  c.suffix = plan_decode(batch, h_kv, max_seq_len - shared_len);
  c.total_splits = c.n_sh + c.suffix.max_splits;
  return c;
}

inline size_t cascade_ws_bytes(int h_q, int head_dim, int batch, int h_kv, int max_seq_len, int shared_len) {
  CascadePlan c = plan_cascade(batch, h_kv, h_q / h_kv, max_seq_len, shared_len);
  const size_t n = size_t(batch) * h_q * c.total_splits;
  return kWsHeader + n * head_dim * sizeof(float) + n * sizeof(float) + 256;
}

cudaError_t launch_copy_h2d(void* dst, const void* src, int64_t bytes, cudaStream_t st);
cudaError_t launch_store_kv(int64_t n, int row_bytes, const int32_t* slots, const void* k, const void* v,
                            void* kpool, void* vpool, int32_t* rtt, const int64_t* rtt_idx, cudaStream_t st);
cudaError_t launch_extend_store(int64_t n, int batch, int row_bytes, const int32_t* qo, const int32_t* ext,
                                const int32_t* prefix, const int32_t* rows, const int32_t* rtt, int64_t rtt_stride,
                                const void* k, const void* v, void* kpool, void* vpool, cudaStream_t st);
int pdl_on();   // RX_PDL knob (decode.cu)
cudaError_t launch_extend_cascade(int head_dim, int G, const ExtendParams& p, const void* q, int batch,
                                  cudaStream_t st);
cudaError_t launch_decode(int head_dim, int G, const DecodeParams& p, int batch, cudaStream_t st, int* launches);
cudaError_t launch_decode_multi(int head_dim, int G, const DecodeParams& p, int batch, cudaStream_t st);
cudaError_t launch_extend(int head_dim, int G, const ExtendParams& p, const void* q, int64_t total_new, int batch,
                          int max_ext, cudaStream_t st);

}  // namespace rx
