// Decode attention over the token-slot KV pool (rx_decode, include/rx.h).
//
// Computes, for each request b and q head h (kv head g = h / G, R14):
//     o = softmax_{i < seq_len}(scale * q . K[rtt[b][i]]) V[rtt[b][i]]
// i.e. one query per request at position seq_len-1 (App. A.1),
// reading the cached prefix through the slot table (one token per page,
// PAPER.md:181 §3).
//
// B200 design (HBM-bound; 2*G FLOP per K/V byte pair):
//  * one CTA per (split, kv head, request); 4 warps each stream their own
//    16-token blocks of the split through a private STAGES-deep cp.async
//    pipeline (16-byte gathers of pool rows by slot, XOR-swizzled smem);
//  * the G query heads of one kv head share every K/V byte (GQA grouping):
//    S^T[16 tok x 8 heads] = K[16 x hd] . Q^T on mma.sync m16n8k16 (heads
//    padded to 8 — G <= 8 so at most 8x waste, still far below the HMMA
//    rate), online softmax in registers, P^T re-fragmented with movmatrix,
//    O^T[hd x 8] += V^T . P^T;
//  * warps merge through shared memory; splits merge by log-sum-exp in a
//    second small kernel (A8), or the CTA writes bf16 output directly when
//    the request has a single split.
//  * MULTI = true: the same kernel for short extends (a jump-forward segment of
//    a few tokens, §4): the 8 MMA columns are (query row j, GQA head h)
//    pairs of one request, each with its own causal limit; one split per
//    request.  Used by rx_extend when every segment fits a few column tiles.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <mutex>
#include <set>
#include <utility>
#include <cstdlib>

#include "params.cuh"
#include "ptx.cuh"

namespace rx {

constexpr int kDecWarps = 4;       // warps per CTA (long splits)
constexpr int kBlk = 16;

// splits of at most this many tokens run 2-warp CTAs (RX_DECODE_SHORT overrides: A/B knob)
static int short_chunk() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RX_DECODE_SHORT");
    v = e ? atoi(e) : 256;
  }
  return v;
}

template <int HD, int STAGES_ = (HD == 128 ? 2 : 6), int WARPS_ = kDecWarps>
struct DecCfg {
  static constexpr int RB = HD * 2;                   // bytes per row
  static constexpr int BLK_BYTES = kBlk * RB;         // one K (or V) block
  static constexpr int STAGES = STAGES_;
  static constexpr int WARPS = WARPS_;
  static constexpr int WARP_BYTES = STAGES * 2 * BLK_BYTES;
  static constexpr int SMEM = WARPS * WARP_BYTES;
  static constexpr int CHUNKS = kBlk * HD / 8;        // 16-byte chunks per block
  static_assert(SMEM >= WARPS * HD * 8 * 4, "merge scratch must fit");
};

// slot > 0: pool row; slot == kNewTok: the step's own new token, read from the k_new / v_new
// argument rows (knew / vnew, this head) — so no CTA has to wait for the pool append; else zeros
constexpr int kNewTok = -2;

template <int HD>
__device__ __forceinline__ void dec_issue_block(uint32_t kdst, uint32_t vdst, const __nv_bfloat16* kpool,
                                                const __nv_bfloat16* vpool, int slot, int h_kv, int g,
                                                const __nv_bfloat16* knew, const __nv_bfloat16* vnew) {
  constexpr int CPR = HD / 8;  // chunks per row
  const int lane = lane_id();
#pragma unroll
  for (int c = 0; c < DecCfg<HD>::CHUNKS / 32; ++c) {
    const int idx = c * 32 + lane;
    const int r = idx / CPR, ch = idx % CPR;
    const int sl = __shfl_sync(0xffffffffu, slot, r);
    const bool ok = sl > 0 || sl == kNewTok;
    const int64_t off = (int64_t(sl > 0 ? sl : 0) * h_kv + g) * HD + ch * 8;
    const uint32_t so = r * DecCfg<HD>::RB + ((ch ^ (r & 7)) << 4);
    cp_async_16(kdst + so, sl == kNewTok ? knew + ch * 8 : kpool + off, ok ? 16u : 0u);
    cp_async_16(vdst + so, sl == kNewTok ? vnew + ch * 8 : vpool + off, ok ? 16u : 0u);
  }
}

template <int HD, int G, int STAGES, bool MULTI = false, int WARPS = kDecWarps>
__global__ void __launch_bounds__(WARPS * 32, 2) decode_kernel(const DecodeParams p) {
  using C = DecCfg<HD, STAGES, WARPS>;
  extern __shared__ __align__(128) uint8_t smem[];
  const int b = MULTI ? int(blockIdx.z) / p.col_tiles : int(blockIdx.z), g = blockIdx.y, s = blockIdx.x;
  // MULTI: this CTA's columns are ct*8 .. ct*8+7 of the request's nq*G (row, head) pairs
  const int ct = MULTI ? int(blockIdx.z) % p.col_tiles : 0;
  const int q0 = MULTI ? p.qo_indptr[b] : b;
  const int nq = MULTI ? p.qo_indptr[b + 1] - q0 : 1;
  if (MULTI && ct * 8 >= nq * G) return;
  const int L = MULTI ? p.prefix_lens[b] + nq : p.seq_lens[b];
  const int start = p.kv_start + s * p.chunk;      // kv_start > 0: cascade (shared prefix elsewhere)
  if (start >= L) return;
  const int end = min(L, start + p.chunk);
  const int nsplit = (L - p.kv_start + p.chunk - 1) / p.chunk;
  const int row = p.rows ? p.rows[b] : b;
  const int32_t* slots = p.rtt + int64_t(row) * p.rtt_stride;

  // Decode-append (rx_decode_append): the newest token's KV arrives with the call.  Position L-1
  // is read from the k_new / v_new argument (kNewTok), and the last split of each (request, kv
  // head) stores that head's row into the pool slot (A5) — for kv head 0 also the slot into the
  // req_to_token row (A4) — at the END, after the dependency wait below.
  const bool append = !MULTI && p.new_slots != nullptr;
  const int new_slot = append ? p.new_slots[b] : 0;
  const __nv_bfloat16* knew_row = append ? p.k_new + (int64_t(b) * p.h_kv + g) * HD : nullptr;
  const __nv_bfloat16* vnew_row = append ? p.v_new + (int64_t(b) * p.h_kv + g) * HD : nullptr;
  // Programmatic dependent launch (launch_decode): this grid may start while the previous decode
  // step / merge still runs.  Positions < stable (written by plain-launched kernels before the
  // decode phase: the prompt) are read at once; everything the previous steps wrote — table
  // entries and K/V of generated positions, the split workspace the previous merge reads — only
  // after griddepcontrol.wait.  stable_lens null: wait before anything.
  const int stable = (MULTI || !p.stable_lens) ? 0 : min(p.stable_lens[b], L - 1);
  bool waited = false;
  auto dep_wait = [&]() {
    if (!waited) {
      pdl_wait();
      waited = true;
    }
  };
  if (stable <= start) dep_wait();
  // with a stable region the next step is released as soon as every CTA has started (it reads only
  // its own stable positions before its wait); without one, after this CTA's streaming (the old
  // schedule: the cascade chain's tcgen05 partial kernel needs whole SMs and must not be delayed)
  const bool early_trigger = !MULTI && p.stable_lens != nullptr && !p.late_trigger;
  if (early_trigger) pdl_launch_dependents();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;

  // Q^T fragments (B operand): b0 = Q[head gq][16kk + 2tq .. +1], b1 = Q[head gq][16kk + 8 + 2tq .. +1]
  uint32_t qf[HD / 16][2];
  {
    // column gq: decode -> head gq of the group (padded past G); MULTI -> row j, head h
    const int cj = MULTI ? (ct * 8 + gq) / G : 0, ch = MULTI ? (ct * 8 + gq) % G : gq;
    const bool qok = MULTI ? cj < nq : gq < G;
    const __nv_bfloat16* qrow = p.q + (int64_t(q0 + (qok ? cj : 0)) * p.h_q + g * G + (qok ? ch : 0)) * HD;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      if (qok) {
        qf[kk][0] = *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 2 * tq);
        qf[kk][1] = *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 8 + 2 * tq);
      } else {
        qf[kk][0] = qf[kk][1] = 0u;
      }
    }
  }

  const uint32_t wbase = smem_u32(smem) + warp * C::WARP_BYTES;
  auto kst = [&](int st) { return wbase + st * 2 * C::BLK_BYTES; };
  auto vst = [&](int st) { return wbase + st * 2 * C::BLK_BYTES + C::BLK_BYTES; };

  const int nblk = (end - start + kBlk - 1) / kBlk;
  const int my = warp < nblk ? (nblk - warp + WARPS - 1) / WARPS : 0;
  auto tok0 = [&](int i) { return start + (warp + i * WARPS) * kBlk; };
  // block i is late if it holds a position >= stable: wait (whole warp) before its table reads
  auto late = [&](int i) { return i < my && tok0(i) + kBlk > stable; };
  auto load_slot = [&](int i) -> int {
    if (late(i)) dep_wait();
    if (i >= my || lane >= kBlk) return 0;
    const int t = tok0(i) + lane;
    return t < end ? ((append && t == L - 1) ? kNewTok : slots[t]) : 0;
  };

#pragma unroll
  for (int st = 0; st < C::STAGES - 1; ++st) {
    const int sl = load_slot(st);
    if (st < my) dec_issue_block<HD>(kst(st), vst(st), p.kpool, p.vpool, sl, p.h_kv, g, knew_row, vnew_row);
    cp_async_commit();
  }
  int slot_pref = load_slot(C::STAGES - 1);

  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  float oacc[HD / 16][4];
#pragma unroll
  for (int mt = 0; mt < HD / 16; ++mt) oacc[mt][0] = oacc[mt][1] = oacc[mt][2] = oacc[mt][3] = 0.f;

  for (int i = 0; i < my; ++i) {
    {
      const int ii = i + C::STAGES - 1;
      if (ii < my) dec_issue_block<HD>(kst(ii % C::STAGES), vst(ii % C::STAGES), p.kpool, p.vpool, slot_pref,
                                       p.h_kv, g, knew_row, vnew_row);
      cp_async_commit();
      slot_pref = load_slot(i + C::STAGES);
    }
    cp_async_wait<C::STAGES - 1>();
    __syncwarp();
    const int st = i % C::STAGES;
    const uint32_t kb = kst(st), vb = vst(st);
    const int nvalid = end - tok0(i);

    float sacc[4] = {0.f, 0.f, 0.f, 0.f};
    {
      const int r = (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        const int ch = 2 * kk + (lane >> 4);
        uint32_t a0, a1, a2, a3;
        ldmatrix_x4(kb + r * C::RB + ((ch ^ (r & 7)) << 4), a0, a1, a2, a3);
        mma_bf16_16816(sacc, a0, a1, a2, a3, qf[kk][0], qf[kk][1]);
      }
    }
    // scale into log2 domain; mask tokens past the end of the split (MULTI: and past each
    // column's own position, causal inside the segment)
    int lim0 = nvalid, lim1 = nvalid;
    if (MULTI) {
      const int base = L - nq - tok0(i);             // position of the segment's first row, block-relative
      lim0 = min(nvalid, base + (ct * 8 + 2 * tq) / G + 1);
      lim1 = min(nvalid, base + (ct * 8 + 2 * tq + 1) / G + 1);
    }
    float s0 = gq < lim0 ? sacc[0] * p.scale_log2 : -INFINITY;
    float s1 = gq < lim1 ? sacc[1] * p.scale_log2 : -INFINITY;
    float s2 = gq + 8 < lim0 ? sacc[2] * p.scale_log2 : -INFINITY;
    float s3 = gq + 8 < lim1 ? sacc[3] * p.scale_log2 : -INFINITY;
    float mx0 = fmaxf(s0, s2), mx1 = fmaxf(s1, s3);
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
    }
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
    // MULTI: a column may meet a fully masked block before any valid key (its running max stays
    // -inf); exponentiate against 0 then, so every factor is 0 instead of NaN
    const float e0 = (MULTI && mn0 == -INFINITY) ? 0.f : mn0;
    const float e1 = (MULTI && mn1 == -INFINITY) ? 0.f : mn1;
    const float c0 = fast_exp2(m0 - e0), c1 = fast_exp2(m1 - e1);
    m0 = mn0;
    m1 = mn1;
    const float p0 = fast_exp2(s0 - e0), p1 = fast_exp2(s1 - e1);
    const float p2 = fast_exp2(s2 - e0), p3 = fast_exp2(s3 - e1);
    l0 = l0 * c0 + p0 + p2;
    l1 = l1 * c1 + p1 + p3;
#pragma unroll
    for (int mt = 0; mt < HD / 16; ++mt) {
      oacc[mt][0] *= c0;
      oacc[mt][1] *= c1;
      oacc[mt][2] *= c0;
      oacc[mt][3] *= c1;
    }
    const uint32_t bx = movmatrix_trans(pack_bf16(p0, p1));
    const uint32_t by = movmatrix_trans(pack_bf16(p2, p3));
    {
      const int m = lane >> 3;
      const int r = (lane & 7) + (m >> 1) * 8;
#pragma unroll
      for (int mt = 0; mt < HD / 16; ++mt) {
        const int ch = 2 * mt + (m & 1);
        uint32_t a0, a1, a2, a3;
        ldmatrix_x4_trans(vb + r * C::RB + ((ch ^ (r & 7)) << 4), a0, a1, a2, a3);
        mma_bf16_16816(oacc[mt], a0, a1, a2, a3, bx, by);
      }
    }
    __syncwarp();
  }
  cp_async_wait<0>();
  dep_wait();   // before writing the output / split workspace and the pool append
  if (!early_trigger) pdl_launch_dependents();
#pragma unroll
  for (int off = 4; off < 32; off <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, off);
    l1 += __shfl_xor_sync(0xffffffffu, l1, off);
  }
  __syncthreads();  // all warps done with their pipelines: reuse smem for the merge

  float* opart = reinterpret_cast<float*>(smem);                  // [warps][HD][8]
  __shared__ float red_m[WARPS][8], red_l[WARPS][8];
  if (gq == 0) {
    red_m[warp][2 * tq] = m0;
    red_m[warp][2 * tq + 1] = m1;
    red_l[warp][2 * tq] = l0;
    red_l[warp][2 * tq + 1] = l1;
  }
  float* ow = opart + warp * HD * 8;
#pragma unroll
  for (int mt = 0; mt < HD / 16; ++mt) {
    const int d = 16 * mt + gq;
    ow[d * 8 + 2 * tq] = oacc[mt][0];
    ow[d * 8 + 2 * tq + 1] = oacc[mt][1];
    ow[(d + 8) * 8 + 2 * tq] = oacc[mt][2];
    ow[(d + 8) * 8 + 2 * tq + 1] = oacc[mt][3];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < (MULTI ? 8 : G) * HD; idx += WARPS * 32) {
    const int h = idx / HD, d = idx % HD;   // MULTI: h is the column
    if (MULTI && (ct * 8 + h) / G >= nq) continue;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) M = fmaxf(M, red_m[w][h]);
    float acc = 0.f, Ls = 0.f;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
      const float f = fast_exp2(red_m[w][h] - M);
      Ls += f * red_l[w][h];
      acc += f * opart[(w * HD + d) * 8 + h];
    }
    if (MULTI) {   // one split; every column saw >= 1 key (key 0, or its own position), so Ls > 0
      const int j = (ct * 8 + h) / G, hq = g * G + (ct * 8 + h) % G;
      if (p.split_base == 0) {
        p.o[(int64_t(q0 + j) * p.h_q + hq) * HD + d] = __float2bfloat16_rn(acc / Ls);
      } else {     // cascade: this is the suffix partial after split_base shared-prefix partials
        const int64_t base = (int64_t(q0 + j) * p.h_q + hq) * p.max_splits + p.split_base;
        p.ws_o[base * HD + d] = acc / Ls;
        if (d == 0) p.ws_lse[base] = M + __log2f(Ls);
      }
      continue;
    }
    const int hq = g * G + h;
    if (nsplit == 1 && p.split_base == 0) {
      out_put(p.out, p.o, p.h_q, HD, b, hq, d, __float2bfloat16_rn(acc / Ls));
    } else {
      const int64_t base = (int64_t(b) * p.h_q + hq) * p.max_splits + p.split_base + s;
      p.ws_o[base * HD + d] = acc / Ls;
      if (d == 0) p.ws_lse[base] = M + __log2f(Ls);
    }
  }
  if (append && s == nsplit - 1) {
    // A5 + A4 of this step (after the dependency wait: the slot may have been freed by a request
    // that finished at the previous step, whose kernel could otherwise still be reading it)
    constexpr int VPR = HD / 8;                      // 16-byte vectors per head row
    const int64_t dst = (int64_t(new_slot) * p.h_kv + g) * HD;
    if (threadIdx.x < VPR)
      reinterpret_cast<uint4*>(const_cast<__nv_bfloat16*>(p.kpool) + dst)[threadIdx.x] =
          reinterpret_cast<const uint4*>(knew_row)[threadIdx.x];
    else if (threadIdx.x < 2 * VPR)
      reinterpret_cast<uint4*>(const_cast<__nv_bfloat16*>(p.vpool) + dst)[threadIdx.x - VPR] =
          reinterpret_cast<const uint4*>(vnew_row)[threadIdx.x - VPR];
    if (g == 0 && threadIdx.x == 2 * VPR) p.rtt_w[int64_t(row) * p.rtt_stride + L - 1] = new_slot;
  }
}

// Log-sum-exp merge of split partials (A8): o = sum_s 2^(lse_s - LSE) o_s.
// One warp per (row, q head), 8 per CTA: each lane owns HD/32 consecutive dims (float2/float4
// reads of every split's partial), the split weights are computed once per warp.
constexpr int kMergeWarps = 8;

template <int HD>
__global__ void __launch_bounds__(kMergeWarps * 32) decode_merge_kernel(const DecodeParams p, int rows) {
  pdl_launch_dependents();   // the next step may be scheduled now: it reads only stable positions
                             // before its own wait (which covers this merge)
  pdl_wait();                // the partials of the preceding grid(s) are complete
  const int lane = threadIdx.x & 31;
  const int64_t pair = int64_t(blockIdx.x) * kMergeWarps + (threadIdx.x >> 5);
  if (pair >= int64_t(rows) * p.h_q) return;
  const int b = int(pair / p.h_q);
  const int nsplit = p.split_base + (p.seq_lens[b] - p.kv_start + p.chunk - 1) / p.chunk;
  if (nsplit <= 1) return;
  const int64_t base = pair * p.max_splits;
  float M = -INFINITY;
  for (int s = lane; s < nsplit; s += 32) M = fmaxf(M, p.ws_lse[base + s]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
  constexpr int V = HD / 32;                       // 4 (hd 128) or 2 (hd 64) floats per lane
  float acc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v] = 0.f;
  float W = 0.f;
  for (int s = 0; s < nsplit; ++s) {
    const float w = fast_exp2(p.ws_lse[base + s] - M);
    W += w;
    const float* src = p.ws_o + (base + s) * HD + lane * V;
    if constexpr (V == 4) {
      const float4 x = *reinterpret_cast<const float4*>(src);
      acc[0] += w * x.x, acc[1] += w * x.y, acc[2] += w * x.z, acc[3] += w * x.w;
    } else {
      const float2 x = *reinterpret_cast<const float2*>(src);
      acc[0] += w * x.x, acc[1] += w * x.y;
    }
  }
  const float inv = 1.f / W;
  const int hq = int(pair - int64_t(b) * p.h_q);
#pragma unroll
  for (int v = 0; v < V; v += 2)
    out_put(p.out, p.o, p.h_q, HD, b, hq, lane * V + v, pack_bf16(acc[v] * inv, acc[v + 1] * inv));
}

static dim3 merge_grid(int rows, int h_q) {
  return dim3(unsigned((int64_t(rows) * h_q + kMergeWarps - 1) / kMergeWarps));
}

// Programmatic dependent launch: decode steps and merges follow each other back to back; with
// programmaticStreamSerialization the next grid is scheduled while the previous one drains (its
// CTAs run their prologue, then griddepcontrol.wait).  RX_PDL=0 launches them plainly (A/B knob).
static bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RX_PDL");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}
int pdl_on() { return pdl_enabled() ? 1 : 0; }

cudaError_t ensure_smem_attr_ptr(const void* kern, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;   // (kernel, device) with the attribute set
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({kern, dev})) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert({kern, dev});
  return e;
}

template <typename Kern, typename... Args>
static cudaError_t launch_pdl(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <int HD, int G, int STAGES>
static cudaError_t launch_decode_t(const DecodeParams& p, int batch, cudaStream_t st, int* launches) {
  dim3 grid(p.max_splits - p.split_base, p.h_kv, batch);   // suffix splits (cascade: shared partials come first)
  cudaError_t e;
  if (p.chunk <= short_chunk()) {
    // short splits (a cascade suffix of ~100-300 tokens, early decode steps): 2 warps per CTA so
    // twice as many CTAs are resident (one wave instead of two or three)
    using C = DecCfg<HD, STAGES, 2>;
    e = ensure_smem_attr(decode_kernel<HD, G, STAGES, false, 2>, C::SMEM);
    if (e != cudaSuccess) return e;
    e = launch_pdl(decode_kernel<HD, G, STAGES, false, 2>, grid, dim3(2 * 32), C::SMEM, st, p);
  } else {
    using C = DecCfg<HD, STAGES>;
    e = ensure_smem_attr(decode_kernel<HD, G, STAGES>, C::SMEM);
    if (e != cudaSuccess) return e;
    e = launch_pdl(decode_kernel<HD, G, STAGES>, grid, dim3(kDecWarps * 32), C::SMEM, st, p);
  }
  if (e != cudaSuccess) return e;
  *launches = 1;
  if (p.max_splits > 1 && p.split_base == 0) {   // cascade: the caller merges after the shared part
    e = launch_pdl(decode_merge_kernel<HD>, merge_grid(batch, p.h_q), dim3(kMergeWarps * 32), 0, st, p, batch);
    if (e != cudaSuccess) return e;
    *launches = 2;
  }
  return cudaPeekAtLastError();
}

template <int HD, int G>
static cudaError_t launch_decode_multi_t(const DecodeParams& p, int batch, cudaStream_t st) {
  constexpr int STG = HD == 64 ? 6 : 2;
  using C = DecCfg<HD, STG>;
  {
    cudaError_t e = ensure_smem_attr(decode_kernel<HD, G, STG, true>, C::SMEM);
    if (e != cudaSuccess) return e;
  }
  dim3 grid(1, p.h_kv, batch * p.col_tiles);
  decode_kernel<HD, G, STG, true><<<grid, kDecWarps * 32, C::SMEM, st>>>(p);
  return cudaPeekAtLastError();
}

cudaError_t launch_decode_multi(int head_dim, int G, const DecodeParams& p, int batch, cudaStream_t st) {
#define RX_DEC_CASE(HD_, G_) \
  if (head_dim == HD_ && G == G_) return launch_decode_multi_t<HD_, G_>(p, batch, st);
  RX_DEC_CASE(64, 1) RX_DEC_CASE(64, 2) RX_DEC_CASE(64, 4) RX_DEC_CASE(64, 8)
  RX_DEC_CASE(128, 1) RX_DEC_CASE(128, 2) RX_DEC_CASE(128, 4) RX_DEC_CASE(128, 8)
#undef RX_DEC_CASE
  return cudaErrorInvalidValue;
}

// Pipeline depth per warp for head_dim 128: 2 (default: 64 KB smem, 3 CTAs/SM;
// measured 6.38 TB/s in the C3 step vs 5.96 for 3 stages / 2 CTAs per SM).  RX_DECODE_STAGES overrides it (development A/B knob).
static int decode_stages() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RX_DECODE_STAGES");
    v = e ? atoi(e) : 2;
    if (v != 2 && v != 3 && v != 4) v = 2;
  }
  return v;
}

cudaError_t launch_decode(int head_dim, int G, const DecodeParams& p, int batch, cudaStream_t st,
                          int* launches) {
  const int stg = decode_stages();
#define RX_DEC_CASE(HD_, G_)                                                                  \
  if (head_dim == HD_ && G == G_) {                                                           \
    if (HD_ == 64) return launch_decode_t<HD_, G_, 6>(p, batch, st, launches);                \
    if (stg == 4) return launch_decode_t<HD_, G_, 4>(p, batch, st, launches);                 \
    if (stg == 3) return launch_decode_t<HD_, G_, 3>(p, batch, st, launches);                 \
    return launch_decode_t<HD_, G_, 2>(p, batch, st, launches);                               \
  }
  RX_DEC_CASE(64, 1) RX_DEC_CASE(64, 2) RX_DEC_CASE(64, 4) RX_DEC_CASE(64, 8)
  RX_DEC_CASE(128, 1) RX_DEC_CASE(128, 2) RX_DEC_CASE(128, 4) RX_DEC_CASE(128, 8)
#undef RX_DEC_CASE
  return cudaErrorInvalidValue;
}

}  // namespace rx
