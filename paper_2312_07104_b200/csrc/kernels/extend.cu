// Extend attention (prefill with radix-prefix reuse) on tcgen05 / TMEM (rx_extend).
//
// Computes, for request b, new token j (absolute position p = prefix_len + j)
// and q head h (kv head g = h / G, R14):
//     o = softmax_{i <= p}(scale * q . K[i]) V[i]
// where K/V rows 0..prefix_len-1 are the CACHED prefix, read from the pool
// through rtt ("reduces the computation of prefill"), and
// rows prefix_len.. are this call's k_new/v_new (read directly; rx_extend
// stores them into their pool slots with a separate launch, A5).
//
// B200 design — persistent, one CTA (12 warps) per SM, work items handed out
// dynamically; an item is (PAIR of q tiles A, B; kv head g; request b):
//  * M = 128 rows per q tile = (128/G tokens) x (G heads of one kv group): GQA
//    packing makes every K/V tile byte serve G heads (R14).  Tiles A and B are
//    consecutive token ranges of the same (b, g), so every K/V tile staged in
//    shared memory feeds two 128-row MMAs (half the L2 -> SMEM traffic per
//    FLOP of a one-tile CTA);
//  * TMEM (512 columns) = S_A | S_B | O_A | O_B: two score tiles and two
//    output accumulators, all fp32;
//  * two softmax warpgroups (warps 4-7: tile A, warps 8-11: tile B; thread =
//    TMEM lane = row) ping-pong on the tensor core: the MMA warp issues, per
//    K/V tile j, O_A += P_A(j-1) V(j-1), S_A(j) = Q_A K(j)^T, then the same for
//    B, so the tensor core computes one tile's GEMMs while the other tile's
//    warpgroup runs its softmax.  Issue order makes the TMEM reuse safe (the
//    MMA pipe executes in order) and makes S_x(j) complete only after
//    O_x += P_x(j-1) V(j-1), so the softmax may rescale O_x in TMEM as soon as
//    it sees S_x(j) (lazy rescale: only when a row max grows by > 8 in log2);
//  * warp 0 = item scheduler + K producer (it takes the next work index just
//    before the CTA needs it and publishes a descriptor ring in shared memory),
//    warp 3 = Q + V producer: cached-prefix K/V by one
//    3-D TMA box per 64 columns when the tile's 128 slots are consecutive (the
//    smallest-first allocator makes that common for prompt tokens), else
//    16-byte cp.async gathers written straight into the 128B-swizzled layout;
//    new K/V by 3-D TMA boxes; K 2-deep and V 3-deep rings (hd 128);
//  * warp 1 = single-thread tcgen05.mma issuer; warp 2 = TMEM owner;
//  * setmaxnreg moves registers from the producer warpgroup (64 each) to the
//    softmax warpgroups (216 each: a whole 128-column S row lives in registers);
//  * A5 (store new K/V into their slots) is a separate, fully parallel kernel
//    launched just before on the same stream (store.cu).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "params.cuh"
#include "ptx.cuh"

namespace rx {

struct ExtendMaps {
  CUtensorMap q;       // 3D (HD, h_q, N)   box (64, G, TOK)
  CUtensorMap knew;    // 3D (HD, h_kv, N)  box (64, 1, 128)
  CUtensorMap vnew;
  CUtensorMap kpool;   // 3D (HD, h_kv, S)  box (64, 1, 128)
  CUtensorMap vpool;
};

constexpr int kExtThreads = 384;    // 12 warps: 4 producer/MMA/scheduler + 2 softmax warpgroups
constexpr int kProducerRegs = 64;   // setmaxnreg budget of warps 0-3
constexpr int kSoftmaxRegs = 216;   // ... and of warps 4-11 (64*128 + 216*256 <= 168*384)
constexpr int kBN = 128;            // kv tokens per tile
constexpr int kTileRowBytes = 128;  // 64 bf16 per swizzled row

template <int HD>
struct ExtCfg {
  static constexpr int NCB = HD / 64;                          // 64-column blocks
  static constexpr int TILE_BYTES = NCB * 128 * kTileRowBytes;  // one 128-row tile (Q, K or V)
  // K_j is released as soon as both S = Q K_j^T retire, V_j only after both P V_j; V(j) is
  // fetched when PV(j - VS) retires and needed at PV(j), so gathered (cp.async) V tiles need the
  // deeper ring: KS 2 / VS 3 measured 787 vs 738 TFLOP/s (KS 3 / VS 2) on half-fragmented C3
  // histories, and 996 vs 955 on contiguous ones (hd 128).
  static constexpr int KS = HD == 128 ? 2 : 4;
  static constexpr int VS = HD == 128 ? 3 : 3;
  static constexpr int SMEM_DATA = (2 + KS + VS) * TILE_BYTES;  // Q_A, Q_B, K ring, V ring
  static constexpr int SMEM = SMEM_DATA + 1024 /*align*/ + 1024 /*barriers + item ring*/;
  static constexpr uint32_t TMEM_COLS = 512;                    // S_A | S_B | O_A | O_B
  static constexpr uint32_t O_COL = 256;                        // O_x at O_COL + x*HD
};
static_assert(ExtCfg<128>::SMEM <= 232448, "extend kernel exceeds the 227 KB opt-in shared memory");

// One work item = (q tiles t0 and t0+1, kv head g, request b); every role of a CTA walks the
// same list.  n[x] = K/V tiles q tile x attends to (0: tile x is past the request's rows).
struct ExtItem {
  int b, g, t0, P, ext, qo, n_pre;
  int n[2];
  int tile0;            // first prefix tile (cascade segment), 0 otherwise
  int split;            // cascade: segment number within its unit (= partial index)
  int unit;             // cascade: (q-tile pair, kv head) unit
  const int32_t* slots;
};

// Item ring: warp 0 resolves the CTA's work items and publishes descriptors in shared memory;
// the 10 consumer warps (MMA, Q/V producer, 8 softmax) read them.
constexpr int kRing = 2;
constexpr int kRingConsumers = 10;

struct RingCursor {
  int slot = 0;
  uint32_t phase = 0;
};

// all lanes of the calling warp read the descriptor; `arrive` marks the lane that releases it
__device__ __forceinline__ bool ring_pop(ExtItem& I, RingCursor& c, const ExtItem* ring, uint64_t* full,
                                         uint64_t* empty, bool arrive) {
  mbar_wait(full + c.slot, c.phase);
  I = ring[c.slot];
  if (arrive) mbar_arrive(empty + c.slot);
  if (++c.slot == kRing) {
    c.slot = 0;
    c.phase ^= 1;
  }
  return I.b >= 0;
}

template <int TOK>
__device__ __forceinline__ bool ext_item(const ExtendParams& p, int qp, int w, ExtItem& it) {
  // (request, kv head) outer, q-tile pair inner (heaviest first): the pairs of one (b, g) run
  // on neighbouring CTAs at the same time, so that head's cached prefix is read from HBM once
  // and re-served from L2.
  const int pair = qp - 1 - w % qp;
  it.t0 = 2 * pair;
  it.tile0 = 0;
  it.split = 0;
  it.unit = 0;
  const int bg = w / qp;
  it.g = bg % p.h_kv;
  it.b = bg / p.h_kv;
  it.ext = p.extend_lens[it.b];
  if (it.t0 * TOK >= it.ext) return false;
  it.P = p.prefix_lens[it.b];
  it.qo = p.qo_indptr[it.b];
  const int row = p.rows ? p.rows[it.b] : it.b;
  it.slots = p.rtt + int64_t(row) * p.rtt_stride;
  it.n_pre = (it.P + kBN - 1) / kBN;
#pragma unroll
  for (int x = 0; x < 2; ++x) {
    const int t = it.t0 + x;
    const int rel_end = min(it.ext, (t + 1) * TOK);
    it.n[x] = t * TOK < it.ext ? it.n_pre + (rel_end + kBN - 1) / kBN : 0;
  }
  return true;
}

// Cascade (shared-prefix) segment: pair-tiles [x, xe) of virtual CTA c, cut at the end of unit
// u = x / tiles (kv head major: u = g * qp + pair).  Returns the end of the segment.
template <int TOK>
__device__ __forceinline__ int64_t cas_segment(const ExtendParams& p, int qp, int c, int64_t x, int64_t xe,
                                               int64_t W, ExtItem& it) {
  const int T = p.cas_tiles;
  const int u = int(x / T);
  const int64_t end = min(xe, int64_t(u + 1) * T);
  it.unit = u;
  it.g = u / qp;
  it.t0 = 2 * (u % qp);
  it.b = 0;
  it.ext = p.batch;
  it.P = p.cas_prefix;
  it.qo = 0;
  const int row = p.rows ? p.rows[0] : 0;
  it.slots = p.rtt + int64_t(row) * p.rtt_stride;
  it.tile0 = int(x - int64_t(u) * T);
  it.n_pre = int(end - x);
  it.n[0] = it.n_pre;
  it.n[1] = (it.t0 + 1) * TOK < it.ext ? it.n_pre : 0;
  it.split = c - cas_cta_of(int64_t(u) * T, W, p.cas_ctas);
  return end;
}

// Where the rows of K/V tile j of item I come from, resolved BEFORE the producer waits for a free
// ring stage (the slot-index loads then overlap that wait): a prefix tile whose 128 slots are
// consecutive is one 3-D TMA box per 64 columns (`tma`, starting at slot s0); a fragmented prefix
// tile is gathered row by row (slot_r[i] = slot of row lane + 32 i, -1 past the prefix); a
// new-KV tile is a TMA box of k_new / v_new.
struct TileSrc {
  bool tma;
  int s0;
  int slot_r[4];
};

__device__ __forceinline__ TileSrc probe_kv_tile(const ExtItem& I, int j, int lane) {
  TileSrc t;
  t.tma = true;
  t.s0 = 0;
  if (j < I.n_pre) {
    const int jt = I.tile0 + j;                   // absolute prefix tile (cascade chunks)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int pos = jt * kBN + lane + 32 * i;
      t.slot_r[i] = pos < I.P ? I.slots[pos] : -1;
    }
    t.s0 = __shfl_sync(0xffffffffu, t.slot_r[0], 0);   // (jt*kBN < P: the tile has >= 1 cached row)
    bool contig = true;
#pragma unroll
    for (int i = 0; i < 4; ++i) contig &= t.slot_r[i] == t.s0 + lane + 32 * i;
    t.tma = __all_sync(0xffffffffu, contig);
  }
  return t;
}

// One K or V tile j of item I into ring stage at smem address d (warp-collective; lane 0 issues
// TMA).  Gathers are per-lane 16-byte cp.async written straight into the 128B-swizzled layout
// (chunk k of row r -> chunk k ^ (r & 7)), rows past the prefix zero-filled.  Every lane arrives
// on `full` (TMA: lane 0 with expect_tx, others plainly; cp.async: .noinc arrivals).
template <int HD>
__device__ __forceinline__ void load_kv_tile(const ExtItem& I, int j, const TileSrc& t, uint32_t d, uint64_t* full,
                                             const CUtensorMap* m_pool, const CUtensorMap* m_new,
                                             const __nv_bfloat16* base_g, int h_kv, int lane) {
  using C = ExtCfg<HD>;
  if (t.tma) {
    if (lane == 0) {
      mbar_arrive_expect_tx(full, C::TILE_BYTES);
      if (j < I.n_pre) {
#pragma unroll
        for (int c = 0; c < C::NCB; ++c) tma_load_3d(d + c * kBN * kTileRowBytes, m_pool, full, c * 64, I.g, t.s0);
      } else {
        const int nn = j - I.n_pre;
#pragma unroll
        for (int c = 0; c < C::NCB; ++c)
          tma_load_3d(d + c * kBN * kTileRowBytes, m_new, full, c * 64, I.g, I.qo + nn * kBN);
      }
    } else {
      mbar_arrive(full);
    }
  } else {
    // lane pair (2k, 2k+1) owns rows k + 16 i (i = 0..7), lane parity picks the 16-byte chunks of
    // a row: one warp instruction moves 16 rows x 32 contiguous bytes (whole sectors), and per row
    // a lane computes one source and one destination base — the 16-byte pieces of a row go out
    // with immediate source offsets (a tile is ~160 instructions per warp, not ~1700)
    constexpr int CPR = HD / 8;                       // 16-byte chunks per row
    const int par = lane & 1, rl = lane >> 1;
    const int kx = (rl & 7) ^ par;                    // swizzle: chunk c of row r -> c ^ (r & 7)
#pragma unroll
    for (int i = 0; i < kBN / 16; ++i) {
      const int row = rl + 16 * i;                    // (row & 7) == (rl & 7)
      const int sl = __shfl_sync(0xffffffffu, t.slot_r[i >> 1], rl + 16 * (i & 1));
      const bool ok = sl > 0;
      const char* src = reinterpret_cast<const char*>(base_g + (int64_t(ok ? sl : 0) * h_kv + I.g) * HD) + par * 16;
      const uint32_t drow = d + row * kTileRowBytes;
#pragma unroll
      for (int m = 0; m < CPR / 2; ++m) {             // chunk c = 2m + par
        const uint32_t dst = drow + ((2 * m) >> 3) * kBN * kTileRowBytes + ((((2 * m) & 7) ^ kx) << 4);
        cp_async_16(dst, src + 32 * m, ok ? 16u : 0u);
      }
    }
    cp_async_mbar_arrive_noinc(full);
  }
}

// exp2 of one half (64 columns) of a score row, its row-sum contribution (two packed fp32-pair
// accumulators), and P (bf16 pairs) into the first 32 TMEM columns of that half's S columns.
// Packed FFMA2 / FADD2 do the scale-subtract, the sums and the polynomial two columns per issue
// slot (the softmax warps are issue-bound).  MUFU ex2 is the other limiter (16/clk/SM vs 8192 MMA
// FLOP/clk): with POLY (an unmasked tile) every 4th column pair is evaluated on the FMA pipe
// instead (exp2_poly3; masked tiles need exact zeros, so MUFU only).
#ifndef RX_EXT_POLY_EVERY
#define RX_EXT_POLY_EVERY 4     // every RX_EXT_POLY_EVERY-th column pair on the FMA pipe (A/B build knob)
#endif

template <bool POLY>
__device__ __forceinline__ void softmax_half(const float* sv, int half, float sc, float nm, uint64_t* rs,
                                             uint32_t t_s) {
  uint32_t pk[kBN / 4];
  const uint64_t sc2 = f2_pack(sc, sc), nm2 = f2_pack(nm, nm);
#pragma unroll
  for (int c = 0; c < kBN / 4; ++c) {
    const int col = half * (kBN / 2) + 2 * c;
    float x0, x1, e0, e1;
    f2_unpack(f2_fma(f2_pack(sv[col], sv[col + 1]), sc2, nm2), x0, x1);
    if (POLY && c % RX_EXT_POLY_EVERY == RX_EXT_POLY_EVERY - 1) {
      exp2_poly3_x2(x0, x1, e0, e1);
    } else {
      e0 = fast_exp2(x0);
      e1 = fast_exp2(x1);
    }
    rs[c & 1] = f2_add(rs[c & 1], f2_pack(e0, e1));
    pk[c] = pack_bf16(e0, e1);
  }
  tmem_st32(t_s + half * 32, pk);
}

template <int HD, int G>
__global__ void __launch_bounds__(kExtThreads, 1)
    extend_kernel(const ExtendParams p, const __grid_constant__ ExtendMaps maps) {
  using C = ExtCfg<HD>;
  constexpr int TOK = 128 / G;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sq = smem_u32(smem);                 // Q tile x at sq + x*TILE_BYTES
  const uint32_t sk = sq + 2 * C::TILE_BYTES;         // K stage s at sk + s*TILE_BYTES
  const uint32_t sv_ = sk + C::KS * C::TILE_BYTES;    // V stage s at sv_ + s*TILE_BYTES
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::SMEM_DATA);
  uint64_t* q_full = bars;                            // [2] per q tile x
  uint64_t* q_empty = bars + 2;                       // [2]
  uint64_t* k_full = bars + 4;                        // [KS]
  uint64_t* k_empty = k_full + C::KS;                 // [KS]
  uint64_t* v_full = k_empty + C::KS;                 // [VS]
  uint64_t* v_empty = v_full + C::VS;                 // [VS]
  uint64_t* s_full = v_empty + C::VS;                 // [2] S_x(j) landed (one phase per tile of x)
  uint64_t* p_full = s_full + 2;                      // [2] P_x(j) written (128 arrivals)
  uint64_t* o_ready = p_full + 2;                     // [2] O_x final (one phase per item of x)
  uint64_t* desc_full = o_ready + 2;                  // [kRing] item descriptors published
  uint64_t* desc_empty = desc_full + kRing;           // [kRing] ... and consumed by the 10 other warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(desc_empty + kRing);
  ExtItem* ring = reinterpret_cast<ExtItem*>(smem + C::SMEM_DATA + 512);

  const int qp = (p.max_qtiles + 1) / 2;              // q-tile pairs per (b, g)
  const int W = qp * p.h_kv * p.batch;                // work indices (non-cascade)
  const int64_t Wc = int64_t(qp) * p.h_kv * p.cas_tiles;   // cascade pair-tiles
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(q_full + i, 1);
      mbar_init(q_empty + i, 1);
      mbar_init(s_full + i, 1);
      mbar_init(p_full + i, 128);
      mbar_init(o_ready + i, 1);
    }
    for (int s = 0; s < C::KS; ++s) {
      mbar_init(k_full + s, 32);   // all producer lanes arrive (TMA: 1 expect_tx + 31; cp.async: 32 noinc)
      mbar_init(k_empty + s, 1);
    }
    for (int s = 0; s < C::VS; ++s) {
      mbar_init(v_full + s, 32);
      mbar_init(v_empty + s, 1);
    }
    for (int i = 0; i < kRing; ++i) {
      mbar_init(desc_full + i, 1);
      mbar_init(desc_empty + i, kRingConsumers);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ item scheduler + K producer
    // Items are handed out dynamically from the work counter in the caller's workspace, so ragged
    // batches (items of 1..N tiles, some q tiles absent) balance across SMs.  This warp takes the
    // next work index only once it has issued every K load of its current item, i.e. just before
    // the CTA needs it: consecutive indices (the q-tile pairs of one (b, g)) then start within a
    // short window on different SMs and share that head's cached prefix through L2 (fetching
    // further ahead spreads their start times over an item's duration, and the prefix is evicted
    // between them: measured 2x the DRAM bytes on fragmented C3 histories).  Descriptors go to
    // the other warps through the ring.
    regs_dealloc<kProducerRegs>();
    if (lane == 0) {
      tma_prefetch_desc(&maps.knew);
      tma_prefetch_desc(&maps.kpool);
    }
    RingCursor c;
    auto publish = [&](const ExtItem& it) {
      mbar_wait(desc_empty + c.slot, c.phase ^ 1);
      if (lane == 0) {
        ring[c.slot] = it;
        mbar_arrive(desc_full + c.slot);
      }
      __syncwarp();
      if (++c.slot == kRing) {
        c.slot = 0;
        c.phase ^= 1;
      }
    };
    int cas_c = -1;                     // cascade: current virtual CTA and its remaining range
    int64_t cas_x = 0, cas_xe = 0;
    auto next = [&](ExtItem& it) -> bool {
      if (p.cascade) {
        if (cas_x >= cas_xe) {
          int c = 0;
          if (lane == 0) c = atomicAdd(&p.sched[0], 1);
          cas_c = __shfl_sync(0xffffffffu, c, 0);
          if (cas_c >= p.cas_ctas) return false;
          cas_x = cas_cut(cas_c, Wc, p.cas_ctas);
          cas_xe = cas_cut(cas_c + 1, Wc, p.cas_ctas);
        }
        cas_x = cas_segment<TOK>(p, qp, cas_c, cas_x, cas_xe, Wc, it);
        return true;
      }
      for (;;) {
        int w = 0;
        if (lane == 0) w = atomicAdd(&p.sched[0], 1);
        w = __shfl_sync(0xffffffffu, w, 0);
        if (w >= W) return false;
        if (ext_item<TOK>(p, qp, w, it)) return true;
      }
    };
    int jg = 0;
    ExtItem I;
    bool have = next(I);
    while (have) {
      publish(I);
      const int N = max(I.n[0], I.n[1]);
      for (int j = 0; j < N; ++j, ++jg) {
        const int st = jg % C::KS, rnd = jg / C::KS;
        const TileSrc t = probe_kv_tile(I, j, lane);
        mbar_wait(k_empty + st, (rnd & 1) ^ 1);
        load_kv_tile<HD>(I, j, t, sk + st * C::TILE_BYTES, k_full + st, &maps.kpool, &maps.knew, p.kpool, p.h_kv,
                         lane);
      }
      have = next(I);
    }
    ExtItem stop{};
    stop.b = -1;
    publish(stop);
  } else if (warp == 3) {
    // ------------------------------------------------------------ Q + V producer
    regs_dealloc<kProducerRegs>();
    if (lane == 0) {
      tma_prefetch_desc(&maps.q);
      tma_prefetch_desc(&maps.vnew);
      tma_prefetch_desc(&maps.vpool);
    }
    int jg = 0, itq0 = 0, itq1 = 0;
    ExtItem I;
    RingCursor rc;
    while (ring_pop(I, rc, ring, desc_full, desc_empty, lane == 0)) {
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        if (I.n[x] == 0) continue;
        int& itq = x ? itq1 : itq0;
        if (itq > 0) mbar_wait(q_empty + x, (itq - 1) & 1);   // the previous item's last S_x retired
        if (lane == 0) {
          mbar_arrive_expect_tx(q_full + x, C::TILE_BYTES);
#pragma unroll
          for (int c = 0; c < C::NCB; ++c)
            tma_load_3d(sq + x * C::TILE_BYTES + c * 128 * kTileRowBytes, &maps.q, q_full + x, c * 64, I.g * G,
                        I.qo + (I.t0 + x) * TOK);
        }
        ++itq;
      }
      const int N = max(I.n[0], I.n[1]);
      for (int j = 0; j < N; ++j, ++jg) {
        const int st = jg % C::VS, rnd = jg / C::VS;
        const TileSrc t = probe_kv_tile(I, j, lane);
        mbar_wait(v_empty + st, (rnd & 1) ^ 1);
        load_kv_tile<HD>(I, j, t, sv_ + st * C::TILE_BYTES, v_full + st, &maps.vpool, &maps.vnew, p.vpool, p.h_kv,
                         lane);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp walks the loop (converged, warp-uniform operands); one elected lane issues
    // each tcgen05.mma / commit.  Per K/V tile j and q tile x: O_x += P_x(j-1) V(j-1), then
    // S_x(j) = Q_x K(j)^T — the ping-pong order (see the header).
    regs_dealloc<kProducerRegs>();
    constexpr uint32_t idesc_s = umma_idesc_bf16(128, kBN, false, false);
    constexpr uint32_t idesc_o = umma_idesc_bf16(128, HD, false, true);
    // Shared-memory descriptors are built once; advancing one by a byte offset inside the (< 227
    // KB) shared window is an add of offset >> 4 to its 14-bit start-address field (no carry).
    const uint64_t dq0 = umma_desc_sw128(sq, 16, 1024);                       // Q_x, K stages: K-major
    const uint64_t dk0 = umma_desc_sw128(sk, 16, 1024);
    const uint64_t dv0 = umma_desc_sw128(sv_, kBN * kTileRowBytes, 1024);     // V stages: MN-major
    int jg = 0, jx0 = 0, jx1 = 0, itx0 = 0, itx1 = 0;
    ExtItem I;
    RingCursor rc;
    while (ring_pop(I, rc, ring, desc_full, desc_empty, lane == 0)) {
      const int n0 = __shfl_sync(0xffffffffu, I.n[0], 0);   // uniform for ptxas
      const int n1 = __shfl_sync(0xffffffffu, I.n[1], 0);
      const int N = max(n0, n1);
      for (int j = 0; j <= N; ++j) {
        const int kg = jg + j;                    // K tile j (global ring index)
        if (j < N) {
          mbar_wait(k_full + kg % C::KS, (kg / C::KS) & 1);
          tc_fence_after();
          fence_proxy_async();                    // cp.async (generic proxy) writes -> the MMA (async proxy)
        }
        bool v_ready = false;
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          const int nx = x ? n1 : n0;
          if (nx == 0) continue;
          const int jx = x ? jx1 : jx0;
          const uint32_t t_s = tmem + x * 128;
          if (j > 0 && j <= nx) {
            // O_x += P_x(j-1) V(j-1), P read from TMEM (A operand), V from the ring
            mbar_wait(p_full + x, (jx + j - 1) & 1);
            const int vg = kg - 1;
            if (!v_ready) {
              mbar_wait(v_full + vg % C::VS, (vg / C::VS) & 1);
              v_ready = true;
              tc_fence_after();
              fence_proxy_async();
            } else {
              tc_fence_after();
            }
            const uint64_t dv = dv0 + uint32_t(((vg % C::VS) * C::TILE_BYTES) >> 4);
            if (elect_one()) {
#pragma unroll
              for (int k = 0; k < kBN / 16; ++k)
                umma_ts(tmem + C::O_COL + x * HD, t_s + k * 8, dv + uint32_t((k * 2048) >> 4), idesc_o,
                        (j > 1 || k > 0) ? 1u : 0u);
              if (j == nx) tc_commit(o_ready + x);        // O_x final for this item
            }
            __syncwarp();
          }
          if (j < nx) {
            if (j == 0) {
              mbar_wait(q_full + x, (x ? itx1 : itx0) & 1);
              tc_fence_after();
            }
            const uint64_t dq = dq0 + uint32_t((x * C::TILE_BYTES) >> 4);
            const uint64_t dk = dk0 + uint32_t(((kg % C::KS) * C::TILE_BYTES) >> 4);
            if (elect_one()) {
#pragma unroll
              for (int k = 0; k < HD / 16; ++k) {
                const uint32_t off = uint32_t(((k >> 2) * 128 * kTileRowBytes + (k & 3) * 32) >> 4);
                umma_ss(t_s, dq + off, dk + off, idesc_s, k > 0);
              }
              tc_commit(s_full + x);
              if (j == nx - 1) tc_commit(q_empty + x);      // last read of Q_x issued
            }
            __syncwarp();
          }
        }
        if (elect_one()) {
          if (j < N) tc_commit(k_empty + kg % C::KS);       // K(j) free once both S(j) retire
          if (j > 0) tc_commit(v_empty + (kg - 1) % C::VS);  // V(j-1) free once both P V(j-1) retire
        }
        __syncwarp();
      }
      jg += N;
      jx0 += n0;
      jx1 += n1;
      itx0 += n0 > 0;
      itx1 += n1 > 0;
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax + epilogue of q tile x
    regs_alloc<kSoftmaxRegs>();
    const int x = (warp - 4) >> 2;
    const int r = (warp & 3) * 32 + lane;          // row = TMEM lane
    const int i_tok = r / G, h = r % G;
    const uint32_t lane_off = uint32_t((warp & 3) * 32) << 16;
    const uint32_t t_s = tmem + lane_off + x * 128;
    const uint32_t t_o = tmem + lane_off + C::O_COL + x * HD;
    int jx = 0, itx = 0;
    ExtItem I;
    RingCursor rc;
    while (ring_pop(I, rc, ring, desc_full, desc_empty, lane == 0)) {
      const int nx = I.n[x];
      if (nx == 0) continue;
      const int rel = (I.t0 + x) * TOK + i_tok;     // position relative to prefix_len
      float m_ref = -INFINITY, l = 0.f;
      for (int j = 0; j < nx; ++j, ++jx) {
        mbar_wait(s_full + x, jx & 1);
        tc_fence_after();
        float sv[kBN];
#pragma unroll
        for (int c = 0; c < kBN / 32; ++c) tmem_ld32(t_s + c * 32, sv + c * 32);
        tmem_ld_wait();
        // mask: prefix tile -> col < P - j*BN ; new tile -> nn*BN + col <= rel.
        // Scores stay raw (unscaled); the scale is folded into the exp2 FFMA.
        const int lim = j < I.n_pre ? I.P - (I.tile0 + j) * kBN - 1 : rel - (j - I.n_pre) * kBN;
        const bool full = __all_sync(0xffffffffu, lim >= kBN - 1);   // warp-uniform
        if (!full) {
#pragma unroll
          for (int c = 0; c < kBN; ++c) sv[c] = c <= lim ? sv[c] : -INFINITY;
        }
        // row max over 128 columns as 8 independent chains
        float mxp[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) mxp[k] = fmaxf(sv[k], sv[k + 8]);
#pragma unroll
        for (int c = 16; c < kBN; c += 16)
#pragma unroll
          for (int k = 0; k < 8; ++k) mxp[k] = fmaxf(mxp[k], fmaxf(sv[c + k], sv[c + k + 8]));
        float mx = fmaxf(fmaxf(fmaxf(mxp[0], mxp[1]), fmaxf(mxp[2], mxp[3])),
                         fmaxf(fmaxf(mxp[4], mxp[5]), fmaxf(mxp[6], mxp[7])));
        mx *= p.scale_log2;
        // Lazy rescale, decided per WARP (tcgen05.ld/st are warp-collective).  S_x(j) retired,
        // and it was issued after O_x += P_x(j-1) V(j-1), so O_x is complete up to j-1.
        if (__any_sync(0xffffffffu, mx > m_ref + 8.f) || j == 0) {
          const float m_new = fmaxf(mx, m_ref);
          const float corr = fast_exp2(m_ref - m_new);
          if (j > 0) {
#pragma unroll
            for (int c = 0; c < HD / 32; ++c) {
              float ov[32];
              tmem_ld32(t_o + c * 32, ov);
              tmem_ld_wait();
              uint32_t ou[32];
#pragma unroll
              for (int e = 0; e < 32; ++e) ou[e] = __float_as_uint(ov[e] * corr);
              tmem_st32(t_o + c * 32, ou);
            }
          }
          l *= corr;
          m_ref = m_new;
        }
        uint64_t rs[2] = {0ull, 0ull};                    // 2 packed (4 scalar) row-sum chains
        const float sc = p.scale_log2, nm = -m_ref;
        if (full) {
          softmax_half<true>(sv, 0, sc, nm, rs, t_s);
          softmax_half<true>(sv, 1, sc, nm, rs, t_s);
        } else {
          softmax_half<false>(sv, 0, sc, nm, rs, t_s);
          softmax_half<false>(sv, 1, sc, nm, rs, t_s);
        }
        float r0, r1, r2, r3;
        f2_unpack(rs[0], r0, r1);
        f2_unpack(rs[1], r2, r3);
        l += (r0 + r1) + (r2 + r3);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(p_full + x);
      }
      // epilogue: O_x complete once this item's last P V landed
      mbar_wait(o_ready + x, itx & 1);
      ++itx;
      if (p.pdl) pdl_wait();   // cascade partials: the previous step's merge must be done reading them
      tc_fence_after();
      const float inv = 1.f / l;
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {
        float ov[32];
        tmem_ld32(t_o + c * 32, ov);
        tmem_ld_wait();
        if (p.cascade) {
          // partial over this segment: normalized fp32 o + log2-domain lse
          if (rel < I.ext) {
            const int64_t pr = (int64_t(rel) * p.h_q + I.g * G + h) * p.part_splits + I.split;
            float4* dst = reinterpret_cast<float4*>(p.part_o + pr * HD + c * 32);
#pragma unroll
            for (int e = 0; e < 8; ++e)
              dst[e] = make_float4(ov[4 * e] * inv, ov[4 * e + 1] * inv, ov[4 * e + 2] * inv, ov[4 * e + 3] * inv);
            if (c == 0) p.part_lse[pr] = m_ref + __log2f(l);
          }
        } else if (rel < I.ext) {
          __nv_bfloat16* orow = p.o + (int64_t(I.qo + rel) * p.h_q + I.g * G + h) * HD;
          uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            uint4 v;
            v.x = pack_bf16(ov[8 * e + 0] * inv, ov[8 * e + 1] * inv);
            v.y = pack_bf16(ov[8 * e + 2] * inv, ov[8 * e + 3] * inv);
            v.z = pack_bf16(ov[8 * e + 4] * inv, ov[8 * e + 5] * inv);
            v.w = pack_bf16(ov[8 * e + 6] * inv, ov[8 * e + 7] * inv);
            dst[e] = v;
          }
        }
      }
      // O_x is read: the next item's first P V into O_x is issued only after this warpgroup's
      // next p_full arrival (the fence orders these TMEM reads before it)
      tc_fence_before();
    }
  } else {
    // ------------------------------------------------------------ warp 2: TMEM owner only
    regs_dealloc<kProducerRegs>();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, C::TMEM_COLS);
  if (p.pdl && threadIdx.x == 0) pdl_wait();   // see ExtendParams::pdl
  // Dynamic work distribution: p.sched[0] = next work index, [1] = CTAs finished, in the caller's
  // workspace header (params.cuh kWsHeader).  Every fetch of this CTA is done: the last CTA resets
  // both, so the workspace is zero again for the next call that uses it.
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&p.sched[1], 1) == int(gridDim.x) - 1) {
      p.sched[0] = 0;
      p.sched[1] = 0;
      __threadfence();
    }
  }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

static bool make_map(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                     const uint32_t* box) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t d[5], s[4];
  cuuint32_t bx[5], es[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    bx[i] = box[i];
    es[i] = 1;
  }
  for (int i = 0; i < rank - 1; ++i) s[i] = strides_bytes[i];
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), d, s, bx, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Pool tensor maps (3-D (HD, h_kv, S), box (64, 1, 128)) depend only on the pool: encoded once and
// reused (a decode run issues a cascade step every ~30 us; cuTensorMapEncodeTiled costs ~1-2 us of
// host time each).  Small per-thread cache keyed by (base, slots, h_kv, HD).
static bool pool_map(CUtensorMap* m, const void* base, uint64_t slots, int h_kv, int hd) {
  struct Ent {
    const void* base;
    uint64_t slots;
    int h_kv, hd;
    CUtensorMap map;
  };
  static thread_local Ent cache[4];
  static thread_local int next = 0;
  for (const Ent& e : cache)
    if (e.base == base && e.slots == slots && e.h_kv == h_kv && e.hd == hd) {
      *m = e.map;
      return true;
    }
  uint64_t dims[3] = {uint64_t(hd), uint64_t(h_kv), slots};
  uint64_t str[2] = {uint64_t(hd) * 2, uint64_t(h_kv) * hd * 2};
  uint32_t box[3] = {64, 1, 128};
  if (!make_map(m, base, 3, dims, str, box)) return false;
  cache[next] = Ent{base, slots, h_kv, hd, *m};
  next = (next + 1) & 3;
  return true;
}

template <int HD, int G>
static cudaError_t launch_extend_t(const ExtendParams& p, const void* q, int64_t total_new, int batch,
                                   int max_ext, cudaStream_t st) {
  // cascade mode: `batch` virtual rows (decode queries), one virtual request; no
  // new tiles (the k_new / v_new maps are encoded over the pools, never used)
  using C = ExtCfg<HD>;
  constexpr int TOK = 128 / G;
  ExtendMaps mp;
  const uint64_t hd = HD;
  const uint64_t N = total_new > 0 ? uint64_t(total_new) : 1;
  {
    uint64_t dims[3] = {hd, uint64_t(p.h_q), N};
    uint64_t str[2] = {hd * 2, uint64_t(p.h_q) * hd * 2};
    uint32_t box[3] = {64, uint32_t(G), uint32_t(TOK)};
    if (!make_map(&mp.q, q, 3, dims, str, box)) return cudaErrorInvalidValue;
  }
  if (!pool_map(&mp.kpool, p.kpool, uint64_t(p.num_slots), p.h_kv, HD) ||
      !pool_map(&mp.vpool, p.vpool, uint64_t(p.num_slots), p.h_kv, HD))
    return cudaErrorInvalidValue;
  if (p.cascade) {   // no new tiles in cascade mode: the new-KV maps are never used
    mp.knew = mp.kpool;
    mp.vnew = mp.vpool;
  } else {
    uint64_t dims[3] = {hd, uint64_t(p.h_kv), N};
    uint64_t str[2] = {hd * 2, uint64_t(p.h_kv) * hd * 2};
    uint32_t box[3] = {64, 1, kBN};
    if (!make_map(&mp.knew, p.k_new, 3, dims, str, box)) return cudaErrorInvalidValue;
    if (!make_map(&mp.vnew, p.v_new, 3, dims, str, box)) return cudaErrorInvalidValue;
  }
  {
    cudaError_t e = ensure_smem_attr(extend_kernel<HD, G>, C::SMEM);
    if (e != cudaSuccess) return e;
  }
  if (!p.sched) return cudaErrorInvalidValue;
  ExtendParams pp = p;
  pp.batch = batch;
  pp.max_qtiles = (max_ext + TOK - 1) / TOK;
  const int64_t qpairs = (pp.max_qtiles + 1) / 2;
  const int64_t items = p.cascade ? int64_t(p.cas_ctas) : qpairs * p.h_kv * batch;
  const int sms = device_sms();
  const int grid = int(items < sms ? items : sms);   // persistent: one CTA per SM
  if (p.pdl) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kExtThreads);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, extend_kernel<HD, G>, pp, mp);
  }
  extend_kernel<HD, G><<<grid, kExtThreads, C::SMEM, st>>>(pp, mp);
  return cudaPeekAtLastError();
}

// Log-sum-exp merge of the cascade partials (A8): row `row`, q head hq (one warp, lanes over the
// head dims) combines its unit's stream-K segment partials [0, parts) and its suffix partials
// [n_sh, n_sh + ns) into bf16 o.  Launched right after the shared-prefix pass (programmatic
// dependent: it waits for that grid, and through it for the suffix kernel, before reading).
constexpr int kCasMergeWarps = 8;

template <int HD>
__global__ void __launch_bounds__(kCasMergeWarps * 32) cascade_merge_kernel(const ExtendParams p, int rows, int G) {
  pdl_launch_dependents();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t pair = int64_t(blockIdx.x) * kCasMergeWarps + (threadIdx.x >> 5);
  if (pair >= int64_t(rows) * p.h_q) return;
  const int row = int(pair / p.h_q), hq = int(pair % p.h_q);
  const int tok = 128 / G;
  const int qp = (p.max_qtiles + 1) / 2;
  const int unit = (hq / G) * qp + (row / tok) / 2;
  const int64_t Wc = int64_t(qp) * p.h_kv * p.cas_tiles;
  const int parts = cas_parts(unit, p.cas_tiles, Wc, p.cas_ctas);
  const int ns = p.cas_fixed_suffix > 0 ? p.cas_fixed_suffix
                                        : (p.cas_seq_lens[row] - p.cas_kv_start + p.cas_chunk - 1) / p.cas_chunk;
  const int nk = parts + ns;
  const int64_t base = pair * p.part_splits;
  auto idx = [&](int k) { return k < parts ? k : p.n_sh + (k - parts); };
  // lane k holds partial k's lse (32 at a time): one load instruction for every lse of the row, the
  // weights by warp reductions, then the partials' float4s with up to 8 loads in flight per lane
  constexpr int V = HD / 32;                       // 4 (hd 128) or 2 (hd 64) floats per lane
  float M = -INFINITY;
  for (int k0 = 0; k0 < nk; k0 += 32)
    M = fmaxf(M, k0 + lane < nk ? p.part_lse[base + idx(k0 + lane)] : -INFINITY);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
  float acc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v] = 0.f;
  float W = 0.f;
  for (int k0 = 0; k0 < nk; k0 += 32) {
    const float wl = k0 + lane < nk ? fast_exp2(p.part_lse[base + idx(k0 + lane)] - M) : 0.f;
    float ws = wl;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ws += __shfl_xor_sync(0xffffffffu, ws, off);
    W += ws;
    const int n = min(32, nk - k0);
#pragma unroll 8
    for (int k = 0; k < n; ++k) {
      const float w = __shfl_sync(0xffffffffu, wl, k);
      const float* src = p.part_o + (base + idx(k0 + k)) * HD + lane * V;
      if constexpr (V == 4) {
        const float4 x = *reinterpret_cast<const float4*>(src);
        acc[0] += w * x.x, acc[1] += w * x.y, acc[2] += w * x.z, acc[3] += w * x.w;
      } else {
        const float2 x = *reinterpret_cast<const float2*>(src);
        acc[0] += w * x.x, acc[1] += w * x.y;
      }
    }
  }
  const float inv = 1.f / W;
#pragma unroll
  for (int v = 0; v < V; v += 2)
    out_put(p.out, p.o, p.h_q, HD, row, hq, lane * V + v, pack_bf16(acc[v] * inv, acc[v + 1] * inv));
}

template <int HD>
static cudaError_t launch_cascade_merge(const ExtendParams& p, int rows, int G, cudaStream_t st) {
  ExtendParams pp = p;
  pp.max_qtiles = (rows + 128 / G - 1) / (128 / G);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned((int64_t(rows) * p.h_q + kCasMergeWarps - 1) / kCasMergeWarps));
  cfg.blockDim = dim3(kCasMergeWarps * 32);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, cascade_merge_kernel<HD>, pp, rows, G);
}

cudaError_t launch_extend_cascade(int head_dim, int G, const ExtendParams& p, const void* q, int batch,
                                  cudaStream_t st) {
  if (batch <= 0 || p.cas_prefix <= 0) return cudaSuccess;
  cudaError_t e = cudaSuccess;
#define RX_EXT_CASE(HD_, G_)                                                            \
  if (head_dim == HD_ && G == G_) {                                                     \
    e = launch_extend_t<HD_, G_>(p, q, batch, batch, batch, st);                        \
    if (e != cudaSuccess) return e;                                                     \
    return launch_cascade_merge<HD_>(p, batch, G, st);                                  \
  }
  RX_EXT_CASE(64, 1) RX_EXT_CASE(64, 2) RX_EXT_CASE(64, 4) RX_EXT_CASE(64, 8)
  RX_EXT_CASE(128, 1) RX_EXT_CASE(128, 2) RX_EXT_CASE(128, 4) RX_EXT_CASE(128, 8)
#undef RX_EXT_CASE
  return cudaErrorInvalidValue;
}

cudaError_t launch_extend(int head_dim, int G, const ExtendParams& p, const void* q, int64_t total_new, int batch,
                          int max_ext, cudaStream_t st) {
  if (max_ext <= 0 || batch <= 0) return cudaSuccess;
#define RX_EXT_CASE(HD_, G_) \
  if (head_dim == HD_ && G == G_) return launch_extend_t<HD_, G_>(p, q, total_new, batch, max_ext, st);
  RX_EXT_CASE(64, 1) RX_EXT_CASE(64, 2) RX_EXT_CASE(64, 4) RX_EXT_CASE(64, 8)
  RX_EXT_CASE(128, 1) RX_EXT_CASE(128, 2) RX_EXT_CASE(128, 4) RX_EXT_CASE(128, 8)
#undef RX_EXT_CASE
  return cudaErrorInvalidValue;
}

}  // namespace rx

