/*
 * rx.h — C ABI of the B200-native RadixAttention hot path (arXiv 2312.07104).
 *
 * Citations: "P:n" = PAPER.md line n (section in brackets), "S:n" = SPEC.md
 * line n, "R<k>" = reading k of DESIGN.md "Readings".
 *
 * Two halves behind one library (librx.so):
 *
 *  1. a host radix tree over a token-slot pool (rx_cache_*, rx_match_prefix,
 *     rx_insert, rx_inc_ref, rx_dec_ref, rx_evict, rx_alloc, rx_free, ...):
 *     the paper's "radix tree to manage a mapping between sequences of tokens,
 *     and their corresponding KV cache tensors" stored "in a non-contiguous,
 *     paged layout, where the size of each page is equivalent to one token"
 *     (P:180-181 [§3]); the tree "is stored on the CPU" (P:187 [§3]).
 *     Pure host code; callable without a GPU.
 *
 *  2. device kernels over that pool (rx_store_kv, rx_extend, rx_decode):
 *     causal attention of new tokens over "cached prefix + new KV" (extend,
 *     prefill reuse, P:171, P:359 [§3, §6]) and of one token per request
 *     (decode, P:495 [App. A.1]).  sm_100a only.  Asynchronous on the given
 *     stream; the caller owns every device buffer and the stream; the library
 *     never allocates device memory.
 *
 * Conventions
 *  - Every call returns rx_status (0 = RX_OK, negative = error); no C++
 *    exception crosses the ABI.  A failed call has no side effect unless
 *    stated otherwise.
 *  - Device pointers are marked d_, host pointers h_ (or unmarked for the
 *    host-only tree calls).  bf16 buffers are passed as void*.
 *  - Slot 0 of the pool is reserved as the padding sink (never allocated), so
 *    allocatable slots are 1 .. num_slots-1.
 *  - rx_cache is single-writer, not thread-safe.
 *  - A launch failure is reported as RX_E_CUDA (cudaPeekAtLastError);
 *    asynchronous device faults surface at the caller's next synchronisation.
 */
#ifndef RX_H_
#define RX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RX_OK = 0,
  RX_E_INVALID = -1,      /* bad argument (null pointer, negative size, out-of-range slot, ...) */
  RX_E_NOMEM = -2,        /* rx_alloc: fewer free slots than requested (no side effect) */
  RX_E_UNDERFLOW = -3,    /* rx_dec_ref would drive a reference count below 0 */
  RX_E_STALE = -4,        /* node handle no longer names a live node */
  RX_E_UNSUPPORTED = -5,  /* attention shape outside what the kernels implement */
  RX_E_CUDA = -6,         /* a CUDA launch / driver call failed */
  RX_E_WORKSPACE = -7,    /* workspace too small: query rx_*_workspace_bytes */
  RX_E_CAPACITY = -8      /* a host output buffer is too small */
} rx_status;

/* Human-readable name of a status code (static string). */
const char* rx_status_str(int status);

/* Library build identification (static string): arch, build flags. */
const char* rx_version(void);

/* ======================================================================= */
/*  1. Radix tree + token-slot pool (host)                                  */
/* ======================================================================= */

typedef struct rx_cache rx_cache;

/* A node handle is the node's creation id (root = 0).  Ids are never reused,
 * and a split keeps the id on the LOWER half (R4), so a handle stays valid
 * until its node is evicted; a pinned node (ref > 0) is never evicted. */
typedef int64_t rx_node;

/* Create a tree + pool of num_slots token slots (num_slots >= 1; slot 0 is
 * reserved).  One object owns both because "cached tokens and the currently
 * running requests share the same memory pool" (P:184 [§3]).
 * *out receives the new object; RX_E_INVALID if num_slots < 1 or out null. */
rx_status rx_cache_create(int64_t num_slots, rx_cache** out);
void rx_cache_destroy(rx_cache* c);

/* Alg. 1 T.match_prefix (P:527 [App. A.2]).
 * Longest prefix of tokens[0..n) present in the tree.  If the match ends in
 * the middle of an edge the edge is split there (R3, R4).  The LRU clock ticks
 * once and every node on the matched path is stamped (R1).
 *   *node        deepest matched node (0 = root when nothing matches)
 *   *matched_len number of matched tokens
 *   slots_out    host int32[>= n]; receives the slots of the matched prefix
 *                in position order (may be null).
 * Never fails on content; empty tree or n == 0 -> (root, 0). */
rx_status rx_match_prefix(rx_cache* c, const int32_t* tokens, int64_t n,
                          rx_node* node, int64_t* matched_len, int32_t* slots_out);

/* Alg. 1 T.insert (P:564 [App. A.2]).
 * Cache tokens[0..n) with their slots[0..n).  Ownership of ALL passed slots
 * moves to the cache: positions already cached keep the tree's slots, and a
 * passed slot that differs there is freed, in position order (R10).
 * The clock ticks once; the walked path and the new leaf are stamped (R1, R9).
 *   *new_cached  tokens added to the tree (n minus the already-cached prefix)
 *   *dup_freed   passed slots returned to the free pool (may be null) */
rx_status rx_insert(rx_cache* c, const int32_t* tokens, const int32_t* slots, int64_t n,
                    int64_t* new_cached, int64_t* dup_freed);

/* Alg. 1 T.increase_ref_counter / decrease_ref_counter;
 * SPEC S:131-139.  +/-1 on every node from `node` up to (excluding) the root.
 * *d_evictable receives the change of rx_evictable_size (<= 0 for inc,
 * >= 0 for dec).  RX_E_UNDERFLOW (no side effect) if a count would go below
 * 0; RX_E_STALE for an evicted node. */
rx_status rx_inc_ref(rx_cache* c, rx_node node, int64_t* d_evictable);
rx_status rx_dec_ref(rx_cache* c, rx_node node, int64_t* d_evictable);

/* Eviction callback: one call per evicted leaf, in eviction order, with that
 * leaf's slots in position order (already returned to the free pool). */
typedef void (*rx_evict_cb)(void* user, const int32_t* slots, int64_t n);

/* "evicts the least recently used leaf first" (P:182 [§3]); Alg. 1 T.evict
 * (P:554).  Removes whole leaves with ref 0 in
 * (last_access, id) order (R2, R5); a parent left childless with ref 0
 * becomes a candidate.  Stops when >= needed tokens were evicted or no
 * candidate remains (falling short is NOT an error: compare *evicted).
 * cb may be null. */
rx_status rx_evict(rx_cache* c, int64_t needed, int64_t* evicted, rx_evict_cb cb, void* user);

/* rx_evict with the evicted leaf's token PATH: cb(user, path, path_len,
 * leaf_start, slots, n) where path[0..path_len) are the tokens from the root
 * to the end of the evicted leaf and the leaf owned path[leaf_start..path_len)
 * (n = path_len - leaf_start slots).  Same eviction order and effects as
 * rx_evict.  This is what a data-parallel worker reports to the router's
 * eviction queue (App. A.4). */
typedef void (*rx_evict_path_cb)(void* user, const int32_t* path, int64_t path_len, int64_t leaf_start,
                                 const int32_t* slots, int64_t n);
rx_status rx_evict_paths(rx_cache* c, int64_t needed, int64_t* evicted, rx_evict_path_cb cb, void* user);

/* Token-slot pool.  rx_alloc returns the n smallest free slots in ascending
 * order into out[0..n) (R8), or RX_E_NOMEM with no side effect.
 * rx_free returns slots to the pool (RX_E_INVALID on a slot out of range or
 * already free; then nothing is freed). */
rx_status rx_alloc(rx_cache* c, int64_t n, int32_t* out);
rx_status rx_free(rx_cache* c, const int32_t* slots, int64_t n);

/* Alg. 1 lines 551-556 with reading R6: try rx_alloc(n); on
 * RX_E_NOMEM evict the shortfall (n - available) and retry once.
 * *evicted receives the tokens evicted (0 if none; may be null); cb as in
 * rx_evict.  Returns RX_E_NOMEM if the retry still fails (the eviction is
 * NOT undone). */
rx_status rx_alloc_evict(rx_cache* c, int64_t n, int32_t* out, int64_t* evicted,
                         rx_evict_cb cb, void* user);

/* Batched forms for a whole scheduling step (one C call instead of one per
 * request; same semantics as calling the single-request function for
 * b = 0 .. batch-1 in order, including the clock ticks).  Request b's tokens
 * are tokens[offsets[b] .. offsets[b+1]) (offsets: int64 [batch+1]).
 *   rx_match_prefix_batch: nodes[b], matched[b]; slots_out (may be null) uses
 *     the same layout as tokens and receives each request's matched slots.
 *   rx_inc_ref_batch: deltas[b] (may be null) = Δevictable of request b.
 *   rx_finish_batch: Alg. 1 "process finished requests":
 *     rx_dec_ref(nodes[b]) then rx_insert(tokens_b, slots_b) for each b;
 *     slots has the same layout as tokens; d_evict[b], new_cached[b],
 *     dup_freed[b] may be null.
 * On an error the call stops at the failing request and returns its status;
 * requests before it have been processed. */
rx_status rx_match_prefix_batch(rx_cache* c, int32_t batch, const int32_t* tokens, const int64_t* offsets,
                                rx_node* nodes, int64_t* matched, int32_t* slots_out);
rx_status rx_inc_ref_batch(rx_cache* c, int32_t batch, const rx_node* nodes, int64_t* deltas);
rx_status rx_finish_batch(rx_cache* c, int32_t batch, const rx_node* nodes, const int32_t* tokens,
                          const int64_t* offsets, const int32_t* slots, int64_t* d_evict,
                          int64_t* new_cached, int64_t* dup_freed);

/* Cache-aware admission: Alg. 1 lines P:522-547 (§3 "Cache-aware scheduling",
 * P:214-219) for one scheduling step, in one call.
 *  1. rx_match_prefix_batch over the waiting queue (request b = prompt
 *     tokens[offsets[b] .. offsets[b+1]), length >= 1, in arrival order) ->
 *     nodes[b], matched[b], slots_out (nullable, same layout as tokens).
 *  2. Order the queue by `policy`:
 *       RX_SCHED_LSPF   longest matched prefix first ("longest-shared-prefix-
 *                       first"; optimal by Theorem 1),
 *                       ties by arrival;
 *       RX_SCHED_FCFS   arrival order (ablation);
 *       RX_SCHED_RANDOM ascending keys[b] (uint64, caller-drawn: the random
 *                       numbers are an input), ties by arrival (ablation).
 *  3. Admit in that order while size_b + current < available + delta_b
 *     (strict), available = evictable + free grown by each
 *     admitted request's rx_inc_ref delta, delta_b = request b's
 *     own pin delta (reading R25: b is pinned, tested, and unpinned again if
 *     it does not fit), current += size_b (reading R7),
 *     size_b = (n_b - min(matched_b, n_b - 1)) + max_new[b] (R7, R11).
 *     Admitted requests stay pinned (rx_inc_ref on nodes[b]).
 * Outputs: admitted[0 .. *n_admitted) = request indices in admission order
 * (caller capacity >= batch); deltas[k] (nullable) = inc_ref delta of the
 * k-th admitted request.  Nothing is allocated: the caller allocates the
 * batch's slots (rx_alloc_evict) and later calls rx_finish_batch.
 * Errors: RX_E_INVALID for a null required pointer, an empty prompt, a
 * negative max_new, an unknown policy, or RANDOM without keys (checked before
 * any side effect); a tree error stops the call and is returned. */
typedef enum { RX_SCHED_LSPF = 0, RX_SCHED_FCFS = 1, RX_SCHED_RANDOM = 2 } rx_sched_policy;
rx_status rx_schedule(rx_cache* c, int32_t batch, const int32_t* tokens, const int64_t* offsets,
                      const int64_t* max_new, int32_t policy, const uint64_t* keys, rx_node* nodes,
                      int64_t* matched, int32_t* slots_out, int32_t* admitted, int32_t* n_admitted,
                      int64_t* deltas);

/* Pure queries (Alg. 1 "T.evictable_size() + P.available_size()", P:534;
 * SPEC S:149-156).  evictable = tokens on non-root nodes with ref 0 (pins
 * propagate to the root, so these are exactly the peelable nodes). */
/* Alg. 1's output loop (§3) for PLAIN decoding — one new token per running
 * request per iteration — planned on the host for up to max_steps iterations in one call (the
 * generated tokens are inputs, so no iteration waits for the device).  Iteration k:
 *   1. B = *n_running; if the next record does not fit in out (4·B words past those already used)
 *      the call returns early;
 *   2. alloc B slots (R6: on RX_E_NOMEM evict the shortfall B - rx_available and retry
 *      once; RX_E_NOMEM again is returned and iteration k is not planned);
 *   3. in batch order (R23) request b = running[j] gets slot j: table[b·stride + cur[b]] = slot,
 *      cur[b] += 1, and the step's record [new slots | seq_lens (= new cur) | rows b | stable[b]]
 *      (int32, B words each — the layout rx_decode_append takes from one staging buffer) is
 *      written at out + step_meta[3k+1]; step_meta[3k] = B, step_meta[3k+2] = max seq_len;
 *   4. every request with cur[b] == end[b] finishes: rx_dec_ref(nodes[b]) then
 *      rx_insert(tokens[offsets[b] .. offsets[b] + end[b]), table row b) — batch order — and
 *      leaves running (kept ascending, compacted in place).
 * State (caller-owned host arrays, updated in place): table int32 [batch, stride] (the host mirror
 * of req_to_token), cur int32 [batch], running int32 [*n_running] (ascending request indices).
 * Inputs: end int32 [batch] (prompt + output length, <= stride, <= the request's token count),
 * stable int32 [batch] (copied into records), nodes [batch] (pinned prefix nodes), tokens/offsets
 * (int64 [batch+1]) the full token streams.  *n_steps = iterations planned.
 * cb (nullable) reports the tree effects in order, vals as listed:
 *   RX_EV_EVICT_RUN (slots of one evicted leaf), RX_EV_EVICT {short, evicted},
 *   RX_EV_ALLOC {B} + slots, RX_EV_FINISH {b, d_evictable, new_cached, dup_freed}.
 * Errors: RX_E_INVALID (null pointer, running not ascending / out of range, cur >= end, end past
 * stride or tokens; checked before any effect); a tree error or RX_E_NOMEM stops the call after
 * the iterations already planned (reported in *n_steps). */
typedef enum { RX_EV_ALLOC = 0, RX_EV_EVICT_RUN = 1, RX_EV_EVICT = 2, RX_EV_FINISH = 3 } rx_step_event;
typedef void (*rx_step_event_cb)(void* user, int32_t kind, const int64_t* vals, const int32_t* slots, int64_t n);
rx_status rx_decode_steps(rx_cache* c, int32_t batch, int32_t* table, int64_t stride, int32_t* cur,
                          const int32_t* end, const int32_t* stable, const rx_node* nodes, const int32_t* tokens,
                          const int64_t* offsets, int32_t* running, int32_t* n_running, int32_t max_steps,
                          int32_t* out, int64_t out_cap, int64_t* step_meta, int32_t* n_steps,
                          rx_step_event_cb cb, void* user);

int64_t rx_evictable_size(const rx_cache* c);
int64_t rx_total_cached(const rx_cache* c);
int64_t rx_available(const rx_cache* c);
int64_t rx_num_slots(const rx_cache* c);
int64_t rx_clock(const rx_cache* c);

/* Deterministic pre-order JSON dump: {"id","tokens","slots","ref",
 * "last_access","children":[...]} with children ordered by first token.
 * Writes at most cap bytes (NUL-terminated) into buf and returns the full
 * length (excluding NUL); call with cap = 0 to size the buffer. */
int64_t rx_dump_json(const rx_cache* c, char* buf, int64_t cap);

/* ----------------------------------------------------------------------- */
/*  Compressed FSM for constrained decoding (§4, App. B; */
/*  SURVEY §8(f) NEXT-4).  Host only.                                       */
/* ----------------------------------------------------------------------- */
/* "converting a regular expression into a finite state machine":
 * rx_fsm_create parses regex[0..len) (ASCII; literals, escapes \d \w \s \n
 * \t and escaped punctuation, classes [..] with ranges and ^, '.', groups,
 * '|', quantifiers * + ? {m} {m,} {m,n}) and builds the MINIMAL DFA over
 * bytes 0..127, dead states removed, states numbered breadth-first from the
 * start state (0) by ascending byte (reading R27; the numbering is unique).
 * RX_E_INVALID on a syntax error or an empty language (no side effect);
 * RX_E_NOMEM on allocation failure.  The vocabulary is byte-level (R26).
 * Queries return -1 for a bad handle/state/byte:
 *   rx_fsm_step        next state after `byte`, or -1 if not allowed;
 *   rx_fsm_is_accepting 1 if the model may stop at `state`;
 *   rx_fsm_allowed     number of allowed bytes; out (nullable, cap >= 128)
 *                      receives them ascending;
 *   rx_fsm_jump        "Jump Forward" along the compressed edge
 *                      (adjacent singular transitions merged): while
 *                      `state` has exactly one allowed byte and is not
 *                      accepting, emit that byte and move; returns the number
 *                      of bytes (0 if `state` is not singular), out (nullable)
 *                      receives them, *end_state (nullable) the state reached;
 *                      -1 if cap is too small. */
typedef struct rx_fsm rx_fsm;
rx_status rx_fsm_create(const char* regex, int64_t len, rx_fsm** out);
void rx_fsm_destroy(rx_fsm* f);
int32_t rx_fsm_num_states(const rx_fsm* f);
int32_t rx_fsm_step(const rx_fsm* f, int32_t state, int32_t byte);
int32_t rx_fsm_is_accepting(const rx_fsm* f, int32_t state);
int32_t rx_fsm_allowed(const rx_fsm* f, int32_t state, uint8_t* out);
int32_t rx_fsm_jump(const rx_fsm* f, int32_t state, uint8_t* out, int32_t cap, int32_t* end_state);

/* ----------------------------------------------------------------------- */
/*  Data-parallel router (App. A.4)          */
/* ----------------------------------------------------------------------- */
/* "each worker maintains its own sub-tree, while the router oversees a
 * meta-tree ... a trie that tracks all sub-trees and their associated
 * devices"; dispatch by affinity (shared-prefix length with a worker and
 * with other requests of the batch); worker evictions are committed to a queue
 * that the router applies later (weakly consistent: a stale entry costs a cold
 * dispatch, never a wrong result).  Up to 64 workers.  Host only.
 * Reading R24: affinity[w] = tokens of the request matched along
 * the meta-tree while w is in every edge's worker set from the root;
 * score[w] = affinity[w] - load_weight * loads[w]; argmax, ties -> smaller
 * load -> smaller id; the chosen worker is credited with the request's tokens
 * immediately (so later requests of the batch sharing them follow it) and
 * loads[w] += tokens not already cached there. */
typedef struct rx_router rx_router;
rx_status rx_router_create(int32_t num_workers, rx_router** out);
void rx_router_destroy(rx_router* r);
/* aff: int64 [num_workers] */
rx_status rx_router_affinity(const rx_router* r, const int32_t* tokens, int64_t n, int64_t* aff);
/* Requests b = 0..batch-1 are tokens[offsets[b] .. offsets[b+1]); loads
 * (int64 [num_workers], in/out) is each worker's outstanding work in tokens;
 * worker_out[b] receives the assignment, affinity_out[b] (nullable) its
 * affinity.  Processes requests in order. */
rx_status rx_router_dispatch(rx_router* r, int32_t batch, const int32_t* tokens, const int64_t* offsets,
                             int64_t* loads, double load_weight, int32_t* worker_out, int64_t* affinity_out);
/* worker cached tokens[0..n) (e.g. after rx_insert on that worker) */
rx_status rx_router_insert(rx_router* r, int32_t worker, const int32_t* tokens, int64_t n);
/* worker evicted the leaf path[leaf_start..path_len) (rx_evict_paths callback) */
rx_status rx_router_queue_evict(rx_router* r, int32_t worker, const int32_t* path, int64_t path_len,
                                int64_t leaf_start);
/* apply the queued evictions in FIFO order; returns how many were applied */
int64_t rx_router_sync(rx_router* r);
int64_t rx_router_queue_len(const rx_router* r);
/* deterministic pre-order JSON {"tokens","mask","children"} (same contract as rx_dump_json) */
int64_t rx_router_dump_json(const rx_router* r, char* buf, int64_t cap);

/* ======================================================================= */
/*  2. Attention over the token-slot KV pool (device, sm_100a)              */
/* ======================================================================= */

/* Shape of one attention call on one GPU (one TP shard, P:235 [§3]).
 *   h_q       query heads in q / o           (this shard)
 *   h_kv      KV heads in k_new / v_new / the pool slice (this shard)
 *   head_dim  64 or 128
 *   sm_scale  softmax scale, normally 1/sqrt(head_dim) (R12)
 * GQA: q head h reads kv head h / (h_q / h_kv) (R14).  Supported: head_dim in
 * {64, 128}, h_q % h_kv == 0, group size h_q/h_kv in {1, 2, 4, 8};
 * otherwise RX_E_UNSUPPORTED.
 *
 * Layouts (all row-major, bf16):
 *   pool      d_k_pool, d_v_pool : [num_slots, h_kv, head_dim]; a slot is one
 *             contiguous row of all local heads (one token per page)
 *   q, o      [tokens, h_q, head_dim]      k_new, v_new  [tokens, h_kv, head_dim]
 *   req_to_token (rtt): int32 [rows, rtt_stride]; rtt[row][p] = slot of
 *             position p of the request in that row (D10 in SURVEY §2).
 *   d_rows    int32 [batch] or null: batch entry b uses rtt row d_rows[b]
 *             (null: row b), so a persistent table is never re-uploaded.
 *
 * Streams and concurrency.  Every device call is asynchronous on the given
 * stream (a cudaStream_t; null = the legacy default stream) and returns after
 * enqueueing its launches; faults surface at the caller's next synchronisation.
 * Calls on DIFFERENT streams may run concurrently on one device provided they
 * use different workspaces and do not write the same pool slots, table rows or
 * outputs.  The library holds no device state between calls: all scheduling
 * state lives in the caller's workspace (below).  Host-side it keeps only
 * per-device, thread-safe caches (kernel attributes, SM counts).
 *
 * Workspaces.  d_ws / ws_bytes is caller-owned device memory (the library never
 * allocates device memory).  Its first 256 bytes are a header holding the
 * persistent extend kernel's work counters: they MUST be zero before the
 * workspace is first used (allocate it zeroed), and every call leaves them zero
 * again; split-KV partials follow the header.  One workspace may serve any
 * sequence of calls on one stream; concurrently running calls need one each.
 * A call given less than its rx_*_workspace_bytes(...) returns RX_E_WORKSPACE.
 */
typedef struct {
  int32_t h_q;
  int32_t h_kv;
  int32_t head_dim;
  float sm_scale;
} rx_attn_cfg;

/* KV store (A5; "the KV cache of the new tokens is stored in the pool" at the
 * slots the allocator returned, P:494-499 [App. A.1], one token per page P:181):
 * k_pool[slots[i]] = k[i]; v_pool[slots[i]] = v[i] for i < n
 * (bit-exact copy).  If d_rtt_index is non-null, also rtt_flat[d_rtt_index[i]]
 * = slots[i] (d_rtt must then be non-null): the decode step's "append one
 * column to req_to_token" in the same launch.  d_k and d_v may both be null
 * when d_rtt_index is given: then only the table entries are written (an
 * output step whose K/V the following rx_extend stores itself, so no row is
 * written twice).  Slots must be distinct and in [1, num_slots).
 * Asynchronous on stream. */
rx_status rx_store_kv(const rx_attn_cfg* cfg, int64_t n, const int32_t* d_slots,
                      const void* d_k, const void* d_v, void* d_k_pool, void* d_v_pool,
                      int64_t num_slots, int32_t* d_rtt, const int64_t* d_rtt_index,
                      void* stream);

/* Host -> device copy of small per-call metadata by the SMs (one kernel on
 * stream): h_src must be pinned host memory (cudaHostAlloc / a pinned torch
 * tensor; RX_E_INVALID otherwise), read over PCIe through its device mapping.
 * Unlike cudaMemcpyAsync it does not queue on the copy engines, where a large
 * input prefetch on another stream would hold it (engines serve copies in
 * submission order).  The host buffer must stay valid until the kernel ran. */
rx_status rx_copy_h2d(void* d_dst, const void* h_src, int64_t bytes, void* stream);

/* Extend (prefill with prefix reuse) for a ragged batch.
 * Request b has prefix_len[b] cached tokens (slots rtt[row_b][0..prefix_len))
 * and extend_len[b] >= 0 new tokens at positions prefix_len .. prefix_len +
 * extend_len - 1, whose slots are rtt[row_b][prefix_len + j].  The call
 *   (1) stores k_new / v_new of every new token into its slot, and
 *   (2) for new token j at absolute position p = prefix_len + j and q head h,
 *       o = softmax_{i <= p}(scale * q . K[i]) V[i]   over the kv head of h
 *       (R13: causal over absolute positions; fp32 accumulation, R15).
 * Hazard-free in one call because new slots are never prefix slots.
 *   d_prefix_lens, d_extend_lens : int32 [batch]        (device)
 *   d_qo_indptr                  : int32 [batch + 1]    (device) exclusive
 *       prefix sum of extend_lens: request b's rows in q/k_new/v_new/o are
 *       [qo_indptr[b], qo_indptr[b+1])
 *   total_new        = qo_indptr[batch] (host copy, sizes the TMA views)
 *   max_extend_len   = max extend_len (host copy, sizes the grid)
 *   max_prefix_len   = max prefix_len (host copy); rtt_stride must be >= every
 *       prefix_len + extend_len (only the maxima are checked)
 * Kernel choice (same results within the attention tolerance): the tcgen05
 * tile kernel, or — when max_extend_len * (h_q / h_kv) <= 32 and batch * h_kv
 * >= 148, i.e. short segments such as jump-forward edges of constrained
 * decoding (§4) — the decode kernel in multi-query mode (one mma.sync
 * column per (row, GQA head), causal per column).  Two launches either way
 * (store, attention).
 * Workspace: d_ws of ws_bytes >= rx_extend_workspace_bytes(...) (the 256-byte
 * header: the tcgen05 kernel's work counters; zero on entry, zero on exit). */
rx_status rx_extend(const rx_attn_cfg* cfg, int32_t batch,
                    const int32_t* d_rtt, int64_t rtt_stride, const int32_t* d_rows,
                    const int32_t* d_prefix_lens, const int32_t* d_extend_lens,
                    const int32_t* d_qo_indptr, int64_t total_new,
                    int32_t max_extend_len, int32_t max_prefix_len,
                    const void* d_q, const void* d_k_new, const void* d_v_new,
                    void* d_k_pool, void* d_v_pool, int64_t num_slots, void* d_o,
                    void* d_ws, size_t ws_bytes, void* stream);

/* rx_extend for a batch whose rows all share cached positions [0, shared_len)
 * (the same slots, i.e. one radix-tree path: the running requests of a
 * few-shot or long-context batch), for short segments (jump-forward steps,
 * §4).  Same result as rx_extend (within the attention tolerance); the
 * shared prefix is attended ONCE for all Σ extend_len rows on the tensor cores
 * (cascade) and each request's own positions
 * [shared_len, prefix_len + j] by the multi-query decode kernel, merged by
 * log-sum-exp.  Preconditions: 0 <= shared_len <= every prefix_len and the
 * slots of positions < shared_len equal in every row (not checked); when
 * shared_len == 0 or the multi-query shape condition of rx_extend fails the
 * call is exactly rx_extend.  Workspace: >= rx_extend_cascade_workspace_bytes
 * (cfg, total_new, shared_len) bytes.  Four launches (store, suffix partial,
 * shared prefix stream-K, log-sum-exp merge). */
size_t rx_extend_cascade_workspace_bytes(const rx_attn_cfg* cfg, int64_t total_new, int32_t shared_len);
rx_status rx_extend_cascade(const rx_attn_cfg* cfg, int32_t batch, const int32_t* d_rtt, int64_t rtt_stride,
                            const int32_t* d_rows, const int32_t* d_prefix_lens, const int32_t* d_extend_lens,
                            const int32_t* d_qo_indptr, int64_t total_new, int32_t max_extend_len,
                            int32_t max_prefix_len, int32_t shared_len, const void* d_q, const void* d_k_new,
                            const void* d_v_new, void* d_k_pool, void* d_v_pool, int64_t num_slots, void* d_o,
                            void* d_ws, size_t ws_bytes, void* stream);

size_t rx_extend_workspace_bytes(const rx_attn_cfg* cfg, int32_t batch, int32_t max_extend_len);

/* Decode: one query per request at position seq_len[b] - 1 (P:495 [App.
 * A.1]), over slots rtt[row_b][0 .. seq_len[b]).  The newest token's KV must
 * already be stored (rx_store_kv) and seq_len counts it; seq_len >= 1
 * (entries < 1 produce undefined rows: validate on the host).
 *   d_seq_lens  int32 [batch] (device);  max_seq_len = its max (host copy;
 *   plans the split-KV partition, so it must be >= every seq_len).
 * Split-KV partials are merged by log-sum-exp in the same call (A8).
 * Workspace: d_ws of ws_bytes >= rx_decode_workspace_bytes(...). */
rx_status rx_decode(const rx_attn_cfg* cfg, int32_t batch,
                    const int32_t* d_rtt, int64_t rtt_stride, const int32_t* d_rows,
                    const int32_t* d_seq_lens, int32_t max_seq_len,
                    const void* d_q, const void* d_k_pool, const void* d_v_pool,
                    int64_t num_slots, void* d_o, void* d_ws, size_t ws_bytes, void* stream);

/* Decode step with the newest token's KV appended in the same launch (A4 + A5
 * + A7 + A8): for every request b, k_new[b] / v_new[b] ([batch, h_kv,
 * head_dim] bf16) are stored into pool slot new_slots[b] (int32 [batch],
 * device), rtt[row_b][seq_len[b] - 1] = new_slots[b] is recorded, and the
 * query attends over positions 0 .. seq_len[b]-1 including the new token.
 * Equivalent to rx_store_kv(...) followed by rx_decode(...), in one kernel
 * (plus the split merge).  d_rtt is written (one entry per request).
 * d_stable_lens (int32 [batch], device, nullable): positions < stable_lens[b]
 * of request b were written by work that completed before the previous
 * rx_decode* call on the stream was launched (e.g. the prompt, stored by the
 * batch's rx_extend).  The kernels are launched as programmatic dependents of
 * the previous step: they read those positions while the previous step still
 * drains and wait for it before anything else (the newest generated
 * positions, the split workspace, the append).  null: wait first. */
rx_status rx_decode_append(const rx_attn_cfg* cfg, int32_t batch,
                           int32_t* d_rtt, int64_t rtt_stride, const int32_t* d_rows,
                           const int32_t* d_seq_lens, const int32_t* d_stable_lens, int32_t max_seq_len,
                           const void* d_q, const void* d_k_new, const void* d_v_new,
                           const int32_t* d_new_slots, void* d_k_pool, void* d_v_pool,
                           int64_t num_slots, void* d_o, void* d_ws, size_t ws_bytes, void* stream);

size_t rx_decode_workspace_bytes(const rx_attn_cfg* cfg, int32_t batch, int32_t max_seq_len);

/* Shared-prefix ("cascade") decode step — SURVEY §8(f) NEXT-1, motivated by
 * "requests with the same prompt prefix can reuse the KV cache" (P:171 [§3])
 * and the shared-prefix kernels cited at P:458 [§7].  Same result as
 * rx_decode_append, but positions [0, shared_len), which must hold the SAME
 * slots in every batch row (a radix node all requests are pinned on; the slots
 * of row d_rows[0] are read), are attended ONCE for the whole batch as a dense
 * tensor-core problem (rows = requests x GQA heads; the (q-tile pair, kv head)
 * x prefix-tile work split stream-K over the SMs), each request's suffix
 * [shared_len, seq_len) by the decode kernel first, and the partials merged by
 * log-sum-exp.  Requires 0 <= shared_len < every seq_len (shared_len == 0
 * falls back to rx_decode_append).  3 launches (suffix, shared, merge).
 * Workspace: rx_decode_cascade_workspace_bytes(cfg, batch, max_seq_len, shared_len). */
rx_status rx_decode_cascade_append(const rx_attn_cfg* cfg, int32_t batch,
                                   int32_t* d_rtt, int64_t rtt_stride, const int32_t* d_rows,
                                   const int32_t* d_seq_lens, const int32_t* d_stable_lens,
                                   int32_t max_seq_len, int32_t shared_len,
                                   const void* d_q, const void* d_k_new, const void* d_v_new,
                                   const int32_t* d_new_slots, void* d_k_pool, void* d_v_pool,
                                   int64_t num_slots, void* d_o, void* d_ws, size_t ws_bytes, void* stream);

size_t rx_decode_cascade_workspace_bytes(const rx_attn_cfg* cfg, int32_t batch, int32_t max_seq_len,
                                         int32_t shared_len);

/* A run of n_steps decode steps in ONE call (Alg. 1's output loop: the
 * host-side per-step launch cost — argument checks, marshalling — paid once per run).
 * Step k is exactly rx_decode_cascade_append(cfg, h_batch[k], d_rtt, rtt_stride,
 * rows, seq_lens, stable, h_max_seq[k], shared_len, h_q[k], h_k_new[k], h_v_new[k],
 * new_slots, d_k_pool, d_v_pool, num_slots, h_o[k], d_ws, ws_bytes, stream)
 * (shared_len == 0: rx_decode_append), with its int32 records read from the device
 * array d_rec at word offset h_rec_off[k]: [new_slots | seq_lens | rows | stable
 * lens], h_batch[k] words each (the rx_decode_steps staging layout; stable lens
 * used only when with_stable != 0).  h_*: host arrays of n_steps entries (device
 * pointers for q / k_new / v_new / o).  Steps are enqueued in order on the stream;
 * the first failing step's status is returned (earlier steps stay enqueued).
 * The workspace must fit every step.
 * tp_world > 0 (TP with the fused gather, §3 rx_decode_append_tp): step k stores
 * its rows into every rank's gathered block h_o[k * tp_world + p] ([batch,
 * tp_h_q_total, head_dim], head offset tp_head_offset) instead of an o; tp_world
 * = 0: h_o[k] is step k's output [batch, h_q, head_dim]. */
rx_status rx_decode_run(const rx_attn_cfg* cfg, int32_t n_steps, const int32_t* h_batch, const int32_t* h_max_seq,
                        int32_t shared_len, int32_t* d_rtt, int64_t rtt_stride, const int32_t* d_rec,
                        const int64_t* h_rec_off, int32_t with_stable, void* const* h_q, void* const* h_k_new,
                        void* const* h_v_new, void* d_k_pool, void* d_v_pool, int64_t num_slots, void* const* h_o,
                        int32_t tp_world, int32_t tp_h_q_total, int32_t tp_head_offset, void* d_ws,
                        size_t ws_bytes, void* stream);

/* ======================================================================= */
/*  3. Tensor-parallel output all-gather over peer memory (A9)              */
/* ======================================================================= */
/* "For tensor parallelism, each GPU maintains a sharded KV cache. There is no
 * need for additional synchronization because the tree operations are the
 * same" (P:235 [§3]): a TP attention call's only exchange is reassembling its
 * output head shards.  Each rank allocates ONE zero-filled device buffer of
 * rx_tp_buffer_bytes(world, cap) bytes (cap = the largest shard in bytes, a
 * multiple of 16), exports it with rx_tp_ipc_handle (RX_TP_HANDLE_BYTES
 * opaque bytes) together with rx_tp_ipc_offset(d_buf) (the buffer's byte
 * offset inside the allocation the handle names — a caching allocator may
 * sub-allocate it; -1 on error), and maps every peer's buffer with
 * rx_tp_ipc_open (+ that peer's offset; on a multi-GPU node: NVLink /
 * NVSwitch peer memory; ranks may also share one device).  rx_tp_allgather(d_src, bytes, peer_bufs, world, rank, cap, seq)
 * then, in one kernel on the stream: stores this rank's shard d_src[0, bytes)
 * into every rank's buffer (P2P stores), publishes seq to every rank, and
 * waits for every rank's seq; when it completes the caller's own buffer holds
 * the gathered output at offset 256 + (seq & 1)·world·cap, shard r at
 * + r·cap.  peer_bufs: host array of world pointers (peer_bufs[rank] = the
 * caller's own buffer).  Every rank must issue the same calls in the same
 * order with seq = 1, 2, 3, ... (the gathered data of call seq stays valid
 * until this rank issues call seq + 2).  world <= 8; bytes <= cap;
 * RX_E_INVALID otherwise.  A rank that never calls leaves its peers waiting
 * (like any collective) — for at most ~30 s, then the kernel traps (a launch
 * error at the next synchronisation) instead of hanging the device. */
#define RX_TP_HANDLE_BYTES 64
size_t rx_tp_buffer_bytes(int32_t world, int64_t cap);
rx_status rx_tp_ipc_handle(void* d_buf, void* handle_out);
int64_t rx_tp_ipc_offset(const void* d_buf);
rx_status rx_tp_ipc_open(const void* handle, void** d_ptr);
rx_status rx_tp_ipc_close(void* d_ptr);
rx_status rx_tp_allgather(const void* d_src, int64_t bytes, void* const* peer_bufs, int32_t world, int32_t rank,
                          int64_t cap, int64_t seq, void* stream);

/* TP decode step with the all-gather FUSED into the attention epilogue (A7 +
 * A8 + A9; the north star's "single all-gather over NVLink reassembling
 * outputs", done as the output stores themselves).  Semantics of
 * rx_decode_cascade_append (shared_len > 0) or rx_decode_append (shared_len
 * == 0) on this rank's heads (cfg->h_q local q heads, cfg->h_kv kv heads), but
 * there is no d_o: the kernel that produces the final bf16 row of (request b,
 * local q head h) stores it into EVERY rank's gathered output
 * out->d_o[p] (p < out->world; [batch, out->h_q_total, head_dim] bf16 on rank
 * p, mapped into this process: NVLink / NVSwitch peer memory via
 * rx_tp_ipc_open, or this rank's own buffer) at row b, head
 * out->head_offset + h.  No separate collective, kernel or copy.  A rank's
 * gathered buffer is complete once every rank has issued its calls and an
 * rx_tp_allgather(bytes = 0) barrier after them has completed on this rank
 * (its flags publish "my stores are done" and wait for every peer's);
 * buffers must not be reused by a peer's later call before this rank is done
 * reading them (double-buffer across barriers).  RX_E_INVALID if out is null,
 * world is outside [1, 8], a destination is null, or the heads do not fit. */
typedef struct {
  void* d_o[8];          /* rank p's gathered output buffer for this call (device address valid here) */
  int32_t world;         /* destinations (ranks) */
  int32_t h_q_total;     /* q heads per gathered row */
  int32_t head_offset;   /* this rank's first q head in the gathered row */
} rx_tp_out;
rx_status rx_decode_append_tp(const rx_attn_cfg* cfg, int32_t batch, int32_t* d_rtt, int64_t rtt_stride,
                              const int32_t* d_rows, const int32_t* d_seq_lens, const int32_t* d_stable_lens,
                              int32_t max_seq_len, int32_t shared_len, const void* d_q, const void* d_k_new,
                              const void* d_v_new, const int32_t* d_new_slots, void* d_k_pool, void* d_v_pool,
                              int64_t num_slots, const rx_tp_out* out, void* d_ws, size_t ws_bytes, void* stream);

/* Number of kernel launches the last successful rx_extend / rx_decode /
 * rx_store_kv call on this thread issued (for launch accounting). */
int32_t rx_last_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* RX_H_ */
