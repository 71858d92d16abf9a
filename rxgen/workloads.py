"""Workload shapes C1-C5 (BASELINE.json "configs") as seeded token streams.

Only inputs live here: attention shapes, pool sizes, and the prompt token
lists / output lengths of each request.  How requests flow through the radix
tree and the kernels is the method, and lives in the oracle and in the
library's harness separately.  Parameters the configs leave open are fixed in
SURVEY.md §8(d) ("Concrete synthetic inputs"); DESIGN.md restates them.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class Shape:
    h_q: int
    h_kv: int
    head_dim: int

    @property
    def group(self) -> int:
        return self.h_q // self.h_kv

    @property
    def sm_scale(self) -> float:
        # Reading R12: 1/sqrt(head_dim), passed as fp32.
        return float(np.float32(1.0 / math.sqrt(self.head_dim)))


@dataclass
class Request:
    """A prompt plus the number of tokens the mock model will generate."""
    prompt: np.ndarray            # int32 tokens
    max_new_tokens: int
    tag: str = ""


@dataclass
class Workload:
    name: str
    shape: Shape
    num_slots: int
    vocab: int
    seed: int
    # phases: list of ("hint", [Request]) / ("batch", [Request]) in order.
    phases: list = field(default_factory=list)
    meta: dict = field(default_factory=dict)


def _rand_tokens(rng, n, vocab):
    return rng.integers(1, vocab, size=n, dtype=np.int64).astype(np.int32)


def c1(seed: int = 0, n_req: int = 16, prefix: int = 64, new: int = 32, decode: int = 16,
       num_slots: int = 4096) -> Workload:
    """C1: 8 q / 2 kv heads, hd 64, 16 requests sharing a 64-token prefix, 32 new each, 16 decode steps."""
    rng = np.random.default_rng(seed)
    vocab = 32000
    pre = _rand_tokens(rng, prefix, vocab)
    reqs = [Request(np.concatenate([pre, _rand_tokens(rng, new, vocab)]), decode, f"r{i}") for i in range(n_req)]
    return Workload("C1", Shape(8, 2, 64), num_slots, vocab, seed,
                    [("hint", [Request(pre, 0, "prefix")]), ("batch", reqs)],
                    {"prefix": prefix, "new": new, "decode": decode})


def c2(seed: int = 0, n_req: int = 64, prefix: int = 1536, new_lo: int = 64, new_hi: int = 192,
       decode: int = 64, num_slots: int = 32768, fixed_new: int | None = None) -> Workload:
    """C2: Llama-2-7B attention (32/32/128), 5-shot MMLU-like batch 64 sharing a ~1.5k prefix."""
    rng = np.random.default_rng(seed)
    vocab = 32000
    pre = _rand_tokens(rng, prefix, vocab)
    reqs = []
    for i in range(n_req):
        n = fixed_new if fixed_new is not None else int(rng.integers(new_lo, new_hi + 1))
        reqs.append(Request(np.concatenate([pre, _rand_tokens(rng, n, vocab)]), decode, f"q{i}"))
    return Workload("C2", Shape(32, 32, 128), num_slots, vocab, seed,
                    [("hint", [Request(pre, 0, "prefix")]), ("batch", reqs)],
                    {"prefix": prefix, "decode": decode})


def c3(seed: int = 0, sessions: int = 256, turns: int = 4, in_lo: int = 256, in_hi: int = 512,
       out_lo: int = 256, out_hi: int = 512, num_slots: int = 1 << 20, system_prompt: int = 0) -> Workload:
    """C3: Llama-3-8B GQA (32/8/128) multi-turn chat; turn t prompt = history + new input.

    The per-turn inputs and output lengths are drawn here; the prompt of turn
    t > 0 depends on the generated answers of turn t-1, which the drivers
    append themselves (meta["turn_inputs"][s][t], meta["turn_outputs"][s][t]).
    """
    rng = np.random.default_rng(seed)
    vocab = 128256
    sysp = _rand_tokens(rng, system_prompt, vocab) if system_prompt else np.zeros(0, np.int32)
    inputs = [[_rand_tokens(rng, int(rng.integers(in_lo, in_hi + 1)), vocab) for _ in range(turns)]
              for _ in range(sessions)]
    outs = [[int(rng.integers(out_lo, out_hi + 1)) for _ in range(turns)] for _ in range(sessions)]
    return Workload("C3", Shape(32, 8, 128), num_slots, vocab, seed, [],
                    {"turn_inputs": inputs, "turn_outputs": outs, "turns": turns, "system": sysp})


def c4(seed: int = 0, root: int = 2048, depth: int = 3, fanout: int = 4, p_lo: int = 32, p_hi: int = 96,
       t_lo: int = 32, t_hi: int = 64, capacity_frac: float = 0.6) -> Workload:
    """C4: tree-of-thought, depth 3 x fan-out 4 on a 2k root, pool at 60% of the tree's distinct tokens.

    meta["nodes"][level] = list of (parent_index, branch_prompt_tokens, thought_len).
    Reading R18 (C4a): capacity = ceil(0.6 * T), T = distinct tokens of the full tree.
    """
    rng = np.random.default_rng(seed)
    vocab = 32000
    rt = _rand_tokens(rng, root, vocab)
    levels = []
    prev = 1
    total = root
    for lvl in range(depth):
        nodes = []
        for parent in range(prev):
            for _ in range(fanout):
                bp = _rand_tokens(rng, int(rng.integers(p_lo, p_hi + 1)), vocab)
                tl = int(rng.integers(t_lo, t_hi + 1))
                nodes.append((parent, bp, tl))
                total += len(bp) + tl
        levels.append(nodes)
        prev = len(nodes)
    cap = int(math.ceil(capacity_frac * total)) + 1   # +1: slot 0 is the padding sink
    return Workload("C4", Shape(32, 32, 128), cap, vocab, seed, [],
                    {"root": rt, "levels": levels, "distinct_tokens": total})


def c5(seed: int = 0, n_req: int = 128, prefix: int = 8192, question: int = 128, decode: int = 32,
       num_slots: int = 65536, ragged: bool = False) -> Workload:
    """C5: Llama-2-70B shape (64/8/128) long-prefix RAG: 8k shared context, batch 128."""
    rng = np.random.default_rng(seed)
    vocab = 32000
    pre = _rand_tokens(rng, prefix, vocab)
    reqs = []
    for i in range(n_req):
        n = int(rng.integers(64, 257)) if ragged else question
        reqs.append(Request(np.concatenate([pre, _rand_tokens(rng, n, vocab)]), decode, f"q{i}"))
    return Workload("C5", Shape(64, 8, 128), num_slots, vocab, seed,
                    [("hint", [Request(pre, 0, "context")]), ("batch", reqs)],
                    {"prefix": prefix, "decode": decode})


def mix(seed: int = 0, groups: int = 4, per_group: int = 16, prefix: int = 1024, q_lo: int = 32, q_hi: int = 96,
        out_lo: int = 8, out_hi: int = 32, num_slots: int = 2600) -> Workload:
    """Scheduling ablation ("FCFS / Random Schedule"): `groups` unrelated few-shot
    prefixes, per_group questions each, arriving interleaved (request i belongs to group i mod groups)
    in ONE waiting queue; the pool holds roughly 1.5 groups, so the admission order decides how often
    a prefix is evicted and recomputed (cache thrashing).  Llama-2-7B attention shape (32/32/128), no
    hint requests.  Phase kind "queue" = Alg. 1 admission waves over the whole queue."""
    rng = np.random.default_rng(seed)
    vocab = 32000
    pres = [_rand_tokens(rng, prefix, vocab) for _ in range(groups)]
    reqs = []
    for i in range(groups * per_group):
        g = i % groups
        q = _rand_tokens(rng, int(rng.integers(q_lo, q_hi + 1)), vocab)
        reqs.append(Request(np.concatenate([pres[g], q]), int(rng.integers(out_lo, out_hi + 1)), f"g{g}r{i}"))
    return Workload("MIX", Shape(32, 32, 128), num_slots, vocab, seed, [("queue", reqs)],
                    {"groups": groups, "prefix": prefix})


def dp_fewshot(seed: int = 0, workers: int = 1, subjects_per_worker: int = 2, prefix: int = 1536,
               per_worker: int = 64, q_lo: int = 64, q_hi: int = 192, decode: int = 16, batches: int = 2,
               num_slots: int = 32768) -> Workload:
    """Data-parallel few-shot serving (App. A.4: "linear scaling and an optimal cache hit
    rate" on MMLU with 4 workers): `workers` x subjects_per_worker unrelated 5-shot-like prefixes
    (MMLU subjects), `batches` batches of per_worker x workers questions each, subject of request i =
    i mod subjects (interleaved arrival), U[q_lo, q_hi] question tokens, `decode` output tokens.
    Weak scaling: subjects and requests grow with the worker count.  Llama-2-7B attention shape
    (32/32/128); num_slots per worker.  Phase kind "dp_batch" = one router dispatch."""
    rng = np.random.default_rng(seed)
    vocab = 32000
    S = workers * subjects_per_worker
    pres = [_rand_tokens(rng, prefix, vocab) for _ in range(S)]
    phases = []
    for b in range(batches):
        reqs = []
        for i in range(per_worker * workers):
            q = _rand_tokens(rng, int(rng.integers(q_lo, q_hi + 1)), vocab)
            reqs.append(Request(np.concatenate([pres[i % S], q]), decode, f"b{b}s{i % S}r{i}"))
        phases.append(("dp_batch", reqs))
    return Workload("DP", Shape(32, 32, 128), num_slots, vocab, seed, phases,
                    {"workers": workers, "subjects": S, "prefix": prefix})


# character-profile JSON schema (cf. the paper's JSON example P:106-108): long constant
# keys (jump-forward edges) between short free fields
JSON_REGEX = (r'\{"name": "[A-Z][a-z]{2,9}", "age": [1-9]\d?, "occupation": "(engineer|doctor|teacher|artist)", '
              r'"city": "[A-Z][a-z]{3,9}", "skills": \["[a-z]{3,8}", "[a-z]{3,8}", "[a-z]{3,8}"\], '
              r'"summary": "[a-z ]{20,60}"\}')


def json_decode(seed: int = 0, n_req: int = 64, prefix: int = 512, doc_lo: int = 64, doc_hi: int = 192,
                compressed: bool = True, regex: str = JSON_REGEX, num_slots: int = 65536) -> Workload:
    """JSON decoding under a regex ("JSON decoding with a schema specified by a regular
    expression"): n_req requests share a `prefix`-token instruction
    (sent first as a hint) plus a U[doc_lo, doc_hi] document each, and generate one JSON
    object constrained by `regex` with a byte-level vocabulary (R26).  compressed=True decodes with
    the compressed FSM (jump forward: a forced edge rides with the preceding token in one extend
    pass), False token by token.  Llama-2-7B attention shape (32/32/128).  The output
    lengths follow from the FSM walk of the mock model (R28); max_new_tokens bounds them."""
    rng = np.random.default_rng(seed)
    vocab = 32000
    pre = _rand_tokens(rng, prefix, vocab)
    reqs = [Request(np.concatenate([pre, _rand_tokens(rng, int(rng.integers(doc_lo, doc_hi + 1)), vocab)]), 512,
                    f"j{i}") for i in range(n_req)]
    return Workload("JSON", Shape(32, 32, 128), num_slots, vocab, seed,
                    [("hint", [Request(pre, 0, "instr")]), ("fsm", reqs)],
                    {"regex": regex, "compressed": compressed, "prefix": prefix})


CONFIGS = {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5, "MIX": mix, "JSON": json_decode}
