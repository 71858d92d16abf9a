"""Seeded synthetic-input generators shared by the oracle and the CUDA path.

This package holds NONE of the method's arithmetic: no radix tree, no slot
allocation, no attention.  It only produces inputs:

* token streams shaped like the paper's workloads (``rxgen.workloads``);
* a counter-based generator (splitmix64) that turns a token prefix into
  per-position hashes, and hashes into bf16 q/k/v values (``rxgen.values``).

K/V at position p depend only on the hash of tokens[0..p] — the paper's
"KV cache computation depends only on prefix tokens" (§3,
PAPER.md:499 App. A.1) — so prefix reuse cannot change an input bit.

Both sides (``oracle/`` and ``paper_2312_07104_b200``) import this package;
neither imports the other.
"""
from .hashing import (GOLDEN, MASK64, splitmix64_int, splitmix64_np,
                      splitmix64_t, prefix_hashes, next_token, sched_keys, fsm_choice)
from .values import gen_values, gen_values_np

__all__ = [
    "GOLDEN", "MASK64", "splitmix64_int", "splitmix64_np", "splitmix64_t",
    "prefix_hashes", "next_token", "sched_keys", "fsm_choice", "gen_values", "gen_values_np",
]
