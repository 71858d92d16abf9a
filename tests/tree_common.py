"""Test-side helpers shared by the oracle-tree and library-tree tests.

``TreeAPI`` is the minimal surface both trees expose to the tests: the oracle
(oracle.radix.RadixCache) and the C-ABI library (via its Python binding) are
driven through small adapters so one op sequence can replay on both.
"""
from __future__ import annotations

import json
import os

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load_fig3():
    with open(os.path.join(GOLDEN, "fig3_radix_trace.json")) as f:
        return json.load(f)


def names_tree(dump: dict, seg_of_token: dict) -> dict:
    """Convert a pre-order dump into {edge label as segment names: subtree}."""
    def label(tokens):
        names = []
        for t in tokens:
            s = seg_of_token[t]
            if not names or names[-1] != s:
                names.append(s)
        return " ".join(names)

    def rec(node):
        return {label(c["tokens"]): rec(c) for c in node["children"]}
    return rec(dump)


def run_fig3(tree, check):
    """Drive a tree through the Fig. 3 golden steps; ``tree`` is an adapter with
    match(tokens)->(handle, m, slots), inc(h), dec(h), evict(k)->(n, runs),
    alloc(n)->slots, insert(tokens, slots)->(new, dup), dump()->dict."""
    g = load_fig3()
    seg = g["segments"]
    seg_of_token = {t: name for name, toks in seg.items() for t in toks}
    slot_token = {}
    for st in g["steps"]:
        reqs = []
        for r in st["batch"]:
            prompt = [t for s in r["prompt"] for t in seg[s]]
            out = [t for s in r["output"] for t in seg[s]]
            reqs.append((prompt, out))
        handles = []
        matched = []
        for prompt, out in reqs:
            h, m, slots = tree.match(prompt)
            matched.append(m)
            use = min(m, len(prompt) - 1)
            handles.append((h, use, list(slots[:use])))
        if "expect_matched" in st:
            check(matched == st["expect_matched"], f"step {st['step']}: matched {matched}")
        for h, _, _ in handles:
            tree.inc(h)
        evicted_names = []
        if st["evict"]:
            n, runs = tree.evict(st["evict"])
            for run in runs:
                toks = [slot_token[s] for s in run]
                names = []
                for t in toks:
                    if not names or names[-1] != seg_of_token[t]:
                        names.append(seg_of_token[t])
                evicted_names.append(" ".join(names))
        check(evicted_names == st["evicted"], f"step {st['step']}: evicted {evicted_names}")
        allocs = []
        for (prompt, out), (h, use, slots) in zip(reqs, handles):
            new = tree.alloc(len(prompt) + len(out) - use)
            full = prompt + out
            for s, t in zip(new, full[use:]):
                slot_token[s] = t
            allocs.append(slots + list(new))
        for (prompt, out), (h, use, _), slots in zip(reqs, handles, allocs):
            tree.dec(h)
            tree.insert(prompt + out, slots)
        got = names_tree(tree.dump(), seg_of_token)
        check(got == st["tree"], f"step {st['step']}: tree {got} != {st['tree']}")
