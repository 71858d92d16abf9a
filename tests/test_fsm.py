"""Compressed FSM (§4, App. B).

Oracle pins (independent of either implementation):
* language: the oracle DFA accepts exactly what Python's `re.fullmatch` accepts (library special
  case), on random strings and on random walks of the DFA;
* minimality (R27): every pair of states is distinguishable (product-automaton BFS finds a
  separating string), and every state reaches acceptance (no dead states);
* the paper's worked example: from the start of the JSON regex the compressed
  edge is the constant `{"summary": "`, decoded in one jump.
Library: rx_fsm_* equals the oracle state for state (transitions, accepting flags, allowed sets,
compressed edges) — bit-exact."""
import random
import re
import zlib
from collections import deque

import pytest

from oracle.fsm import FSM
from paper_2312_07104_b200 import Fsm, RxError

REGEXES = [
    r'\{"summary": "[a-z ]{1,20}", "grade": "[ABCD][+-]?"\}',
    r'(ab|cd)*e', r'\d{2,4}-\w+', r'[^a]x?', r'a{3}b{0,2}c+',
    r'(Excellent|Above Average|Fair|Below Average)', r'(a|a)(b|b)*', r'a*a*a*', r'[\]a-]+x', r'.\s\w?',
    r'\{"name": "\w{1,8}", "age": \d{1,2}, "job": "(engineer|doctor|teacher)"\}',
    r'(x|xy|xyz){2,3}', r'((a|b)c)+d?',
]
ALPH = 'abcdexyz-_{}":ABCD+ 0123456789summarygrade,\n'


def _rand_regex(rng, depth=0):
    r = rng.random()
    if depth > 2 or r < 0.35:
        return rng.choice(["a", "b", "c", "[ab]", "[^a]", "\\d", "x", "."])
    if r < 0.55:
        return _rand_regex(rng, depth + 1) + _rand_regex(rng, depth + 1)
    if r < 0.7:
        return "(" + _rand_regex(rng, depth + 1) + "|" + _rand_regex(rng, depth + 1) + ")"
    q = rng.choice(["*", "+", "?", "{2}", "{1,3}", "{0,2}", "{2,}"])
    return "(" + _rand_regex(rng, depth + 1) + ")" + q


@pytest.mark.parametrize("rx", REGEXES + [_rand_regex(random.Random(s)) for s in range(20)])
def test_oracle_language_equals_re(rx):
    f = FSM(rx)
    cre = re.compile(rx)
    rng = random.Random(zlib.crc32(rx.encode()))
    for _ in range(2000):
        s = "".join(rng.choice(ALPH) for _ in range(rng.randrange(0, 14)))
        assert bool(cre.fullmatch(s)) == f.matches(s.encode()), (rx, s)
    for _ in range(200):                      # random walks accept only matching strings
        st, out = 0, []
        while len(out) < 64:
            opts = f.allowed(st) + ([None] if f.accepting[st] else [])
            c = rng.choice(opts)
            if c is None:
                assert cre.fullmatch(bytes(out).decode()), (rx, bytes(out))
                break
            out.append(c)
            st = f.step(st, c)


@pytest.mark.parametrize("rx", REGEXES)
def test_oracle_minimal_and_trim(rx):
    f = FSM(rx)
    n = f.num_states
    # every state reaches acceptance
    for s in range(n):
        seen, q = {s}, deque([s])
        ok = False
        while q:
            u = q.popleft()
            ok |= f.accepting[u]
            for t in f.trans[u].values():
                if t not in seen:
                    seen.add(t)
                    q.append(t)
        assert ok
    # every pair is distinguishable (-1 = dead)
    def acc(u):
        return u >= 0 and f.accepting[u]

    def nxt(u, b):
        return f.step(u, b) if u >= 0 else -1
    for a in range(n):
        for b in range(a + 1, n):
            seen, q, found = {(a, b)}, deque([(a, b)]), False
            while q and not found:
                u, v = q.popleft()
                if acc(u) != acc(v):
                    found = True
                    break
                for c in set(f.trans[u]) | set(f.trans[v]) if u >= 0 and v >= 0 else \
                        (set(f.trans[u]) if u >= 0 else set(f.trans[v])):
                    p = (nxt(u, c), nxt(v, c))
                    if p not in seen:
                        seen.add(p)
                        q.append(p)
            assert found, (rx, a, b)


def test_paper_example_jump_forward():
    """`{"summary": "` is a constant of the regex and is decoded in one step."""
    f = FSM(r'\{"summary": "[a-z ]{1,20}", "grade": "[ABCD][+-]?"\}')
    forced, end = f.jump(0)
    assert bytes(forced) == b'{"summary": "'
    assert not f.singular(end) and len(f.allowed(end)) == 27
    # after the summary text closes, `", "grade": "` is the next compressed edge
    st = end
    for c in b'abc':
        st = f.step(st, c)
    st = f.step(st, ord('"'))
    forced, end2 = f.jump(st)
    assert bytes(forced) == b', "grade": "'
    assert f.allowed(end2) == [ord(c) for c in "ABCD"]
    # a grade letter is followed by a choice ([+-]? then the closing quote), not a jump
    st = f.step(end2, ord("A"))
    assert f.jump(st)[0] == [] and f.allowed(st) == [ord('"'), ord("+"), ord("-")]


@pytest.mark.parametrize("rx", REGEXES + [_rand_regex(random.Random(100 + s)) for s in range(30)])
def test_library_fsm_equals_oracle(rx):
    o, l = FSM(rx), Fsm(rx)
    assert o.num_states == l.num_states
    for s in range(o.num_states):
        for b in range(128):
            assert o.step(s, b) == l.rx_fsm_step(s, b)
        assert o.accepting[s] == l.rx_fsm_is_accepting(s)
        assert o.allowed(s) == l.rx_fsm_allowed(s)
        assert o.jump(s) == l.rx_fsm_jump(s)
    assert l.rx_fsm_step(o.num_states, 0) == -1 and l.rx_fsm_step(0, 128) == -1


@pytest.mark.parametrize("bad", ["(", "a)", "[ab", "*a", "a{3,1}", "a{", "a|*"])
def test_library_fsm_syntax_errors(bad):
    with pytest.raises(RxError):
        Fsm(bad)


# ------------------------------------------------------------------ JSON decoding workload (plan pass)
def _json_runs(n_req=10, **kw):
    from oracle.driver import OracleEngine
    from paper_2312_07104_b200.engine import Engine
    from rxgen import workloads
    out = {}
    for comp in (True, False):
        wl = workloads.json_decode(n_req=n_req, compressed=comp, **kw)
        e = Engine(wl, plan_only=True, record=True)
        e.run_workload()
        o = OracleEngine(wl)
        o.run_workload()
        out[comp] = (wl, e, o)
    return out


def test_json_trace_equal_and_modes_agree():
    """Library flow (C++ FSM + tree) == oracle flow (Python FSM + tree) in both modes; both modes
    produce the same token streams (jump forward changes how many passes, not what is decoded),
    every output is valid JSON matching the regex, and the compressed mode needs exactly
    1 + (#sampled tokens) passes per request while the normal mode needs 1 + (#output tokens)."""
    import json as _json
    from rxgen import workloads
    runs = _json_runs()
    cre = re.compile(workloads.JSON_REGEX)
    streams = {}
    for comp, (wl, e, o) in runs.items():
        assert o.trace == e.trace
        ins = [t for t in o.trace if t[0] == "insert"]
        assert len(ins) == 11                                     # hint + 10 requests
        streams[comp] = [t for t in o.trace if t[0] in ("match", "insert", "dec_ref")]
    assert streams[True][1:] != [] and len(streams[True]) == len(streams[False])
    wl_c, e_c, o_c = runs[True]
    wl_n, e_n, o_n = runs[False]
    # same decoded text in both modes
    fsm = FSM(workloads.JSON_REGEX)
    forced0 = len(fsm.jump(0)[0])
    n_out_total = 0
    fc = {k[1]: v for k, v in e_c._full_cache.items() if k[0] == "fsm"}
    fn = {k[1]: v for k, v in e_n._full_cache.items() if k[0] == "fsm"}
    assert fc.keys() == fn.keys() and len(fc) == 10
    for tag in fc:
        assert list(fc[tag][0]) == list(fn[tag][0])
        assert fn[tag][2] == 0 and all(x == 1 for x in fn[tag][3])
    texts = []
    for key, val in e_c._full_cache.items():
        if key[0] != "fsm":
            continue
        toks, hs, first, segs = val
        n_prompt = key[2]
        out = bytes(int(t) - 1 for t in toks[n_prompt:]).decode()
        assert cre.fullmatch(out), out
        obj = _json.loads(out)
        assert set(obj) == {"name", "age", "occupation", "city", "skills", "summary"}
        assert first == forced0 and sum(segs) + first == len(toks) - n_prompt
        n_out_total += len(toks) - n_prompt
        texts.append(out)
    assert len(set(texts)) == len(texts)                           # requests decode different objects
    # passes: normal = 1 prefill + one per output token (lockstep: max over the batch)
    assert o_n.decode_calls == max(len(e_n._full_cache[k][0]) - k[2] for k in e_n._full_cache if k[0] == "fsm")
    assert o_c.extend_calls + o_c.decode_calls < o_n.extend_calls + o_n.decode_calls
