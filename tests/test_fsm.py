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
    rng = random.Random(hash(rx) & 0xFFFF)
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
