"""ORACLE (test infrastructure only — never imported by the product path).

Compressed finite-state machine for constrained decoding (§4, App. B P:680-688;
SURVEY §8(f) NEXT-4), written step by step from the paper:

  "converting a regular expression into a finite state machine (FSM)" — here a Thompson
  NFA over bytes and the subset construction, the textbook route;
  "compresses adjacent singular-transition edges in the FSM into single edges" — a state
  is *singular* when it has exactly one outgoing transition and is not accepting (an accepting
  state also allows stopping, so it is a choice point); a compressed edge follows singular states
  until the first non-singular one;
  "Jump Forward": at a singular state the whole compressed edge is emitted at once.

Reading R26: the vocabulary is byte-level (one token per byte, token = byte + 1), so
"retokenization" of the jumped string is the identity; the grammar is a regex subset:
literals, escapes (\\d \\w \\s and escaped punctuation), classes [..] with ranges and ^, '.', groups
(...), alternation |, and the quantifiers * + ? {m} {m,} {m,n}.

Reading R27: the DFA is the minimal one (dead states dropped, equivalent states merged), numbered in
breadth-first order from the start state visiting transitions by ascending byte; the minimal DFA
is unique up to renaming and this numbering fixes the names, so two correct implementations agree
state for state.
"""
from __future__ import annotations

from collections import deque

ALPHABET = range(128)   # ASCII


# ------------------------------------------------------------------ regex -> AST
class _Parser:
    def __init__(self, s: str):
        self.s = s
        self.i = 0

    def peek(self):
        return self.s[self.i] if self.i < len(self.s) else None

    def take(self):
        c = self.s[self.i]
        self.i += 1
        return c

    def parse(self):
        node = self.alt()
        if self.i != len(self.s):
            raise ValueError(f"unexpected {self.s[self.i]!r} at {self.i}")
        return node

    def alt(self):
        branches = [self.concat()]
        while self.peek() == "|":
            self.take()
            branches.append(self.concat())
        return branches[0] if len(branches) == 1 else ("alt", branches)

    def concat(self):
        items = []
        while self.peek() is not None and self.peek() not in "|)":
            items.append(self.repeat())
        return ("cat", items)

    def repeat(self):
        atom = self.atom()
        while self.peek() is not None and self.peek() in "*+?{":
            c = self.take()
            if c == "*":
                atom = ("rep", atom, 0, None)
            elif c == "+":
                atom = ("rep", atom, 1, None)
            elif c == "?":
                atom = ("rep", atom, 0, 1)
            else:
                j = self.s.index("}", self.i)
                body = self.s[self.i:j]
                self.i = j + 1
                if "," in body:
                    a, b = body.split(",", 1)
                    lo, hi = int(a), (int(b) if b.strip() else None)
                else:
                    lo = hi = int(body)
                if hi is not None and hi < lo:
                    raise ValueError("bad repeat bounds")
                atom = ("rep", atom, lo, hi)
        return atom

    def atom(self):
        c = self.take()
        if c == "(":
            node = self.alt()
            if self.peek() != ")":
                raise ValueError("unbalanced (")
            self.take()
            return node
        if c == "[":
            return ("set", self.char_class())
        if c == ".":
            return ("set", frozenset(b for b in ALPHABET if b != ord("\n")))
        if c == "\\":
            return ("set", self.escape())
        if c in "*+?{)|":
            raise ValueError(f"unexpected {c!r}")
        return ("set", frozenset([ord(c)]))

    def escape(self):
        c = self.take()
        if c == "d":
            return frozenset(range(ord("0"), ord("9") + 1))
        if c == "w":
            return frozenset([*range(ord("0"), ord("9") + 1), *range(ord("a"), ord("z") + 1),
                              *range(ord("A"), ord("Z") + 1), ord("_")])
        if c == "s":
            return frozenset(map(ord, " \t\n\r\f\v"))
        if c == "n":
            return frozenset([ord("\n")])
        if c == "t":
            return frozenset([ord("\t")])
        return frozenset([ord(c)])

    def char_class(self):
        neg = False
        if self.peek() == "^":
            self.take()
            neg = True
        out = set()
        first = True
        while True:
            c = self.peek()
            if c is None:
                raise ValueError("unbalanced [")
            if c == "]" and not first:
                self.take()
                break
            first = False
            self.take()
            if c == "\\":
                lo_set = self.escape()
                if len(lo_set) != 1:
                    out |= lo_set
                    continue
                lo = next(iter(lo_set))
            else:
                lo = ord(c)
            if self.peek() == "-" and self.i + 1 < len(self.s) and self.s[self.i + 1] != "]":
                self.take()
                h = self.take()
                hi = next(iter(self.escape())) if h == "\\" else ord(h)
                out |= set(range(lo, hi + 1))
            else:
                out.add(lo)
        if neg:
            out = set(ALPHABET) - out
        return frozenset(b for b in out if b in ALPHABET)


# ------------------------------------------------------------------ AST -> Thompson NFA
class _NFA:
    def __init__(self):
        self.eps = []      # state -> list of states
        self.edges = []    # state -> list of (frozenset bytes, state)

    def new(self):
        self.eps.append([])
        self.edges.append([])
        return len(self.eps) - 1

    def build(self, node):
        """-> (start, end) fragment"""
        kind = node[0]
        if kind == "set":
            a, b = self.new(), self.new()
            self.edges[a].append((node[1], b))
            return a, b
        if kind == "cat":
            a = self.new()
            cur = a
            for item in node[1]:
                s, e = self.build(item)
                self.eps[cur].append(s)
                cur = e
            return a, cur
        if kind == "alt":
            a, b = self.new(), self.new()
            for br in node[1]:
                s, e = self.build(br)
                self.eps[a].append(s)
                self.eps[e].append(b)
            return a, b
        if kind == "rep":
            _, sub, lo, hi = node
            a = self.new()
            cur = a
            for _ in range(lo):                       # mandatory copies
                s, e = self.build(sub)
                self.eps[cur].append(s)
                cur = e
            if hi is None:                            # Kleene star on one more copy
                s, e = self.build(sub)
                b = self.new()
                self.eps[cur] += [s, b]
                self.eps[e] += [s, b]
                return a, b
            b = self.new()
            self.eps[cur].append(b)
            for _ in range(hi - lo):                  # optional copies
                s, e = self.build(sub)
                self.eps[cur].append(s)
                self.eps[e].append(b)
                cur = e
            return a, b
        raise ValueError(kind)

    def closure(self, states):
        out = set(states)
        stack = list(states)
        while stack:
            s = stack.pop()
            for t in self.eps[s]:
                if t not in out:
                    out.add(t)
                    stack.append(t)
        return frozenset(out)


# ------------------------------------------------------------------ subset construction + compression
class FSM:
    """Minimal DFA over ASCII bytes with canonical numbering (R27) and compressed edges."""

    def __init__(self, regex: str):
        ast = _Parser(regex).parse()
        nfa = _NFA()
        start, end = nfa.build(ast)
        # subset construction (textbook), exploring transitions by ascending byte
        s0 = nfa.closure([start])
        sets = {s0: 0}
        order = [s0]
        trans = [{}]
        q = deque([s0])
        while q:
            S = q.popleft()
            i = sets[S]
            for b in ALPHABET:
                nxt = set()
                for s in S:
                    for cs, t in nfa.edges[s]:
                        if b in cs:
                            nxt.add(t)
                if not nxt:
                    continue
                T = nfa.closure(nxt)
                if T not in sets:
                    sets[T] = len(order)
                    order.append(T)
                    trans.append({})
                    q.append(T)
                trans[i][b] = sets[T]
        acc = [end in S for S in order]
        # keep states that can reach an accepting state (drop dead ones), then renumber BFS (R27)
        live = {i for i in range(len(order)) if acc[i]}
        changed = True
        while changed:
            changed = False
            for i in range(len(order)):
                if i not in live and any(t in live for t in trans[i].values()):
                    live.add(i)
                    changed = True
        if 0 not in live:
            raise ValueError("regex matches nothing")
        trans = [{b: t for b, t in trans[i].items() if t in live} for i in range(len(order))]
        # minimise (Moore's partition refinement; a missing transition goes to the implicit dead
        # state): the minimal DFA is unique up to isomorphism, so with the BFS numbering below
        # any correct construction yields the same state ids (R27)
        cls = {i: int(acc[i]) for i in live}
        while True:
            sig = {i: (cls[i], tuple(sorted((b, cls[t]) for b, t in trans[i].items()))) for i in live}
            ids = {}
            new_cls = {i: ids.setdefault(sig[i], len(ids)) for i in sorted(live)}
            if len(ids) == len(set(cls.values())):
                break
            cls = new_cls
        cls = new_cls
        rep = {}
        for i in sorted(live):
            rep.setdefault(cls[i], i)
        new_id = {cls[0]: 0}
        bfs = deque([cls[0]])
        while bfs:
            c = bfs.popleft()
            i = rep[c]
            for b in sorted(trans[i]):
                tc = cls[trans[i][b]]
                if tc not in new_id:
                    new_id[tc] = len(new_id)
                    bfs.append(tc)
        n = len(new_id)
        self.trans = [dict() for _ in range(n)]
        self.accepting = [False] * n
        for c, new in new_id.items():
            i = rep[c]
            self.accepting[new] = acc[i]
            for b, t in trans[i].items():
                self.trans[new][b] = new_id[cls[t]]

    @property
    def num_states(self):
        return len(self.trans)

    def step(self, state: int, byte: int) -> int:
        """next state, or -1 when the byte is not allowed"""
        return self.trans[state].get(byte, -1)

    def allowed(self, state: int):
        """bytes allowed at `state`, ascending"""
        return sorted(self.trans[state])

    def singular(self, state: int) -> bool:
        """exactly one outgoing transition and no option to stop"""
        return len(self.trans[state]) == 1 and not self.accepting[state]

    def jump(self, state: int):
        """Jump Forward: the compressed edge from `state` -> (bytes, end state).
        Empty when `state` is not singular."""
        out = []
        seen = set()
        while self.singular(state) and state not in seen:
            seen.add(state)
            (b, t), = self.trans[state].items()
            out.append(b)
            state = t
        return out, state

    def matches(self, s: bytes) -> bool:
        st = 0
        for b in s:
            st = self.step(st, b)
            if st < 0:
                return False
        return self.accepting[st]
