// fsm.cc — compressed finite-state machine for constrained decoding (§4 P:255-266,
// App. B).  Host C++ behind the C ABI (include/rx.h, rx_fsm_*).
//
//   regex --(recursive-descent parse)--> AST --(Thompson)--> NFA --(subset construction)--> DFA
//   --(trim dead states, Moore refinement)--> minimal DFA, numbered breadth-first from the start
//   state by ascending byte (reading R27: the minimal DFA with this numbering is unique, so the
//   oracle and this library agree state for state).
//
// Compression ("compresses adjacent singular-transition edges ... into single edges"): a
// state is singular when it has exactly one outgoing byte and is not accepting; rx_fsm_jump
// follows singular states and returns the whole compressed edge (Jump Forward).  Byte-level
// vocabulary (reading R26), so retokenization is the identity.
#include <algorithm>
#include <array>
#include <bitset>
#include <cstdint>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "rx.h"

namespace {

constexpr int kSigma = 128;  // ASCII
using ByteSet = std::bitset<kSigma>;

// ---------------------------------------------------------------- AST
struct Ast {
  enum Kind { kSet, kCat, kAlt, kRep } kind;
  ByteSet set;
  std::vector<std::unique_ptr<Ast>> kids;
  int lo = 0, hi = -1;  // kRep: hi = -1 means unbounded
};
using AstP = std::unique_ptr<Ast>;

struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

class Parser {
 public:
  Parser(const char* s, size_t n) : s_(s), n_(n) {}
  AstP Parse() {
    AstP a = Alternation();
    if (i_ != n_) throw ParseError("trailing input");
    return a;
  }

 private:
  const char* s_;
  size_t n_, i_ = 0;
  bool More() const { return i_ < n_; }
  char Peek() const { return s_[i_]; }
  char Take() {
    if (!More()) throw ParseError("unexpected end");
    return s_[i_++];
  }

  AstP Alternation() {
    auto alt = std::make_unique<Ast>();
    alt->kind = Ast::kAlt;
    alt->kids.push_back(Concatenation());
    while (More() && Peek() == '|') {
      ++i_;
      alt->kids.push_back(Concatenation());
    }
    if (alt->kids.size() == 1) return std::move(alt->kids[0]);
    return alt;
  }
  AstP Concatenation() {
    auto cat = std::make_unique<Ast>();
    cat->kind = Ast::kCat;
    while (More() && Peek() != '|' && Peek() != ')') cat->kids.push_back(Repetition());
    return cat;
  }
  int Number() {
    int v = 0, digits = 0;
    while (More() && Peek() >= '0' && Peek() <= '9') {
      v = v * 10 + (Take() - '0');
      if (++digits > 6) throw ParseError("repeat bound too large");
    }
    if (!digits) throw ParseError("expected a number");
    return v;
  }
  AstP Repetition() {
    AstP a = Atom();
    while (More() && (Peek() == '*' || Peek() == '+' || Peek() == '?' || Peek() == '{')) {
      auto r = std::make_unique<Ast>();
      r->kind = Ast::kRep;
      char c = Take();
      if (c == '*') {
        r->lo = 0, r->hi = -1;
      } else if (c == '+') {
        r->lo = 1, r->hi = -1;
      } else if (c == '?') {
        r->lo = 0, r->hi = 1;
      } else {
        r->lo = Number();
        r->hi = r->lo;
        if (More() && Peek() == ',') {
          ++i_;
          r->hi = (More() && Peek() == '}') ? -1 : Number();
        }
        if (Take() != '}') throw ParseError("expected }");
        if (r->hi != -1 && r->hi < r->lo) throw ParseError("bad repeat bounds");
      }
      r->kids.push_back(std::move(a));
      a = std::move(r);
    }
    return a;
  }
  static ByteSet Range(int a, int b) {
    ByteSet s;
    for (int c = a; c <= b && c < kSigma; ++c) s.set(size_t(c));
    return s;
  }
  ByteSet Escape() {
    char c = Take();
    switch (c) {
      case 'd': return Range('0', '9');
      case 'w': return Range('0', '9') | Range('a', 'z') | Range('A', 'Z') | Range('_', '_');
      case 's': {
        ByteSet s;
        for (char x : std::string(" \t\n\r\f\v")) s.set(size_t(x));
        return s;
      }
      case 'n': return Range('\n', '\n');
      case 't': return Range('\t', '\t');
      default: return Range((unsigned char)c, (unsigned char)c);
    }
  }
  ByteSet Class() {
    bool neg = false;
    if (More() && Peek() == '^') {
      ++i_;
      neg = true;
    }
    ByteSet out;
    bool first = true;
    for (;;) {
      if (!More()) throw ParseError("unbalanced [");
      char c = Take();
      if (c == ']' && !first) break;
      first = false;
      int lo;
      if (c == '\\') {
        ByteSet e = Escape();
        if (e.count() != 1) {
          out |= e;
          continue;
        }
        lo = 0;
        while (!e.test(size_t(lo))) ++lo;
      } else {
        lo = (unsigned char)c;
      }
      if (More() && Peek() == '-' && i_ + 1 < n_ && s_[i_ + 1] != ']') {
        ++i_;
        char h = Take();
        int hi;
        if (h == '\\') {
          ByteSet e = Escape();
          hi = 0;
          while (hi < kSigma && !e.test(size_t(hi))) ++hi;
        } else {
          hi = (unsigned char)h;
        }
        out |= Range(lo, hi);
      } else if (lo < kSigma) {
        out.set(size_t(lo));
      }
    }
    if (neg) out.flip();
    return out;
  }
  AstP Atom() {
    char c = Take();
    auto a = std::make_unique<Ast>();
    a->kind = Ast::kSet;
    if (c == '(') {
      AstP inner = Alternation();
      if (Take() != ')') throw ParseError("unbalanced (");
      return inner;
    }
    if (c == '[') {
      a->set = Class();
    } else if (c == '.') {
      a->set.set();
      a->set.reset(size_t('\n'));
    } else if (c == '\\') {
      a->set = Escape();
    } else if (c == '*' || c == '+' || c == '?' || c == '{' || c == ')' || c == '|') {
      throw ParseError("misplaced operator");
    } else {
      if ((unsigned char)c >= kSigma) throw ParseError("non-ASCII byte");
      a->set.set(size_t((unsigned char)c));
    }
    return a;
  }
};

// ---------------------------------------------------------------- Thompson NFA
struct Nfa {
  std::vector<std::vector<int>> eps;
  std::vector<std::vector<std::pair<ByteSet, int>>> edge;
  int New() {
    eps.emplace_back();
    edge.emplace_back();
    if (eps.size() > (1u << 20)) throw ParseError("NFA too large");
    return int(eps.size()) - 1;
  }
  // returns {start, end}
  std::pair<int, int> Build(const Ast& a) {
    switch (a.kind) {
      case Ast::kSet: {
        int s = New(), e = New();
        edge[size_t(s)].push_back({a.set, e});
        return {s, e};
      }
      case Ast::kCat: {
        int s = New(), cur = s;
        for (auto& k : a.kids) {
          auto f = Build(*k);
          eps[size_t(cur)].push_back(f.first);
          cur = f.second;
        }
        return {s, cur};
      }
      case Ast::kAlt: {
        int s = New(), e = New();
        for (auto& k : a.kids) {
          auto f = Build(*k);
          eps[size_t(s)].push_back(f.first);
          eps[size_t(f.second)].push_back(e);
        }
        return {s, e};
      }
      case Ast::kRep: {
        int s = New(), cur = s;
        for (int i = 0; i < a.lo; ++i) {
          auto f = Build(*a.kids[0]);
          eps[size_t(cur)].push_back(f.first);
          cur = f.second;
        }
        int e = New();
        if (a.hi < 0) {
          auto f = Build(*a.kids[0]);
          eps[size_t(cur)].push_back(f.first);
          eps[size_t(cur)].push_back(e);
          eps[size_t(f.second)].push_back(f.first);
          eps[size_t(f.second)].push_back(e);
          return {s, e};
        }
        eps[size_t(cur)].push_back(e);
        for (int i = a.lo; i < a.hi; ++i) {
          auto f = Build(*a.kids[0]);
          eps[size_t(cur)].push_back(f.first);
          eps[size_t(f.second)].push_back(e);
          cur = f.second;
        }
        return {s, e};
      }
    }
    throw ParseError("bad AST");
  }
  void Closure(std::vector<int>& set) const {
    std::vector<char> in(eps.size(), 0);
    for (int s : set) in[size_t(s)] = 1;
    std::vector<int> stack(set);
    while (!stack.empty()) {
      int s = stack.back();
      stack.pop_back();
      for (int t : eps[size_t(s)])
        if (!in[size_t(t)]) {
          in[size_t(t)] = 1;
          set.push_back(t);
          stack.push_back(t);
        }
    }
    std::sort(set.begin(), set.end());
  }
};

}  // namespace

struct rx_fsm {
  int32_t n = 0;
  std::vector<std::array<int32_t, kSigma>> next;  // -1 = not allowed
  std::vector<uint8_t> accept;
  std::vector<int16_t> out_degree;
};

namespace {

void BuildFsm(const char* re, size_t len, rx_fsm* f) {
  AstP ast = Parser(re, len).Parse();
  Nfa nfa;
  auto [start, end] = nfa.Build(*ast);
  // subset construction
  std::map<std::vector<int>, int> id;
  std::vector<std::vector<int>> sets;
  std::vector<std::array<int32_t, kSigma>> tr;
  std::vector<int> s0{start};
  nfa.Closure(s0);
  id[s0] = 0;
  sets.push_back(s0);
  tr.emplace_back();
  tr.back().fill(-1);
  for (size_t q = 0; q < sets.size(); ++q) {
    for (int b = 0; b < kSigma; ++b) {
      std::vector<int> nx;
      for (int s : sets[q])
        for (auto& [cs, t] : nfa.edge[size_t(s)])
          if (cs.test(size_t(b))) nx.push_back(t);
      if (nx.empty()) continue;
      std::sort(nx.begin(), nx.end());
      nx.erase(std::unique(nx.begin(), nx.end()), nx.end());
      nfa.Closure(nx);
      auto it = id.find(nx);
      int t;
      if (it == id.end()) {
        t = int(sets.size());
        if (t > (1 << 16)) throw ParseError("DFA too large");
        id.emplace(nx, t);
        sets.push_back(nx);
        tr.emplace_back();
        tr.back().fill(-1);
      } else {
        t = it->second;
      }
      tr[q][size_t(b)] = t;
    }
  }
  const int nd = int(sets.size());
  std::vector<char> acc(static_cast<size_t>(nd));
  for (int q = 0; q < nd; ++q) acc[size_t(q)] = std::binary_search(sets[size_t(q)].begin(), sets[size_t(q)].end(), end);
  // trim: live = can reach an accepting state (reverse reachability)
  std::vector<std::vector<int>> rev(static_cast<size_t>(nd));
  for (int q = 0; q < nd; ++q)
    for (int b = 0; b < kSigma; ++b)
      if (tr[size_t(q)][size_t(b)] >= 0) rev[size_t(tr[size_t(q)][size_t(b)])].push_back(q);
  std::vector<char> live(static_cast<size_t>(nd), 0);
  std::deque<int> work;
  for (int q = 0; q < nd; ++q)
    if (acc[size_t(q)]) live[size_t(q)] = 1, work.push_back(q);
  while (!work.empty()) {
    int q = work.front();
    work.pop_front();
    for (int p : rev[size_t(q)])
      if (!live[size_t(p)]) live[size_t(p)] = 1, work.push_back(p);
  }
  if (!live[0]) throw ParseError("empty language");
  for (int q = 0; q < nd; ++q)
    for (int b = 0; b < kSigma; ++b) {
      int32_t& t = tr[size_t(q)][size_t(b)];
      if (t >= 0 && !live[size_t(t)]) t = -1;
    }
  // Moore refinement over live states (dead = implicit class -1)
  std::vector<int> cls(static_cast<size_t>(nd), -1);
  int ncls = 0;
  {
    int a = -1, r = -1;
    for (int q = 0; q < nd; ++q)
      if (live[size_t(q)]) {
        int& k = acc[size_t(q)] ? a : r;
        if (k < 0) k = ncls++;
        cls[size_t(q)] = k;
      }
  }
  for (;;) {
    std::map<std::vector<int>, int> sig_id;
    std::vector<int> nc(static_cast<size_t>(nd), -1);
    for (int q = 0; q < nd; ++q) {
      if (!live[size_t(q)]) continue;
      std::vector<int> sig;
      sig.reserve(kSigma + 1);
      sig.push_back(cls[size_t(q)]);
      for (int b = 0; b < kSigma; ++b) {
        int t = tr[size_t(q)][size_t(b)];
        sig.push_back(t >= 0 ? cls[size_t(t)] : -1);
      }
      auto it = sig_id.emplace(std::move(sig), int(sig_id.size())).first;
      nc[size_t(q)] = it->second;
    }
    const int n2 = int(sig_id.size());
    cls.swap(nc);
    if (n2 == ncls) break;
    ncls = n2;
  }
  // canonical BFS numbering of the classes
  std::vector<int> rep(static_cast<size_t>(ncls), -1), num(static_cast<size_t>(ncls), -1);
  for (int q = 0; q < nd; ++q)
    if (live[size_t(q)] && rep[size_t(cls[size_t(q)])] < 0) rep[size_t(cls[size_t(q)])] = q;
  std::vector<int> order{cls[0]};
  num[size_t(cls[0])] = 0;
  for (size_t i = 0; i < order.size(); ++i) {
    int q = rep[size_t(order[i])];
    for (int b = 0; b < kSigma; ++b) {
      int t = tr[size_t(q)][size_t(b)];
      if (t < 0) continue;
      int c = cls[size_t(t)];
      if (num[size_t(c)] < 0) {
        num[size_t(c)] = int(order.size());
        order.push_back(c);
      }
    }
  }
  f->n = int32_t(order.size());
  f->next.assign(size_t(f->n), {});
  f->accept.assign(size_t(f->n), 0);
  f->out_degree.assign(size_t(f->n), 0);
  for (int i = 0; i < f->n; ++i) {
    int q = rep[size_t(order[size_t(i)])];
    f->accept[size_t(i)] = uint8_t(acc[size_t(q)]);
    for (int b = 0; b < kSigma; ++b) {
      int t = tr[size_t(q)][size_t(b)];
      f->next[size_t(i)][size_t(b)] = t >= 0 ? num[size_t(cls[size_t(t)])] : -1;
      f->out_degree[size_t(i)] += t >= 0;
    }
  }
}

inline bool Singular(const rx_fsm* f, int32_t s) { return f->out_degree[size_t(s)] == 1 && !f->accept[size_t(s)]; }

}  // namespace

extern "C" {

rx_status rx_fsm_create(const char* regex, int64_t len, rx_fsm** out) {
  if (!out || (!regex && len > 0) || len < 0) return RX_E_INVALID;
  *out = nullptr;
  auto f = std::make_unique<rx_fsm>();
  try {
    BuildFsm(regex ? regex : "", size_t(len), f.get());
  } catch (const ParseError&) {
    return RX_E_INVALID;
  } catch (const std::bad_alloc&) {
    return RX_E_NOMEM;
  }
  *out = f.release();
  return RX_OK;
}

void rx_fsm_destroy(rx_fsm* f) { delete f; }

int32_t rx_fsm_num_states(const rx_fsm* f) { return f ? f->n : -1; }

int32_t rx_fsm_step(const rx_fsm* f, int32_t state, int32_t byte) {
  if (!f || state < 0 || state >= f->n || byte < 0 || byte >= kSigma) return -1;
  return f->next[size_t(state)][size_t(byte)];
}

int32_t rx_fsm_is_accepting(const rx_fsm* f, int32_t state) {
  if (!f || state < 0 || state >= f->n) return -1;
  return f->accept[size_t(state)];
}

int32_t rx_fsm_allowed(const rx_fsm* f, int32_t state, uint8_t* out) {
  if (!f || state < 0 || state >= f->n) return -1;
  int32_t k = 0;
  for (int b = 0; b < kSigma; ++b)
    if (f->next[size_t(state)][size_t(b)] >= 0) {
      if (out) out[k] = uint8_t(b);
      ++k;
    }
  return k;
}

int32_t rx_fsm_jump(const rx_fsm* f, int32_t state, uint8_t* out, int32_t cap, int32_t* end_state) {
  if (!f || state < 0 || state >= f->n || cap < 0) return -1;
  int32_t k = 0;
  // a singular chain visits each state at most once (every kept state reaches acceptance)
  while (Singular(f, state)) {
    int b = 0;
    while (f->next[size_t(state)][size_t(b)] < 0) ++b;
    if (k >= cap) return -1;
    if (out) out[k] = uint8_t(b);
    ++k;
    state = f->next[size_t(state)][size_t(b)];
  }
  if (end_state) *end_state = state;
  return k;
}

}  // extern "C"
