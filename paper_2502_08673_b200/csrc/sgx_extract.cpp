// Circuit extraction (Algorithm 1 of arXiv 2502.08673) and the gate-level
// build, natively: CNF -> ExtractionResult -> Circuit, with the reference's
// exact decisions (extract.cpp:43-172), Boolean algebra (boolexpr.cpp) and
// netlist construction (circuit.cpp:60-122), so the circuit -- node for node --
// equals what satgrad builds for the same CNF.  Paths are relative to
// /root/reference/proj.
//
// What is different is the cost model.  The reference re-scans every
// variable of the sub-clause buffer after each appended clause, building
// expression trees and truth tables for each, and rebuilds a hash set of the
// buffer's variables per clause (shares_var): quadratic in the buffer, which
// is what makes extraction slow on large CNFs.  Here:
//   * expressions are hash-consed (structural equality is id equality, and a
//     decomposition memo is keyed by id);
//   * the complement test of a candidate runs on truth tables built directly
//     from its clauses -- no expression is built unless it succeeds;
//   * a candidate's outcome is a function of the buffered clauses that mention
//     it (and its role, which only changes together with them), so a failed
//     candidate is cached until one of its clauses arrives or leaves; each
//     appended clause re-tests only the variables whose clause set changed, in
//     the reference's descending order;
//   * per-variable occurrence counts replace shares_var's set rebuild.
#include "sgx_extract.hpp"

#include <algorithm>
#include <cstring>
#include <set>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

namespace sgx::ext {

namespace {

// ExprKind order of boolexpr.hpp (compare() orders by it).
enum Kind : uint8_t { kC0, kC1, kVar, kNot, kAnd, kOr, kXor, kXnor };

constexpr int kMaxTT = 16;  // kMaxTruthTableVars, truth_table.hpp

// ---------------------------------------------------------------- truth tables
// Bit r of a table over n variables is the function at the assignment whose
// variable i is (r >> i) & 1 (truth_table.hpp).
struct TT {
  // one inline word for <= 6 variables (nearly every table), heap words above
  int n = 0;
  size_t nw = 1;
  uint64_t one = 0;
  std::vector<uint64_t> big;
  explicit TT(int nv = 0) : n(nv), nw(nv <= 6 ? 1 : size_t{1} << (nv - 6)) {
    if (nw > 1) big.assign(nw, 0);
  }
  uint64_t* w() { return nw == 1 ? &one : big.data(); }
  const uint64_t* w() const { return nw == 1 ? &one : big.data(); }
  uint64_t top() const { return n >= 6 ? ~0ull : ((1ull << (1u << n)) - 1ull); }
  void mask() { w()[nw - 1] &= top(); }
  static TT var(int nv, int i) {
    static const uint64_t pat[6] = {0xAAAAAAAAAAAAAAAAull, 0xCCCCCCCCCCCCCCCCull, 0xF0F0F0F0F0F0F0F0ull,
                                    0xFF00FF00FF00FF00ull, 0xFFFF0000FFFF0000ull, 0xFFFFFFFF00000000ull};
    TT t(nv);
    uint64_t* x = t.w();
    for (size_t j = 0; j < t.nw; ++j) x[j] = i < 6 ? pat[i] : (((j >> (i - 6)) & 1) ? ~0ull : 0ull);
    t.mask();
    return t;
  }
  void flip() {
    uint64_t* x = w();
    for (size_t j = 0; j < nw; ++j) x[j] = ~x[j];
    mask();
  }
  bool zero() const {
    const uint64_t* x = w();
    for (size_t j = 0; j < nw; ++j)
      if (x[j]) return false;
    return true;
  }
  bool ones() const {
    const uint64_t* x = w();
    for (size_t j = 0; j + 1 < nw; ++j)
      if (x[j] != ~0ull) return false;
    return x[nw - 1] == top();
  }
  bool complement_of(const TT& o) const {
    const uint64_t *x = w(), *y = o.w();
    for (size_t j = 0; j + 1 < nw; ++j)
      if ((x[j] ^ y[j]) != ~0ull) return false;
    return (x[nw - 1] ^ y[nw - 1]) == top();
  }
  bool operator==(const TT& o) const { return nw == o.nw && std::equal(w(), w() + nw, o.w()); }
  bool bit(uint32_t r) const { return (w()[r >> 6] >> (r & 63)) & 1ull; }
  uint32_t rows() const { return 1u << n; }
};

TT parity_tt(int nv) {
  TT t(nv);
  for (int i = 0; i < nv; ++i) {
    const TT v = TT::var(nv, i);
    for (size_t j = 0; j < t.nw; ++j) t.w()[j] ^= v.w()[j];
  }
  return t;
}

// ------------------------------------------------------- hash-consed exprs
class Exprs {
 public:
  Exprs() {
    mk(kC0, 0, nullptr, 0);  // id 0
    mk(kC1, 0, nullptr, 0);  // id 1
  }
  Kind kind(int e) const { return static_cast<Kind>(nodes_[e].kind); }
  int var(int e) const { return nodes_[e].var; }
  int nkids(int e) const { return nodes_[e].n; }
  const int* kids(int e) const { return kids_.data() + nodes_[e].off; }
  bool is_const(int e) const { return e <= 1; }

  // boolexpr.cpp:22-46 (distinct ids are structurally distinct)
  int compare(int a, int b) const {
    if (a == b) return 0;
    if (kind(a) != kind(b)) return kind(a) < kind(b) ? -1 : 1;
    if (kind(a) == kVar) return var(a) < var(b) ? -1 : (var(a) > var(b) ? 1 : 0);
    const int na = nkids(a), nb = nkids(b);
    const int n = std::min(na, nb);
    for (int i = 0; i < n; ++i) {
      const int c = compare(kids(a)[i], kids(b)[i]);
      if (c != 0) return c;
    }
    return na == nb ? 0 : (na < nb ? -1 : 1);
  }
  void sort(std::vector<int>& v) const {
    std::sort(v.begin(), v.end(), [this](int a, int b) { return compare(a, b) < 0; });
  }

  int cnst(bool v) const { return v ? 1 : 0; }
  int var_expr(int v) {
    if (v <= 0) throw std::invalid_argument("variable index must be positive");
    if (static_cast<size_t>(v) >= var_id_.size()) var_id_.resize(static_cast<size_t>(v) * 2 + 16, -1);
    int& id = var_id_[v];
    if (id < 0) id = mk(kVar, v, nullptr, 0);
    return id;
  }
  // boolexpr.cpp:61-72
  int not_(int e) {
    switch (kind(e)) {
      case kC0: return 1;
      case kC1: return 0;
      case kNot: return kids(e)[0];
      default: return mk(kNot, 0, &e, 1);
    }
  }
  int literal(int lit) {
    if (lit > 0) return var_expr(lit);
    const size_t v = static_cast<size_t>(-lit);
    if (v >= nvar_id_.size()) nvar_id_.resize(v * 2 + 16, -1);
    if (nvar_id_[v] < 0) nvar_id_[v] = not_(var_expr(-lit));
    return nvar_id_[v];
  }

  // boolexpr.cpp:74-132
  int nary(Kind k, const std::vector<int>& es) {
    std::vector<int>& kids = nk_;  // scratch: nary never re-enters itself
    kids.clear();
    if (k == kAnd || k == kOr) {
      const bool is_and = k == kAnd;
      for (int e : es) {
        if (kind(e) == k) {
          for (int i = 0; i < nkids(e); ++i) kids.push_back(kids_[nodes_[e].off + i]);
        } else if (kind(e) == kC0) {
          if (is_and) return 0;
        } else if (kind(e) == kC1) {
          if (!is_and) return 1;
        } else {
          kids.push_back(e);
        }
      }
      if (kids.empty()) return cnst(is_and);
      if (kids.size() == 1) return kids[0];
      sort(kids);
      return mk(k, 0, kids.data(), static_cast<int>(kids.size()));
    }
    bool flip = k == kXnor;
    for (int e : es) {
      switch (kind(e)) {
        case kXor:
          for (int i = 0; i < nkids(e); ++i) kids.push_back(kids_[nodes_[e].off + i]);
          break;
        case kXnor:
          flip = !flip;
          for (int i = 0; i < nkids(e); ++i) kids.push_back(kids_[nodes_[e].off + i]);
          break;
        case kC0:
          break;
        case kC1:
          flip = !flip;
          break;
        default:
          kids.push_back(e);
      }
    }
    if (kids.empty()) return cnst(flip);
    if (kids.size() == 1) return flip ? not_(kids[0]) : kids[0];
    sort(kids);
    return mk(flip ? kXnor : kXor, 0, kids.data(), static_cast<int>(kids.size()));
  }
  std::vector<int> kid_vec(int e) const { return std::vector<int>(kids(e), kids(e) + nkids(e)); }

  // boolexpr.cpp:169-175 (sorted, unique)
  std::vector<int> support(int e) {
    std::vector<int> out;
    ++epoch_;
    if (seen_.size() < nodes_.size()) seen_.resize(nodes_.size() * 2, 0);
    std::vector<int> st{e};
    while (!st.empty()) {
      const int x = st.back();
      st.pop_back();
      if (seen_[x] == epoch_) continue;
      seen_[x] = epoch_;
      if (kind(x) == kVar) {
        out.push_back(var(x));
      } else {
        for (int i = 0; i < nkids(x); ++i) st.push_back(kids(x)[i]);
      }
    }
    std::sort(out.begin(), out.end());
    out.erase(std::unique(out.begin(), out.end()), out.end());
    return out;
  }

  // boolexpr.cpp:210-245
  TT table(int e, const std::vector<int>& vars) const {
    const int n = static_cast<int>(vars.size());
    switch (kind(e)) {
      case kC0: return TT(n);
      case kC1: {
        TT t(n);
        t.flip();
        return t;
      }
      case kVar: {
        const auto it = std::lower_bound(vars.begin(), vars.end(), var(e));
        if (it == vars.end() || *it != var(e)) throw std::invalid_argument("variable order misses x" + std::to_string(var(e)));
        return TT::var(n, static_cast<int>(it - vars.begin()));
      }
      case kNot: {
        TT t = table(kids(e)[0], vars);
        t.flip();
        return t;
      }
      default: {
        TT acc = table(kids(e)[0], vars);
        for (int i = 1; i < nkids(e); ++i) {
          const TT t = table(kids(e)[i], vars);
          uint64_t* x = acc.w();
          const uint64_t* y = t.w();
          for (size_t j = 0; j < acc.nw; ++j)
            x[j] = kind(e) == kAnd ? (x[j] & y[j]) : kind(e) == kOr ? (x[j] | y[j]) : (x[j] ^ y[j]);
        }
        if (kind(e) == kXnor) acc.flip();
        return acc;
      }
    }
  }

  // ---- simplify (boolexpr.cpp:286-522)
  int rebuild_and_or(Kind k, const std::vector<int>& sorted) {
    std::vector<int> kids;
    kids.reserve(sorted.size());
    for (int c : sorted)
      if (kids.empty() || kids.back() != c) kids.push_back(c);
    bool any_not = false;
    for (int c : kids) any_not |= kind(c) == kNot;
    if (any_not) {
      ++epoch_;
      if (seen_.size() < nodes_.size()) seen_.resize(nodes_.size() * 2, 0);
      for (int c : kids) seen_[c] = epoch_;
      for (int c : kids)
        if (kind(c) == kNot && seen_[kids_[nodes_[c].off]] == epoch_) return cnst(k == kOr);
    }
    return nary(k, kids);
  }
  int rebuild_xor(Kind k, const std::vector<int>& in) {
    bool flip = k == kXnor;
    std::vector<int> kids;
    kids.reserve(in.size());
    for (int c : in) {
      if (kind(c) == kNot) {
        flip = !flip;
        kids.push_back(kids_[nodes_[c].off]);
      } else {
        kids.push_back(c);
      }
    }
    sort(kids);
    std::vector<int> kept;
    for (size_t i = 0; i < kids.size();) {
      if (i + 1 < kids.size() && kids[i] == kids[i + 1]) {
        i += 2;
      } else {
        kept.push_back(kids[i]);
        ++i;
      }
    }
    return nary(flip ? kXnor : kXor, kept);
  }
  int local_pass(int e) {
    switch (kind(e)) {
      case kC0:
      case kC1:
      case kVar: return e;
      case kNot: return not_(local_pass(kids(e)[0]));
      default: {
        const Kind k = kind(e);
        std::vector<int> kids;
        kids.reserve(nkids(e));
        for (int i = 0; i < nkids(e); ++i) kids.push_back(local_pass(kids_[nodes_[e].off + i]));
        const int flat = nary(k, kids);
        if (kind(flat) == kAnd || kind(flat) == kOr) return rebuild_and_or(kind(flat), kid_vec(flat));
        if (kind(flat) == kXor || kind(flat) == kXnor) return rebuild_xor(kind(flat), kid_vec(flat));
        return flat;
      }
    }
  }
  int local_fixpoint(int e) {
    int cur = e;
    for (int round = 0; round < 8; ++round) {
      const int next = local_pass(cur);
      if (next == cur) break;
      cur = next;
    }
    return cur;
  }
  int simplify(int e, int minimize_cap) {
    const int base = local_fixpoint(e);
    if (is_const(base) || kind(base) == kVar) return base;
    const std::vector<int> vars = support(base);
    if (static_cast<int>(vars.size()) > minimize_cap) return base;
    const TT tt = table(base, vars);
    if (tt.zero()) return 0;
    if (tt.ones()) return 1;
    std::vector<int> cand;
    if (vars.size() >= 2) {
      const TT par = parity_tt(static_cast<int>(vars.size()));
      const bool eq = tt == par;
      if (eq || tt.complement_of(par)) {
        std::vector<int> vs;
        for (int v : vars) vs.push_back(var_expr(v));
        cand.push_back(nary(eq ? kXor : kXnor, vs));
      }
    }
    cand.push_back(sop(tt, vars));
    cand.push_back(base);
    size_t best = 0;
    int best_cost = gate_equivalents(cand[0]);
    for (size_t i = 1; i < cand.size(); ++i) {
      const int c = gate_equivalents(cand[i]);
      if (c < best_cost) {
        best_cost = c;
        best = i;
      }
    }
    return cand[best];
  }

  // ---- two-input decomposition (boolexpr.cpp:524-589, circuit.cpp:60-122)
  struct Ref {
    uint8_t src;  // 0 var, 1 gate, 2 const
    int index;
  };
  struct Gate {
    uint8_t op;  // 0 Not, 1 And2, 2 Or2, 3 Xor2, 4 Xnor2
    Ref a, b;
  };
  Ref decompose(int e, std::vector<Gate>& out, std::unordered_map<int, Ref>& memo) {
    if (auto it = memo.find(e); it != memo.end()) return it->second;
    Ref r{};
    switch (kind(e)) {
      case kC0: r = {2, 0}; break;
      case kC1: r = {2, 1}; break;
      case kVar: r = {0, var(e)}; break;
      case kNot: {
        const Ref a = decompose(kids(e)[0], out, memo);
        out.push_back({0, a, {}});
        r = {1, static_cast<int>(out.size()) - 1};
        break;
      }
      default: {
        const Kind k = kind(e);
        const int n = nkids(e);
        std::vector<Ref> refs;
        refs.reserve(n);
        for (int i = 0; i < n; ++i) refs.push_back(decompose(kids_[nodes_[e].off + i], out, memo));
        const uint8_t chain = k == kAnd ? 1 : k == kOr ? 2 : 3;
        Ref acc = refs[0];
        for (int i = 1; i < n; ++i) {
          const uint8_t op = (k == kXnor && i + 1 == n) ? 4 : chain;
          out.push_back({op, acc, refs[i]});
          acc = {1, static_cast<int>(out.size()) - 1};
        }
        r = acc;
      }
    }
    memo.emplace(e, r);
    return r;
  }
  // Non-Not gates of decompose_two_input(e): the decomposition memo gives each
  // distinct subexpression its gates once, and an n-ary node chains n - 1.
  int gate_equivalents(int e) {
    ++epoch_;
    if (seen_.size() < nodes_.size()) seen_.resize(nodes_.size() * 2, 0);
    int n = 0;
    stack_.clear();
    stack_.push_back(e);
    while (!stack_.empty()) {
      const int x = stack_.back();
      stack_.pop_back();
      if (seen_[x] == epoch_) continue;
      seen_[x] = epoch_;
      if (kind(x) >= kAnd) n += nkids(x) - 1;
      for (int i = 0; i < nkids(x); ++i) stack_.push_back(kids(x)[i]);
    }
    return n;
  }

 private:
  struct Node {
    uint8_t kind;
    int var, off, n, next;
  };
  std::vector<Node> nodes_;
  std::vector<int> kids_;
  std::vector<uint32_t> seen_;
  std::vector<int> stack_;
  std::vector<int> var_id_, nvar_id_;  // var -> Var node, var -> Not(Var) node
  std::vector<int> nk_;                // nary scratch
  uint32_t epoch_ = 0;

  static uint64_t mix(uint64_t h, uint64_t x) {
    h ^= x + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
    return h * 0xBF58476D1CE4E5B9ull;
  }
  // open-addressing intern table: slot -> node id (-1 empty), power-of-two size
  std::vector<int> slots_ = std::vector<int>(1 << 12, -1);
  std::vector<uint64_t> hash_;  // per node
  bool same(int x, Kind k, int v, const int* kids, int n) const {
    const Node& nd = nodes_[x];
    return nd.kind == k && nd.var == v && nd.n == n && std::equal(kids, kids + n, kids_.begin() + nd.off);
  }
  int mk(Kind k, int v, const int* kids, int n) {
    uint64_t h = mix(static_cast<uint64_t>(k) + 1, static_cast<uint64_t>(static_cast<uint32_t>(v)));
    for (int i = 0; i < n; ++i) h = mix(h, static_cast<uint64_t>(kids[i]));
    size_t mask = slots_.size() - 1, i = (h ^ (h >> 29)) & mask;
    for (; slots_[i] >= 0; i = (i + 1) & mask)
      if (hash_[slots_[i]] == h && same(slots_[i], k, v, kids, n)) return slots_[i];
    const int id = static_cast<int>(nodes_.size());
    nodes_.push_back({static_cast<uint8_t>(k), v, static_cast<int>(kids_.size()), n, -1});
    kids_.insert(kids_.end(), kids, kids + n);
    hash_.push_back(h);
    slots_[i] = id;
    if (nodes_.size() * 2 > slots_.size()) {  // grow at 50 % load
      std::vector<int> ns(slots_.size() * 2, -1);
      const size_t m2 = ns.size() - 1;
      for (int x = 0; x < static_cast<int>(nodes_.size()); ++x) {
        size_t j = (hash_[x] ^ (hash_[x] >> 29)) & m2;
        while (ns[j] >= 0) j = (j + 1) & m2;
        ns[j] = x;
      }
      slots_.swap(ns);
    }
    return id;
  }

  // Quine-McCluskey + essential primes + greedy cover (boolexpr.cpp:366-478).
  // The prime set of a function is unique, so primes are found by probing
  // each implicant's one-bit neighbours instead of all pairs; the (value,
  // mask) order, the essential pass and the greedy tie-break are the
  // reference's.
  struct Imp {
    uint32_t value, mask;
    bool operator<(const Imp& o) const { return value != o.value ? value < o.value : mask < o.mask; }
    bool operator==(const Imp& o) const { return value == o.value && mask == o.mask; }
    bool covers(uint32_t m) const { return (m & ~mask) == value; }
  };
  std::vector<uint32_t> qm_min_;  // sop scratch (sop never re-enters)
  std::vector<Imp> qm_cur_, qm_next_, qm_primes_;
  std::vector<char> qm_cov_, qm_cho_;
  int sop(const TT& tt, const std::vector<int>& vars) {
    const int nv = static_cast<int>(vars.size());
    std::vector<uint32_t>& minterms = qm_min_;  // scratch (sop never re-enters)
    minterms.clear();
    for (uint32_t r = 0; r < tt.rows(); ++r)
      if (tt.bit(r)) minterms.push_back(r);
    if (minterms.empty()) return 0;
    if (minterms.size() == tt.rows()) return 1;
    std::vector<Imp>&cur = qm_cur_, &primes = qm_primes_, &next = qm_next_;
    cur.clear();
    primes.clear();
    for (uint32_t m : minterms) cur.push_back({m, 0});
    while (!cur.empty()) {
      // cur is sorted and unique (every mask of one popcount)
      auto has = [&](uint32_t value, uint32_t mask) {
        return std::binary_search(cur.begin(), cur.end(), Imp{value, mask});
      };
      next.clear();
      for (const Imp& x : cur) {
        bool combined = false;
        for (int b = 0; b < nv; ++b) {
          const uint32_t d = 1u << b;
          if (x.mask & d) continue;
          if (has(x.value ^ d, x.mask)) {
            combined = true;
            next.push_back({x.value & ~d, x.mask | d});
          }
        }
        if (!combined) primes.push_back(x);
      }
      std::sort(next.begin(), next.end());
      next.erase(std::unique(next.begin(), next.end()), next.end());
      cur.swap(next);
    }
    std::sort(primes.begin(), primes.end());
    primes.erase(std::unique(primes.begin(), primes.end()), primes.end());

    std::vector<char>&covered = qm_cov_, &chosen = qm_cho_;
    covered.assign(minterms.size(), 0);
    chosen.assign(primes.size(), 0);
    size_t uncovered = minterms.size();
    auto take = [&](size_t p) {
      chosen[p] = 1;
      for (size_t mj = 0; mj < minterms.size(); ++mj)
        if (!covered[mj] && primes[p].covers(minterms[mj])) {
          covered[mj] = 1;
          --uncovered;
        }
    };
    for (size_t mi = 0; mi < minterms.size(); ++mi) {
      size_t hits = 0, last = 0;
      for (size_t pi = 0; pi < primes.size(); ++pi)
        if (primes[pi].covers(minterms[mi])) {
          ++hits;
          last = pi;
          if (hits > 1) break;
        }
      if (hits == 1 && !chosen[last]) take(last);
    }
    while (uncovered > 0) {
      size_t best = primes.size(), best_gain = 0;
      for (size_t pi = 0; pi < primes.size(); ++pi) {
        if (chosen[pi]) continue;
        size_t gain = 0;
        for (size_t mj = 0; mj < minterms.size(); ++mj)
          if (!covered[mj] && primes[pi].covers(minterms[mj])) ++gain;
        if (gain > best_gain) {
          best_gain = gain;
          best = pi;
        }
      }
      take(best);
    }
    std::vector<int> terms;
    for (size_t pi = 0; pi < primes.size(); ++pi) {
      if (!chosen[pi]) continue;
      std::vector<int> lits;
      for (int b = 0; b < nv; ++b) {
        if (primes[pi].mask & (1u << b)) continue;
        const int v = var_expr(vars[b]);
        lits.push_back(((primes[pi].value >> b) & 1) ? v : not_(v));
      }
      terms.push_back(nary(kAnd, lits));
    }
    return nary(kOr, terms);
  }
};

// ------------------------------------------------------------- extraction
enum Role : uint8_t { kNone, kPi, kDefined };

class Extractor {
 public:
  Extractor(int num_vars, const int32_t* ptr, const int32_t* lit, int64_t n_clauses, int complement_cap,
            int minimize_cap)
      : nv_(num_vars), ptr_(ptr), lit_(lit), nc_(n_clauses), ccap_(std::min(complement_cap, kMaxTT)),
        mcap_(minimize_cap), role_(num_vars + 1, kNone), cnt_(num_vars + 1, 0), occ_(num_vars + 1),
        po_state_(num_vars + 1, 0), const_def_(num_vars + 1, 0), in_iv_(num_vars + 1, 0) {}

  void run(Result& R) {
    R.num_vars = nv_;
    next_aux_ = nv_;
    alive_.assign(static_cast<size_t>(nc_), 0);
    for (int64_t c = 0; c < nc_; ++c) {
      for (int64_t k = ptr_[c]; k < ptr_[c + 1]; ++k) {
        const int v = std::abs(lit_[k]);
        if (v < 1 || v > nv_) throw std::invalid_argument("literal out of range");
      }
      if (n_alive_ > 0 && !shares_var(c)) fallback(R);
      push(c);
      try_commit(R);
    }
    fallback(R);
    for (int v = 1; v <= nv_; ++v)
      if (role_[v] == kNone) {
        role_[v] = kPi;
        R.pi.push_back(v);
      }
    for (int v : iv_order_)
      if (in_iv_[v]) R.iv.push_back(v);
  }

  Exprs X;
  std::vector<std::pair<int, int>> be;  // (var, expr id), commit order

 private:
  int nv_;
  const int32_t *ptr_, *lit_;
  int64_t nc_;
  int ccap_, mcap_;
  std::vector<Role> role_;
  std::vector<int> cnt_;                 // literal occurrences in the buffer
  std::vector<std::vector<int64_t>> occ_;  // buffered clauses per var, buffer order (lazy: dead ids skipped)
  std::vector<int64_t> sc_;              // buffer, in order (lazy: dead ids skipped)
  std::vector<char> alive_;
  int64_t n_alive_ = 0;
  std::set<int> dirty_;                  // buffered vars whose outcome is not known to fail
  std::vector<uint8_t> po_state_;        // 0 none, 1 target 0, 2 target 1
  std::vector<uint8_t> const_def_;       // 0 none, 1 const 0, 2 const 1
  std::vector<char> in_iv_;
  std::vector<int> iv_order_;
  int next_aux_ = 0;
  std::vector<int> conj_, disj_;  // definition_expr scratch
  std::vector<int> cs_;             // complement scratch
  std::vector<int64_t> cf_, cg_;

  int var_at(int64_t k) const { return std::abs(lit_[k]); }

  bool shares_var(int64_t c) const {
    for (int64_t k = ptr_[c]; k < ptr_[c + 1]; ++k)
      if (cnt_[var_at(k)] > 0) return true;
    return false;
  }
  void push(int64_t c) {
    sc_.push_back(c);
    alive_[c] = 1;
    ++n_alive_;
    for (int64_t k = ptr_[c]; k < ptr_[c + 1]; ++k) {
      const int v = var_at(k);
      if (cnt_[v]++ == 0 || occ_[v].empty() || occ_[v].back() != c) occ_[v].push_back(c);
      dirty_.insert(v);
    }
  }
  void remove(int64_t c) {
    alive_[c] = 0;
    --n_alive_;
    for (int64_t k = ptr_[c]; k < ptr_[c + 1]; ++k) {
      const int v = var_at(k);
      if (--cnt_[v] == 0) {
        dirty_.erase(v);
        occ_[v].clear();
      } else {
        dirty_.insert(v);
      }
    }
  }
  void compact() {
    if (static_cast<int64_t>(sc_.size()) > 2 * n_alive_ + 64) {
      size_t j = 0;
      for (int64_t c : sc_)
        if (alive_[c]) sc_[j++] = c;
      sc_.resize(j);
    }
  }
  // buffered clauses mentioning v, buffer order
  const std::vector<int64_t>& clauses_of(int v) {
    auto& o = occ_[v];
    size_t j = 0;
    for (int64_t c : o)
      if (alive_[c]) o[j++] = c;
    o.resize(j);
    return o;
  }

  void mark_unsat(Result& R, const std::string& note) {
    if (!R.unsat) {
      R.unsat = true;
      R.unsat_note = note;
    }
  }
  // extract.cpp:59-79
  void add_po(Result& R, int v, bool target) {
    if (po_state_[v]) {
      if ((po_state_[v] == 2) != target) mark_unsat(R, "x" + std::to_string(v) + " is forced to both 0 and 1");
      return;
    }
    if (const_def_[v] && (const_def_[v] == 2) != target) {
      mark_unsat(R, "x" + std::to_string(v) + " is defined as constant " + (const_def_[v] == 2 ? "1" : "0") +
                        " but forced to " + (target ? "1" : "0"));
      return;
    }
    po_state_[v] = target ? 2 : 1;
    R.po.push_back({v, target});
    in_iv_[v] = 0;
  }
  // extract.cpp:83-94
  void classify_inputs(Result& R, const std::vector<int64_t>& consumed, int except) {
    for (int64_t c : consumed)
      for (int64_t k = ptr_[c]; k < ptr_[c + 1]; ++k) {
        const int v = var_at(k);
        if (v == except) continue;
        if (role_[v] == kNone) {
          role_[v] = kPi;
          R.pi.push_back(v);
        }
      }
  }
  // extract.cpp:96-108 + handle_underspecified (:19-30)
  void fallback(Result& R) {
    if (n_alive_ == 0) return;
    std::vector<int64_t> all;
    for (int64_t c : sc_)
      if (alive_[c]) all.push_back(c);
    const int aux = ++next_aux_;
    std::vector<int> conj;
    conj.reserve(all.size());
    for (int64_t c : all) {
      std::vector<int> disj;
      for (int64_t k = ptr_[c]; k < ptr_[c + 1]; ++k) disj.push_back(X.literal(lit_[k]));
      conj.push_back(X.nary(kOr, disj));
    }
    const int e = X.simplify(X.nary(kAnd, conj), mcap_);
    if (e == 0) mark_unsat(R, "residual clause group is contradictory");
    be.emplace_back(aux, e);
    R.aux.push_back(aux);
    R.po.push_back({aux, true});
    classify_inputs(R, all, 0);
    for (int64_t c : all) remove(c);
    sc_.clear();
    dirty_.clear();
  }

  // Complement test of find_boolean_expression((v,0)) and ((v,1)) on the
  // union support (boolexpr.cpp:247-284), computed from the clauses.
  // Returns true iff is_complement(...) == Ternary::True.
  bool complement(int v, const std::vector<int64_t>& cls) {
    // f: clauses with ~v and not v; g: clauses with v and not ~v
    bool f_any = false, g_any = false, f_zero = false, g_zero = false;
    std::vector<int>& s = cs_;
    std::vector<int64_t>&fc = cf_, &gc = cg_;
    s.clear();
    fc.clear();
    gc.clear();
    for (int64_t c : cls) {
      bool pos = false, neg = false;
      int others = 0;
      for (int64_t k = ptr_[c]; k < ptr_[c + 1]; ++k) {
        const int l = lit_[k];
        if (l == v) pos = true;
        else if (l == -v) neg = true;
        else ++others;
      }
      if (pos == neg) continue;  // tautology (or v absent)
      if (neg) {
        f_any = true;
        if (others == 0) f_zero = true;
        fc.push_back(c);
      } else {
        g_any = true;
        if (others == 0) g_zero = true;
        gc.push_back(c);
      }
    }
    // An empty disjunction makes the whole conjunction 0 (no support); no
    // clause at all makes it 1 (boolexpr.cpp:74-100).
    auto collect = [&](const std::vector<int64_t>& cs) {
      for (int64_t c : cs)
        for (int64_t k = ptr_[c]; k < ptr_[c + 1]; ++k)
          if (var_at(k) != v) s.push_back(var_at(k));
    };
    if (f_any && !f_zero) collect(fc);
    if (g_any && !g_zero) collect(gc);
    std::sort(s.begin(), s.end());
    s.erase(std::unique(s.begin(), s.end()), s.end());
    if (static_cast<int>(s.size()) > ccap_) return false;  // Undecided
    const int n = static_cast<int>(s.size());
    if (n <= 6) {  // one word per table (gate encodings: 2-4 variables)
      static const uint64_t pat[6] = {0xAAAAAAAAAAAAAAAAull, 0xCCCCCCCCCCCCCCCCull, 0xF0F0F0F0F0F0F0F0ull,
                                      0xFF00FF00FF00FF00ull, 0xFFFF0000FFFF0000ull, 0xFFFFFFFF00000000ull};
      const uint64_t top = n == 6 ? ~0ull : ((1ull << (1u << n)) - 1ull);
      auto conj1 = [&](bool any, bool zero, const std::vector<int64_t>& cs) -> uint64_t {
        if (!any) return top;
        if (zero) return 0;
        uint64_t t = top;
        for (int64_t c : cs) {
          uint64_t d = 0;
          for (int64_t k = ptr_[c]; k < ptr_[c + 1]; ++k) {
            const int l = lit_[k];
            if (std::abs(l) == v) continue;
            const int i = static_cast<int>(std::lower_bound(s.begin(), s.end(), std::abs(l)) - s.begin());
            d |= l < 0 ? ~pat[i] : pat[i];
          }
          t &= d;
        }
        return t & top;
      };
      return (conj1(f_any, f_zero, fc) ^ conj1(g_any, g_zero, gc)) == top;
    }
    auto conj_tt = [&](bool any, bool zero, const std::vector<int64_t>& cs) {
      TT t(n);
      if (!any) {
        t.flip();
        return t;
      }
      if (zero) return t;
      t.flip();
      for (int64_t c : cs) {
        TT d(n);
        for (int64_t k = ptr_[c]; k < ptr_[c + 1]; ++k) {
          const int l = lit_[k];
          if (std::abs(l) == v) continue;
          const int i = static_cast<int>(std::lower_bound(s.begin(), s.end(), std::abs(l)) - s.begin());
          TT x = TT::var(n, i);
          if (l < 0) x.flip();
          for (size_t j = 0; j < d.nw; ++j) d.w()[j] |= x.w()[j];
        }
        for (size_t j = 0; j < t.nw; ++j) t.w()[j] &= d.w()[j];
      }
      return t;
    };
    return conj_tt(f_any, f_zero, fc).complement_of(conj_tt(g_any, g_zero, gc));
  }

  // find_boolean_expression(target = (v, negated = false)) (boolexpr.cpp:247-264)
  int definition_expr(int v, const std::vector<int64_t>& cls) {
    std::vector<int>& conj = conj_;
    conj.clear();
    for (int64_t c : cls) {
      bool pos = false, neg = false;
      for (int64_t k = ptr_[c]; k < ptr_[c + 1]; ++k) {
        if (lit_[k] == v) pos = true;
        if (lit_[k] == -v) neg = true;
      }
      if (!neg || pos) continue;
      std::vector<int>& disj = disj_;
      disj.clear();
      for (int64_t k = ptr_[c]; k < ptr_[c + 1]; ++k)
        if (var_at(k) != v) disj.push_back(X.literal(lit_[k]));
      conj.push_back(X.nary(kOr, disj));
    }
    return X.nary(kAnd, conj);
  }

  // extract.cpp:110-152
  void try_commit(Result& R) {
    while (!dirty_.empty()) {
      const int v = *dirty_.rbegin();  // descending index order
      const std::vector<int64_t>& cls = clauses_of(v);
      bool commit = false;
      if (complement(v, cls)) {
        const int def = X.simplify(definition_expr(v, cls), mcap_);
        if (role_[v] == kNone) {
          be.emplace_back(v, def);
          role_[v] = kDefined;
          if (X.is_const(def)) {
            const_def_[v] = def == 1 ? 2 : 1;
            add_po(R, v, def == 1);
          } else {
            in_iv_[v] = 1;
            iv_order_.push_back(v);
          }
          commit = true;
        } else if (X.is_const(def)) {
          add_po(R, v, def == 1);
          commit = true;
        }
      }
      if (!commit) {
        dirty_.erase(std::prev(dirty_.end()));
        continue;
      }
      std::vector<int64_t> consumed(cls.begin(), cls.end());
      classify_inputs(R, consumed, v);
      for (int64_t c : consumed) remove(c);
      compact();
      return;
    }
  }
};

}  // namespace

void extract_build(int num_vars, const int32_t* clause_ptr, const int32_t* clause_lit, int64_t n_clauses,
                   int complement_cap, int minimize_cap, Result& R) {
  Extractor E(num_vars, clause_ptr, clause_lit, n_clauses, complement_cap, minimize_cap);
  E.run(R);
  // build (circuit.cpp:60-122)
  std::vector<int> node_of(static_cast<size_t>(num_vars) + R.aux.size() + 1, -1);
  auto push_node = [&](int kind, int a, int b, int var) {
    R.kind.push_back(kind);
    R.a.push_back(a);
    R.b.push_back(b);
    R.var.push_back(var);
    return static_cast<int>(R.kind.size()) - 1;
  };
  auto node = [&](int v) {
    if (v <= 0 || v >= static_cast<int>(node_of.size()) || node_of[v] < 0)
      throw std::invalid_argument("x" + std::to_string(v) + " has no circuit node");
    return node_of[v];
  };
  for (int v : R.pi) {
    const int id = push_node(0, -1, -1, v);
    if (node_of[v] < 0) node_of[v] = id;
  }
  static const int kOpKind[5] = {4, 5, 6, 7, 8};  // Not, And2, Or2, Xor2, Xnor2 -> GateKind
  for (const auto& [dv, expr] : E.be) {
    std::vector<Exprs::Gate> gates;
    std::unordered_map<int, Exprs::Ref> memo;
    const Exprs::Ref out = E.X.decompose(expr, gates, memo);
    std::vector<int> gate_node(gates.size(), -1);
    auto resolve = [&](const Exprs::Ref& r) {
      if (r.src == 0) return node(r.index);
      if (r.src == 1) return gate_node[r.index];
      throw std::logic_error("constant operand in decomposition");
    };
    for (size_t i = 0; i < gates.size(); ++i) {
      const Exprs::Gate& g = gates[i];
      const int a = resolve(g.a);
      const int b = g.op == 0 ? -1 : resolve(g.b);
      gate_node[i] = push_node(kOpKind[g.op], a, b, 0);
    }
    int on;
    if (out.src == 1) on = gate_node[out.index];
    else if (out.src == 0) on = push_node(3, node(out.index), -1, 0);
    else on = push_node(out.index ? 2 : 1, -1, -1, 0);
    R.var[on] = dv;
    if (node_of[dv] < 0) node_of[dv] = on;
  }
  R.n_defs = static_cast<int64_t>(E.be.size());
}

}  // namespace sgx::ext
