#include "sgx_layout.hpp"

#include <algorithm>
#include <array>
#include <exception>
#include <future>
#include <thread>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <queue>
#include <cstdlib>
#include <stdexcept>
#include <string>

namespace sgx {

namespace {

int operand_count(int32_t k) {
  switch (k) {
    case SGX_INPUT:
    case SGX_CONST0:
    case SGX_CONST1:
      return 0;
    case SGX_BUF:
    case SGX_NOT:
      return 1;
    default:
      return 2;
  }
}

std::string xv(int v) { return "x" + std::to_string(v); }

// 32-row bit gate (circuit.cpp:137-144) with its operands read through
// negations nx, ny, as the algebraic normal form over the raw operand words
// X, Y: f = c0 ^ c1 X ^ c2 Y ^ c3 XY, coefficient k in bit k.  One branch-free
// formula then evaluates every gate kind (lanes of a warp run mixed kinds).
int32_t anf_of(int32_t kind, int nx, int ny) {
  auto g = [&](int x, int y) {
    x ^= nx;
    y ^= ny;
    switch (kind) {
      case SGX_CONST0: return 0;
      case SGX_CONST1: return 1;
      case SGX_BUF: return x;
      case SGX_NOT: return x ^ 1;
      case SGX_AND2: return x & y;
      case SGX_OR2: return x | y;
      case SGX_XOR2: return x ^ y;
      default: return (x ^ y) ^ 1;  // XNOR2
    }
  };
  const int t00 = g(0, 0), t01 = g(0, 1), t10 = g(1, 0), t11 = g(1, 1);
  return t00 | ((t00 ^ t10) << 1) | ((t00 ^ t01) << 2) | ((t00 ^ t01 ^ t10 ^ t11) << 3);
}

// Harvest clause set: the CNF minus the clauses every harvested row satisfies
// by construction.  The harvest evaluates every gate (eval_discrete,
// circuit.cpp:124-152) before it checks the CNF (sampler.cpp:140-147,
// cnf.cpp:129-147), and a row is valid only if its outputs also match their
// targets.  So a clause C is implied -- true on every row that passes the
// other checks -- when, for some CNF variable o of C defined by a gate, C
// holds for every assignment of o's support (the CNF variables and inputs
// the gate's definition reads, through unnamed internal nodes) with o set to
// its definition's value; or when C has a literal an output target forces
// true.  Both are exhaustive checks of a small truth table (support <= 10),
// so dropping C changes no row's verdict: the valid mask, and hence the
// harvest's counts and keys, are bit-identical to checking the whole CNF.
// SGX_ALL_CLAUSES=1 keeps every clause (A/B and parity tests).
void harvest_clauses(Layout& L) {
  const int64_t nc = static_cast<int64_t>(L.clause_ptr.size()) - 1;
  L.hclause_ptr.assign(1, 0);
  L.hclause_lit.clear();
  L.n_implied = 0;
  L.clause_implied.assign(static_cast<size_t>(std::max<int64_t>(nc, 0)), 0);
  const char* all = getenv("SGX_ALL_CLAUSES");
  const bool keep_all = all && all[0] == '1';
  constexpr int kMaxSup = 10, kWords = (1 << kMaxSup) / 64, kMaxNodes = 256;
  using TT = std::array<uint64_t, kWords>;
  const int n = L.n_nodes;
  auto named = [&](int i) { return L.var[i] >= 1 && L.var[i] <= L.num_vars; };
  // Per defining node (a gate carrying a CNF variable): its support vars and
  // truth table over them, built on first use.  sup empty + ok=false: no table.
  struct Def {
    bool done = false, ok = false;
    std::vector<int32_t> sup;  // CNF variables, truth-table bit order
    TT tt{};
  };
  std::vector<Def> defs(static_cast<size_t>(L.max_var) + 1);
  std::vector<int32_t> mark(n, -1), stack;
  std::vector<TT> val(n);
  int32_t epoch = 0;
  // truth table of support variable j: bit r = bit j of r (the same for
  // every support size k; a k-variable table uses its first 2^k bits)
  std::array<TT, kMaxSup> pat{};
  for (int j = 0; j < kMaxSup; ++j)
    for (int r = 0; r < (1 << kMaxSup); ++r)
      if ((r >> j) & 1) pat[j][r >> 6] |= uint64_t{1} << (r & 63);
  auto words_of = [](int k) { return k <= 6 ? 1 : 1 << (k - 6); };
  auto define = [&](int v) -> Def& {
    Def& D = defs[v];
    if (D.done) return D;
    D.done = true;
    const int g = L.node_of_var[v];
    if (g < 0 || L.kind[g] == SGX_INPUT) return D;
    // internal nodes (reachable from g through unnamed nodes), index order
    ++epoch;
    std::vector<int32_t> inner, leaves;
    stack.assign(1, g);
    mark[g] = epoch;
    while (!stack.empty()) {
      const int x = stack.back();
      stack.pop_back();
      if (x != g && (named(x) || L.kind[x] == SGX_INPUT)) {
        leaves.push_back(x);
        if (static_cast<int>(leaves.size()) > kMaxSup) return D;
        continue;
      }
      inner.push_back(x);
      if (static_cast<int>(inner.size()) > kMaxNodes) return D;
      const int oc = operand_count(L.kind[x]);
      for (int s = 0; s < oc; ++s) {
        const int y = s == 0 ? L.a[x] : L.b[x];
        if (mark[y] != epoch) {
          mark[y] = epoch;
          stack.push_back(y);
        }
      }
    }
    std::sort(leaves.begin(), leaves.end());
    std::sort(inner.begin(), inner.end());
    const int k = static_cast<int>(leaves.size()), nw = words_of(k);
    for (int j = 0; j < k; ++j) {
      const int x = leaves[j];
      if (!named(x)) return D;  // an input without a CNF variable: keep the clause
      D.sup.push_back(L.var[x]);
      val[x] = pat[j];
    }
    for (int x : inner) {
      const TT& A = val[L.a[x] >= 0 ? L.a[x] : x];
      const TT& B = val[L.b[x] >= 0 ? L.b[x] : x];
      TT& o = val[x];
      for (int w = 0; w < nw; ++w) {
        switch (L.kind[x]) {
          case SGX_CONST0: o[w] = 0; break;
          case SGX_CONST1: o[w] = ~uint64_t{0}; break;
          case SGX_BUF: o[w] = A[w]; break;
          case SGX_NOT: o[w] = ~A[w]; break;
          case SGX_AND2: o[w] = A[w] & B[w]; break;
          case SGX_OR2: o[w] = A[w] | B[w]; break;
          case SGX_XOR2: o[w] = A[w] ^ B[w]; break;
          default: o[w] = ~(A[w] ^ B[w]); break;  // XNOR2
        }
      }
    }
    D.tt = val[g];
    D.ok = true;
    return D;
  };
  // literal forced true by an output target
  std::vector<int8_t> po_val(static_cast<size_t>(L.max_var) + 1, -1);
  for (size_t m = 0; m < L.out_node.size(); ++m) {
    const int v = L.var[L.out_node[m]];
    if (v >= 1 && v <= L.num_vars) po_val[v] = L.out_tgt[m] ? 1 : 0;
  }
  auto implied = [&](int64_t c) {
    const int64_t l0 = L.clause_ptr[c], l1 = L.clause_ptr[c + 1];
    for (int64_t l = l0; l < l1; ++l) {
      const int32_t lit = L.clause_lit[l];
      const int v = lit < 0 ? -lit : lit;
      if (po_val[v] >= 0 && po_val[v] == (lit > 0 ? 1 : 0)) return true;
    }
    for (int64_t l = l0; l < l1; ++l) {
      const int32_t lo = L.clause_lit[l];
      Def& D = define(lo < 0 ? -lo : lo);
      if (!D.ok) continue;
      const int k = static_cast<int>(D.sup.size()), nw = words_of(k);
      TT sat;
      for (int w = 0; w < nw; ++w) sat[w] = lo > 0 ? D.tt[w] : ~D.tt[w];
      for (int64_t m = l0; m < l1; ++m) {
        const int32_t lit = L.clause_lit[m];
        const int v = lit < 0 ? -lit : lit;
        if (v == (lo < 0 ? -lo : lo)) {
          if ((lit > 0) != (lo > 0)) return true;  // o and -o: a tautology
          continue;
        }
        const auto it = std::find(D.sup.begin(), D.sup.end(), v);
        if (it == D.sup.end()) continue;  // free variable: may be false
        const TT& p = pat[it - D.sup.begin()];
        for (int w = 0; w < nw; ++w) sat[w] |= lit > 0 ? p[w] : ~p[w];
      }
      const int rows = 1 << k;
      bool full = true;
      for (int r = 0; r < rows && full; r += 64) {
        const uint64_t want = rows - r >= 64 ? ~uint64_t{0} : ((uint64_t{1} << (rows - r)) - 1);
        full = (sat[r >> 6] & want) == want;
      }
      if (full) return true;
    }
    return false;
  };
  for (int64_t c = 0; c < nc; ++c) {
    if (!keep_all && implied(c)) {
      ++L.n_implied;
      L.clause_implied[c] = 1;
      continue;
    }
    L.hclause_lit.insert(L.hclause_lit.end(), L.clause_lit.begin() + L.clause_ptr[c],
                         L.clause_lit.begin() + L.clause_ptr[c + 1]);
    L.hclause_ptr.push_back(static_cast<int64_t>(L.hclause_lit.size()));
  }
  if (getenv("SGX_TRACE"))
    fprintf(stderr, "[sgx] harvest clauses: %lld of %lld implied by gate definitions / targets, %lld checked\n",
            static_cast<long long>(L.n_implied), static_cast<long long>(nc),
            static_cast<long long>(L.hclause_ptr.size()) - 1);
}

// SGX_TRACE stage timer for the layout compiler.
struct Lap {
  bool on = getenv("SGX_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void operator()(const char* what) {
    if (!on) return;
    const auto n = std::chrono::steady_clock::now();
    fprintf(stderr, "[sgx] layout   %-14s %.2f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

// One node's micro-op run (BEGIN ... END) as edge records (kR* flags): the
// BEGIN / SUB_BEGIN / SUB_END / END control rides on the neighbouring edge.
void run_records(const std::vector<I4>& run, std::vector<I4>& out) {
  const int32_t w = run.front().y;
  const int32_t b = run.front().x;
  int32_t pend = kRFirst | ((b & kSeedBit) ? kRSeed : 0) | ((b & kTargetBit) ? kRTarget : 0);
  int32_t spend = 0;
  bool sub_has = false;
  const size_t start = out.size();
  for (size_t t = 1; t < run.size(); ++t) {
    const I4& o = run[t];
    const int32_t code = o.x & 0xff;
    if (code == kEdge) {
      int32_t f = ((o.x >> kKindShift) & 0xf) | ((o.x & kNegOtherBit) ? kRNegOther : 0) | pend;
      pend = 0;
      if (o.x & kInSubBit) {
        f |= kRInSub | spend;
        spend = 0;
        sub_has = true;
      }
      out.push_back({f, o.y, o.z, w});
    } else if (code == kSubBegin) {
      spend = kRSubFirst | ((o.x & kSeedBit) ? kRSubSeed : 0) | ((o.x & kTargetBit) ? kRSubTarget : 0) |
              ((o.x & kNegSelfBit) ? kRNegSelf : 0);
      sub_has = false;
    } else if (code == kSubEnd) {
      const int32_t se = kRSubLast | ((((o.x >> kKindShift) & 0xf) == SGX_NOT) ? kRSubNot : 0);
      if (sub_has) {
        out.back().x |= se;
      } else {  // empty SUB run (a seeded folded output with no consumers)
        out.push_back({kRInSub | spend | pend | se, -1, -1, w});
        spend = pend = 0;
      }
    } else if (code == kEnd) {
      if (out.size() == start) {  // no edge at all
        out.push_back({pend, -1, -1, w});
        pend = 0;
      }
      if (o.y >= 0 || o.z >= 0) out.back().x |= kRLast;
    }
  }
  for (size_t k = start; k < out.size(); ++k)
    if ((out[k].x & (kRInSub | kRSubFirst | kRSubLast | kRSeed | kRSubSeed)) || out[k].y < 0) out[k].x |= kRSlow;
  for (size_t k = start; k < out.size(); ++k) {
    const int32_t f = out[k].x;
    if ((f & kRInSub) && (f & kRSubFirst) && (f & kRSubLast) && !(f & (kRSeed | kRSubSeed)) && out[k].y >= 0)
      out[k].x |= kRSubOne;
  }
}

// Soft program over the nodes with in_set[i] != 0 (closed under operands).
//
// NOT / BUF folding: a NOT or BUF node whose operand is materialized is
// VIRTUAL -- it owns no tape row; consumers read its operand's row and apply
// 1 - x (NOT) on the fly, which is the exact operation the reference performs
// (autodiff.cpp:110-113), so values stay bit-identical.  In the backward pass
// a virtual consumer j of node i contributes -adj[j] (NOT) / +adj[j] (BUF),
// where adj[j] is summed first, in its own order, by a nested SUB run
// (autodiff.cpp:225-233 pushed in descending id order).  A NOT/BUF whose
// operand is itself virtual stays materialized, so nesting depth is one.
SoftProgram build_soft(const Layout& L, const std::vector<uint8_t>& in_set) {
  Lap lap;
  SoftProgram P;
  const int n = L.n_nodes;
  P.row_of_node.assign(n, -1);

  std::vector<uint8_t> virt(n, 0);
  for (int i = 0; i < n; ++i)
    if (in_set[i] && (L.kind[i] == SGX_NOT || L.kind[i] == SGX_BUF) && !virt[L.a[i]]) virt[i] = 1;
  // Operand reference: (materialized base node, negate).
  auto base_of = [&](int x) { return virt[x] ? L.a[x] : x; };
  auto neg_of = [&](int x) { return virt[x] && L.kind[x] == SGX_NOT; };

  // Levels over the materialized DAG.
  std::vector<int32_t> lev(n, 0);
  int max_level = -1;
  for (int i = 0; i < n; ++i) {
    if (!in_set[i] || virt[i]) continue;
    int oc = operand_count(L.kind[i]);
    if (oc >= 1) lev[i] = lev[base_of(L.a[i])] + 1;
    if (oc == 2) lev[i] = std::max(lev[i], lev[base_of(L.b[i])] + 1);
    max_level = std::max(max_level, lev[i]);
  }
  if (!(getenv("SGX_SCHED") && std::string(getenv("SGX_SCHED")) == "asap")) {
    // ALAP: every node one level below its earliest consumer, so adjoint and
    // value rows are re-read soon after they are written (L2 reuse distance).
    std::vector<int32_t> alap(n, max_level);
    for (int j = n - 1; j >= 0; --j) {
      if (!in_set[j] || virt[j]) continue;
      const int oc = operand_count(L.kind[j]);
      if (oc >= 1) alap[base_of(L.a[j])] = std::min(alap[base_of(L.a[j])], alap[j] - 1);
      if (oc == 2) alap[base_of(L.b[j])] = std::min(alap[base_of(L.b[j])], alap[j] - 1);
    }
    for (int i = 0; i < n; ++i)
      if (in_set[i] && !virt[i]) lev[i] = alap[i];
  }
  P.n_levels = max_level + 1;
  std::vector<std::vector<int32_t>> by_level(P.n_levels);
  for (int i = 0; i < n; ++i)
    if (in_set[i] && !virt[i]) by_level[lev[i]].push_back(i);

  std::vector<int32_t> col_of_node(n, -1);
  for (size_t j = 0; j < L.cpi.size(); ++j) col_of_node[L.node_of_var[L.cpi[j]]] = static_cast<int32_t>(j);
  std::vector<int32_t> seed_of_node(n, -1);
  for (size_t m = 0; m < L.out_node.size(); ++m)
    if (in_set[L.out_node[m]]) seed_of_node[L.out_node[m]] = static_cast<int32_t>(m);

  // Forward: per level, nodes dealt round-robin to kWarps warps (after
  // sorting by kind), each warp's list cut into kind-homogeneous groups of at
  // most kGroup ops.  Rows are assigned in emission order, so a group's
  // outputs are consecutive rows.
  // Last forward level reading each (materialized) node: operand loads at that
  // level are the row's last forward use and go to L2 as evict_first.
  // A read also leaves first when the row's NEXT forward read is more than
  // SGX_FWD_FAR levels later (default 48): the row would not survive in L2
  // that long at 512 tiles in flight, and keeping it displaces rows that would
  // (row-granular model, C4: forward DRAM reads 5.77 -> 4.98 GB).
  // read_lv[row]: the levels reading it, ascending (each op at most once).
  const int far = [] {  // read per layout build (forced-variant tests set it per run)
    const char* e = getenv("SGX_FWD_FAR");
    const int v = e ? atoi(e) : 48;
    return v > 0 ? v : (1 << 30);
  }();
  std::vector<std::vector<int32_t>> read_lv(n);
  for (int i = 0; i < n; ++i) {
    if (!in_set[i] || virt[i]) continue;
    const int oc = operand_count(L.kind[i]);
    if (oc >= 1) read_lv[base_of(L.a[i])].push_back(lev[i]);
    if (oc == 2) read_lv[base_of(L.b[i])].push_back(lev[i]);
  }
  for (auto& v : read_lv) std::sort(v.begin(), v.end());
  auto cold_read = [&](int row_node, int l) {  // no read of row_node within `far` levels after l
    const auto& v = read_lv[row_node];
    auto it = std::upper_bound(v.begin(), v.end(), l);
    return it == v.end() || *it - l > far;
  };
  int32_t next_row = 0;
  auto enc = [&](int x) {  // operand encoding: row << 1 | negate
    int bse = base_of(x);
    return (P.row_of_node[bse] << 1) | (neg_of(x) ? 1 : 0);
  };
  for (int l = 0; l < P.n_levels; ++l) {
    std::vector<int32_t> nodes = by_level[l];
    std::stable_sort(nodes.begin(), nodes.end(), [&](int x, int y) { return L.kind[x] < L.kind[y]; });
    std::vector<std::vector<int32_t>> per(kWarps);
    for (size_t t = 0; t < nodes.size(); ++t) per[t % kWarps].push_back(nodes[t]);
    for (int w = 0; w < kWarps; ++w) {
      const auto& lst = per[w];
      int32_t first = static_cast<int32_t>(P.fwd.size() / kGroupRecs);
      int32_t groups = 0;
      for (size_t t = 0; t < lst.size();) {
        const int32_t k = L.kind[lst[t]];
        size_t e = t;
        while (e < lst.size() && L.kind[lst[e]] == k && e - t < static_cast<size_t>(kGroup)) ++e;
        const int32_t cnt = static_cast<int32_t>(e - t);
        // header .w: bit 2k+j = operand j of op k is its row's last forward read
        I4 head{k, cnt, next_row, 0};
        std::vector<int32_t> operands(2 * kGroup, 0);
        for (size_t u = t; u < e; ++u) {
          const int i = lst[u];
          P.row_of_node[i] = next_row++;
          P.node_of_row.push_back(i);
          int oc = operand_count(k);
          if (k == SGX_INPUT) operands[2 * (u - t)] = col_of_node[i];
          if (oc >= 1) operands[2 * (u - t)] = enc(L.a[i]);
          if (oc == 2) operands[2 * (u - t) + 1] = enc(L.b[i]);
          if (oc >= 1 && cold_read(base_of(L.a[i]), lev[i])) head.w |= 1 << (2 * (u - t));
          if (oc == 2 && cold_read(base_of(L.b[i]), lev[i])) head.w |= 1 << (2 * (u - t) + 1);
        }
        P.fwd.push_back(head);
        for (int q = 0; q < kGroup / 2; ++q)
          P.fwd.push_back({operands[4 * q], operands[4 * q + 1], operands[4 * q + 2], operands[4 * q + 3]});
        ++groups;
        t = e;
      }
      P.fwd_lvl.push_back(first);
      P.fwd_lvl.push_back(groups);
    }
  }
  P.n_rows = next_row;
  for (int i = 0; i < n; ++i) P.n_set += in_set[i] ? 1 : 0;
  {  // staged forward blocks (see SoftProgram::fblk)
    const int nhdr = 1 + (kWarps + 1) / 2;
    std::vector<int32_t> starts;
    for (int l = 0; l < P.n_levels; ++l) {
      const int32_t start = static_cast<int32_t>(P.fblk.size());
      starts.push_back(start);
      P.fblk.resize(P.fblk.size() + nhdr, I4{0, 0, 0, 0});
      for (int w = 0; w < kWarps; ++w) {
        const int32_t first = P.fwd_lvl[2 * (l * kWarps + w)], cnt = P.fwd_lvl[2 * (l * kWarps + w) + 1];
        int32_t* h = &P.fblk[start + 1 + w / 2].x + 2 * (w & 1);
        h[0] = static_cast<int32_t>(P.fblk.size()) - start;
        h[1] = cnt;
        P.fblk.insert(P.fblk.end(), P.fwd.begin() + static_cast<size_t>(first) * kGroupRecs,
                      P.fwd.begin() + static_cast<size_t>(first + cnt) * kGroupRecs);
      }
      const int32_t n4 = static_cast<int32_t>(P.fblk.size()) - start;
      P.fblk_lvl.push_back(start);
      P.fblk_lvl.push_back(n4);
      P.fblk_max = std::max(P.fblk_max, n4);
    }
    for (int l = 0; l + 1 < P.n_levels; ++l) {
      P.fblk[starts[l]].x = P.fblk_lvl[2 * (l + 1)];
      P.fblk[starts[l]].y = P.fblk_lvl[2 * (l + 1) + 1];
    }
  }
  // Virtual nodes read as their base row (for the taps / outputs).
  P.virt_base.assign(n, -1);
  P.virt_neg.assign(n, 0);
  for (int i = 0; i < n; ++i)
    if (in_set[i] && virt[i]) {
      P.virt_base[i] = P.row_of_node[L.a[i]];
      P.virt_neg[i] = neg_of(i) ? 1 : 0;
    }
  P.out_enc.resize(L.out_node.size());
  for (size_t m = 0; m < L.out_node.size(); ++m)
    P.out_enc[m] = in_set[L.out_node[m]] ? enc(L.out_node[m]) : -1;
  P.col_row.assign(L.cpi.size(), -1);
  for (size_t j = 0; j < L.cpi.size(); ++j) P.col_row[j] = P.row_of_node[L.node_of_var[L.cpi[j]]];

  lap("fwd");
  // Fan-out lists inside the set: consumers in descending id, a-slot first.
  std::vector<int32_t> fo_cnt(n + 1, 0);
  for (int j = 0; j < n; ++j) {
    if (!in_set[j]) continue;
    int oc = operand_count(L.kind[j]);
    if (oc >= 1) ++fo_cnt[L.a[j]];
    if (oc == 2) ++fo_cnt[L.b[j]];
  }
  std::vector<int64_t> fo_ptr(n + 1, 0);
  for (int i = 0; i < n; ++i) fo_ptr[i + 1] = fo_ptr[i] + fo_cnt[i];
  P.n_edges = fo_ptr[n];
  std::vector<int64_t> fill(fo_ptr.begin(), fo_ptr.end() - 1);
  struct Edge {
    int32_t consumer, other;
  };
  std::vector<Edge> fo(static_cast<size_t>(P.n_edges));
  for (int j = n - 1; j >= 0; --j) {  // descending consumer id
    if (!in_set[j]) continue;
    int oc = operand_count(L.kind[j]);
    if (oc >= 1) fo[fill[L.a[j]]++] = {j, oc == 2 ? L.b[j] : -1};
    if (oc == 2) fo[fill[L.b[j]]++] = {j, L.a[j]};
  }
  auto seed_flags = [&](int node) {
    int32_t m = seed_of_node[node];
    return m >= 0 ? (kSeedBit | (L.out_tgt[m] ? kTargetBit : 0)) : 0;
  };
  // EDGE from materialized consumer j; `sub` marks edges inside a SUB run.
  auto edge = [&](std::vector<I4>& run, const Edge& e, int32_t sub) {
    int32_t ck = L.kind[e.consumer];
    int32_t x = kEdge | (ck << kKindShift) | sub;
    int32_t other = -1;
    if (e.other >= 0) {
      other = P.row_of_node[base_of(e.other)];
      if (neg_of(e.other)) x |= kNegOtherBit;
    }
    run.push_back({x, P.row_of_node[e.consumer], other, 0});
  };

  // Backward, levels high to low: each node's micro-op run (the reference's
  // summation order) becomes edge records; a node's records stay whole
  // inside one warp's stream, nodes go longest-first to the least loaded warp.
  for (int l = P.n_levels - 1; l >= 0; --l) {
    std::vector<std::vector<I4>> recs;
    for (int i : by_level[l]) {
      int32_t k = L.kind[i];
      bool is_col_input = k == SGX_INPUT && col_of_node[i] >= 0;
      bool has_operands = operand_count(k) > 0;
      if (!is_col_input && !has_operands) continue;  // CONST / 0.5-input: adjoint unused
      const int32_t r = P.row_of_node[i];
      std::vector<I4> run;
      run.push_back({kBegin | seed_flags(i), r, 0, 0});
      for (int64_t e = fo_ptr[i]; e < fo_ptr[i + 1]; ++e) {
        const int j = fo[e].consumer;
        if (!virt[j]) {
          edge(run, fo[e], 0);
          continue;
        }
        // adj[j] for virtual j (its value is T(v_i)), then -/+ into acc.
        int32_t sb = kSubBegin | seed_flags(j) | (L.kind[j] == SGX_NOT ? kNegSelfBit : 0);
        run.push_back({sb, r, 0, 0});
        for (int64_t f = fo_ptr[j]; f < fo_ptr[j + 1]; ++f) edge(run, fo[f], kInSubBit);
        run.push_back({kSubEnd | (L.kind[j] << kKindShift), 0, 0, 0});
      }
      run.push_back({kEnd, has_operands ? r : -1, is_col_input ? col_of_node[i] : -1, 0});
      std::vector<I4> rr;
      run_records(run, rr);
      recs.push_back(std::move(rr));
    }
    std::stable_sort(recs.begin(), recs.end(),
                     [](const auto& x, const auto& y) { return x.size() > y.size(); });
    // SGX_BWD_SPLIT=cap (default 160; 0 = off; large cones only, the on-chip
    // and circuit-specialised programs keep one pass per level): a level with
    // more than `cap` records runs as several passes of at most ~cap records
    // (node runs stay whole).  Nodes of one level are independent, so a
    // barrier between them changes nothing but the staged blocks' size: at
    // <= ~190 int4 per block a third data stage fits at 4 CTAs per SM (C4:
    // 632 -> 724 passes, C2 66 -> 129; live bench C4 backward -0.7 %, C2 -3 %).
    const int split_cap = [] {
      const char* e = getenv("SGX_BWD_SPLIT");
      return e ? atoi(e) : 160;
    }();
    size_t total = 0;
    for (auto& r : recs) total += r.size();
    const size_t cap = (split_cap > 0 && next_row > 1536 && total > static_cast<size_t>(split_cap))
                           ? static_cast<size_t>(split_cap) : total + 1;
    const size_t n_sub = (total + cap - 1) / cap;
    std::vector<std::vector<const std::vector<I4>*>> sub(std::max<size_t>(n_sub, 1));
    {
      std::vector<size_t> load(sub.size(), 0);  // longest runs first, to the least loaded sub-pass
      for (auto& r : recs) {
        size_t best = 0;
        for (size_t q = 1; q < sub.size(); ++q)
          if (load[q] < load[best]) best = q;
        sub[best].push_back(&r);
        load[best] += r.size();
      }
    }
    for (auto& group : sub) {
      std::vector<std::vector<I4>> rper(kWarps);
      for (auto* r : group) {
        int best = 0;
        for (int w = 1; w < kWarps; ++w)
          if (rper[w].size() < rper[best].size()) best = w;
        rper[best].insert(rper[best].end(), r->begin(), r->end());
      }
      for (int w = 0; w < kWarps; ++w) {
        P.rec_lvl.push_back(static_cast<int32_t>(P.rec.size()));
        P.rec_lvl.push_back(static_cast<int32_t>(rper[w].size()));
        P.rec.insert(P.rec.end(), rper[w].begin(), rper[w].end());
      }
    }
  }
  const int n_bwd_passes = static_cast<int>(P.rec_lvl.size() / (2 * kWarps));
  lap("bwd records");
  if (getenv("SGX_TRACE_DIST")) {  // reuse distances of the backward's row reads, in passes
    const int nl = n_bwd_passes;
    std::vector<int32_t> def_pass(P.n_rows, -1), last_t(P.n_rows, -1);
    std::vector<int64_t> hA(8, 0), hT(8, 0);
    auto bucket = [](int d) { return d <= 0 ? 0 : d == 1 ? 1 : d <= 2 ? 2 : d <= 4 ? 3 : d <= 8 ? 4 : d <= 32 ? 5 : d <= 128 ? 6 : 7; };
    int64_t nA = 0, nT = 0;
    for (int li = 0; li < nl; ++li)
      for (int w = 0; w < kWarps; ++w) {
        const int32_t first = P.rec_lvl[2 * (li * kWarps + w)], cnt = P.rec_lvl[2 * (li * kWarps + w) + 1];
        for (int32_t k = first; k < first + cnt; ++k) {
          const I4 r = P.rec[k];
          if (r.y >= 0) { ++hA[bucket(li - def_pass[r.y])]; ++nA; }
          if (r.z >= 0) {  // tape row re-read distance (passes since its previous backward read)
            if (last_t[r.z] >= 0) ++hT[bucket(li - last_t[r.z])]; else ++hT[0];
            last_t[r.z] = li;
            ++nT;
          }
          if (r.x & kRLast) def_pass[r.w] = li;
        }
      }
    {  // live sets per pass: adjoint rows (defined .. last read), tape rows (first .. last backward read)
      std::vector<int32_t> a_def(P.n_rows, -1), a_last(P.n_rows, -1), t_first(P.n_rows, -1), t_last(P.n_rows, -1);
      for (int li = 0; li < nl; ++li)
        for (int w = 0; w < kWarps; ++w) {
          const int32_t first = P.rec_lvl[2 * (li * kWarps + w)], cnt = P.rec_lvl[2 * (li * kWarps + w) + 1];
          for (int32_t k = first; k < first + cnt; ++k) {
            const I4 r = P.rec[k];
            if (r.y >= 0) a_last[r.y] = li;
            if (r.z >= 0) {
              if (t_first[r.z] < 0) t_first[r.z] = li;
              t_last[r.z] = li;
            }
            if (r.x & kRLast) a_def[r.w] = li;
          }
        }
      std::vector<int32_t> dA(nl + 1, 0), dT(nl + 1, 0), dU(nl + 1, 0);
      for (int r = 0; r < P.n_rows; ++r) {
        if (a_def[r] >= 0 && a_last[r] > a_def[r]) { ++dA[a_def[r] + 1]; --dA[a_last[r] + 1]; }
        if (t_first[r] >= 0 && t_last[r] > t_first[r]) { ++dT[t_first[r] + 1]; --dT[t_last[r] + 1]; }
        if (t_first[r] >= 0) { ++dU[t_first[r]]; --dU[t_last[r] + 1]; }
      }
      int32_t ca = 0, ct = 0, cu = 0, ma = 0, mt = 0, mu = 0;
      int64_t sa = 0, st = 0;
      for (int li = 0; li <= nl; ++li) {
        ca += dA[li]; ct += dT[li]; cu += dU[li];
        ma = std::max(ma, ca); mt = std::max(mt, ct); mu = std::max(mu, cu);
        sa += ca; st += ct;
      }
      int32_t never = 0;
      for (int r = 0; r < P.n_rows; ++r) never += t_first[r] < 0 ? 1 : 0;
      fprintf(stderr, "[sgx] bwd live rows across passes: adjoint max %d mean %.0f; tape (between reads) max %d mean %.0f; tape incl. single-read max %d; rows never read by the backward %d\n",
              ma, double(sa) / nl, mt, double(st) / nl, mu, never);
    }
    {
      int64_t slow = 0, sub = 0, lastc = 0, nrec = 0, sfirst = 0, slast = 0, sboth = 0;
      for (int li = 0; li < nl; ++li)
        for (int w = 0; w < kWarps; ++w) {
          const int32_t first = P.rec_lvl[2 * (li * kWarps + w)], cnt = P.rec_lvl[2 * (li * kWarps + w) + 1];
          for (int32_t k = first; k < first + cnt; ++k) {
            ++nrec;
            slow += (P.rec[k].x & kRSlow) ? 1 : 0;
            sub += (P.rec[k].x & kRInSub) ? 1 : 0;
            lastc += (P.rec[k].x & kRLast) ? 1 : 0;
            sfirst += (P.rec[k].x & kRSubFirst) ? 1 : 0;
            slast += (P.rec[k].x & kRSubLast) ? 1 : 0;
            sboth += ((P.rec[k].x & kRSubFirst) && (P.rec[k].x & kRSubLast)) ? 1 : 0;
          }
        }
      {
        std::vector<uint8_t> is_in(P.n_rows, 0);
        for (int32_t r : P.col_row)
          if (r >= 0) is_in[r] = 1;
        int64_t tin = 0, tall = 0;
        for (int li = 0; li < nl; ++li)
          for (int w = 0; w < kWarps; ++w) {
            const int32_t first = P.rec_lvl[2 * (li * kWarps + w)], cnt = P.rec_lvl[2 * (li * kWarps + w) + 1];
            for (int32_t k = first; k < first + cnt; ++k)
              if (P.rec[k].z >= 0) {
                ++tall;
                tin += is_in[P.rec[k].z];
              }
          }
        fprintf(stderr, "[sgx] bwd tape reads of column-input rows: %lld of %lld\n", (long long)tin, (long long)tall);
      }
      fprintf(stderr, "[sgx] bwd records: %lld, slow %lld (in SUB runs %lld: first %lld, last %lld, both %lld), node ends %lld\n",
              (long long)nrec, (long long)slow, (long long)sub, (long long)sfirst, (long long)slast, (long long)sboth,
              (long long)lastc);
    }
    fprintf(stderr, "[sgx] bwd reads: %lld adjoint, %lld tape (rows %d, passes %d)\n", (long long)nA, (long long)nT, P.n_rows, nl);
    const char* names[8] = {"<=0", "1", "2", "3-4", "5-8", "9-32", "33-128", ">128"};
    for (int b = 0; b < 8; ++b)
      fprintf(stderr, "[sgx]   distance %-7s adjoint %6.2f%%  tape re-read (<=0: first read) %6.2f%%\n", names[b], 100.0 * hA[b] / std::max<int64_t>(1, nA),
              100.0 * hT[b] / std::max<int64_t>(1, nT));
  }
  // Tape reads with a near next read keep their row in L2 (kRYKeep): another
  // record reads the same tape row within SGX_BWD_KEEP passes (default 4;
  // 0 = every tape read evict_first).  Row-granular model, C4: backward DRAM
  // 29.9 -> 28.0 GB per launch.
  {
    const int keep = [] {
      const char* e = getenv("SGX_BWD_KEEP");
      return e ? atoi(e) : 4;
    }();
    if (keep > 0) {
      const int nl = n_bwd_passes;
      std::vector<std::vector<int32_t>> treads(P.n_rows);  // passes reading each tape row, ascending
      for (int li = 0; li < nl; ++li)
        for (int w = 0; w < kWarps; ++w) {
          const int32_t first = P.rec_lvl[2 * (li * kWarps + w)], cnt = P.rec_lvl[2 * (li * kWarps + w) + 1];
          for (int32_t k = first; k < first + cnt; ++k)
            if (P.rec[k].z >= 0) treads[P.rec[k].z].push_back(li);
        }
      for (int li = 0; li < nl; ++li)
        for (int w = 0; w < kWarps; ++w) {
          const int32_t first = P.rec_lvl[2 * (li * kWarps + w)], cnt = P.rec_lvl[2 * (li * kWarps + w) + 1];
          for (int32_t k = first; k < first + cnt; ++k) {
            const int32_t z = P.rec[k].z;
            if (z < 0) continue;
            const auto& v = treads[z];  // another read in [li, li + keep] besides this one?
            const auto n_near = std::upper_bound(v.begin(), v.end(), li + keep) - std::lower_bound(v.begin(), v.end(), li);
            if (n_near >= 2) P.rec[k].x |= kRYKeep;
          }
        }
    }
  }
  // Dead-adjoint lists: the last pass reading each adjoint row (a record's
  // .y), passes numbered in backward order.
  {
    const int nl = n_bwd_passes;
    std::vector<int32_t> last(P.n_rows, -1);
    for (int li = 0; li < nl; ++li)
      for (int w = 0; w < kWarps; ++w) {
        const int32_t first = P.rec_lvl[2 * (li * kWarps + w)], cnt = P.rec_lvl[2 * (li * kWarps + w) + 1];
        for (int32_t k = first; k < first + cnt; ++k)
          if (P.rec[k].y >= 0) last[P.rec[k].y] = li;
      }
    std::vector<uint8_t> is_col(P.n_rows, 0);
    for (int32_t r : P.col_row)
      if (r >= 0) is_col[r] = 1;
    std::vector<std::vector<int32_t>> by(nl);
    for (int32_t r = 0; r < P.n_rows; ++r)
      if (last[r] >= 0 && !is_col[r]) by[last[r]].push_back(r);
    for (int li = 0; li < nl; ++li) {
      P.dead_lvl.push_back(static_cast<int32_t>(P.dead.size()));
      P.dead_lvl.push_back(static_cast<int32_t>(by[li].size()));
      P.dead.insert(P.dead.end(), by[li].begin(), by[li].end());
    }
    // Block li: header {dead_rel, n_dead, next_start, next_n4}, then per warp
    // {first_rel, count} (two warps per int4), the records, the dead rows.
    const int nhdr = 1 + (kWarps + 1) / 2;
    std::vector<int32_t> starts;
    for (int li = 0; li < nl; ++li) {
      const int32_t start = static_cast<int32_t>(P.sblk.size());
      starts.push_back(start);
      P.sblk.resize(P.sblk.size() + nhdr, I4{0, 0, 0, 0});
      for (int w = 0; w < kWarps; ++w) {
        const int32_t first = P.rec_lvl[2 * (li * kWarps + w)], cnt = P.rec_lvl[2 * (li * kWarps + w) + 1];
        int32_t* h = &P.sblk[start + 1 + w / 2].x + 2 * (w & 1);
        h[0] = static_cast<int32_t>(P.sblk.size()) - start;
        h[1] = cnt;
        P.srec_lvl.push_back(h[0]);
        P.srec_lvl.push_back(cnt);
        P.sblk.insert(P.sblk.end(), P.rec.begin() + first, P.rec.begin() + first + cnt);
      }
      const int32_t dstart = static_cast<int32_t>(P.sblk.size()) - start;
      const std::vector<int32_t> none;
      const std::vector<int32_t>& d = li > 0 ? by[li - 1] : none;
      for (size_t k = 0; k < d.size(); k += 4) {
        I4 q{-1, -1, -1, -1};
        int32_t* qq = &q.x;
        for (size_t j = 0; j < 4 && k + j < d.size(); ++j) qq[j] = d[k + j];
        P.sblk.push_back(q);
      }
      const int32_t n4 = static_cast<int32_t>(P.sblk.size()) - start;
      P.sblk[start].x = dstart;
      P.sblk[start].y = static_cast<int32_t>(d.size());
      P.sblk_lvl.insert(P.sblk_lvl.end(), {start, n4, dstart, static_cast<int32_t>(d.size())});
      P.sblk_max = std::max(P.sblk_max, n4);
    }
    for (int li = 0; li + 1 < nl; ++li) {
      P.sblk[starts[li]].z = P.sblk_lvl[4 * (li + 1)];
      P.sblk[starts[li]].w = P.sblk_lvl[4 * (li + 1) + 1];
    }
    if (nl > 0) P.tail_dead = by[nl - 1];
    if (getenv("SGX_TRACE"))
      fprintf(stderr, "[sgx] staged blocks: backward %d passes, max %d int4 (%d B); forward max %d int4 (%d B)\n",
              nl, P.sblk_max, P.sblk_max * 16, P.fblk_max, P.fblk_max * 16);
  }
  if (P.n_rows <= 1024) {  // on-chip program (SoftProgram::oc_*); larger tapes cannot fit a warp's share
    for (int l = 0; l < P.n_levels; ++l) {
      P.oc_fwd_lvl.push_back(static_cast<int32_t>(P.oc_fwd.size() / kGroupRecs));
      for (int w = 0; w < kWarps; ++w) {
        const int32_t first = P.fwd_lvl[2 * (l * kWarps + w)], cnt = P.fwd_lvl[2 * (l * kWarps + w) + 1];
        P.oc_fwd.insert(P.oc_fwd.end(), P.fwd.begin() + static_cast<size_t>(first) * kGroupRecs,
                        P.fwd.begin() + static_cast<size_t>(first + cnt) * kGroupRecs);
      }
      P.oc_fwd_lvl.push_back(static_cast<int32_t>(P.oc_fwd.size() / kGroupRecs) - P.oc_fwd_lvl.back());
    }
    const int nl = P.n_levels;
    for (int li = 0; li < nl; ++li) {
      P.oc_rec_lvl.push_back(static_cast<int32_t>(P.oc_rec.size()));
      for (int w = 0; w < kWarps; ++w) {
        const int32_t first = P.rec_lvl[2 * (li * kWarps + w)], cnt = P.rec_lvl[2 * (li * kWarps + w) + 1];
        P.oc_rec.insert(P.oc_rec.end(), P.rec.begin() + first, P.rec.begin() + first + cnt);
        for (auto it = P.oc_rec.end() - cnt; it != P.oc_rec.end(); ++it) it->x &= ~(kRSubOne | kRYKeep);
      }
      P.oc_rec_lvl.push_back(static_cast<int32_t>(P.oc_rec.size()) - P.oc_rec_lvl.back());
    }
    // adjoint live ranges over the record stream: defined at the node's
    // kRLast record, dead after its last reader (.y); column inputs live on
    // to the epilogue
    const int64_t nr = static_cast<int64_t>(P.oc_rec.size());
    std::vector<int64_t> last(P.n_rows, -1);
    for (int64_t k = 0; k < nr; ++k)
      if (P.oc_rec[k].y >= 0) last[P.oc_rec[k].y] = k;
    for (int32_t r : P.col_row)
      if (r >= 0) last[r] = nr;
    std::vector<int32_t> slot(P.n_rows, -1);
    std::vector<std::vector<int32_t>> free_after(nr + 1);
    std::priority_queue<int32_t, std::vector<int32_t>, std::greater<>> freeq;
    int32_t nslots = 0;
    for (int64_t k = 0; k < nr; ++k) {
      I4& r = P.oc_rec[k];
      if (r.y >= 0) r.y = slot[r.y];  // the consumer's adjoint (defined earlier)
      if (r.x & kRLast) {
        const int32_t own = r.w;
        int32_t sl;
        if (freeq.empty()) {
          sl = nslots++;
        } else {
          sl = freeq.top();
          freeq.pop();
        }
        slot[own] = sl;
        r.x |= sl << kOcSlotShift;
        if (last[own] < 0) {
          freeq.push(sl);  // never read: reusable at once
        } else if (last[own] < nr) {
          free_after[last[own]].push_back(sl);
        }
      }
      for (int32_t sl : free_after[k]) freeq.push(sl);
    }
    P.oc_adj_slots = std::max(nslots, 1);
    if (getenv("SGX_TRACE"))
      fprintf(stderr, "[sgx] on-chip program: %d tape rows, %d adjoint slots, %zu groups, %lld records\n", P.n_rows,
              P.oc_adj_slots, P.oc_fwd.size() / kGroupRecs, static_cast<long long>(nr));
    P.oc_col_slot.assign(P.col_row.size(), -1);
    for (size_t j = 0; j < P.col_row.size(); ++j)
      if (P.col_row[j] >= 0) P.oc_col_slot[j] = slot[P.col_row[j]];
  }
  // Slack so a chunk of records may read past the last one.
  for (int k = 0; k < kU; ++k) P.rec.push_back({0, -1, -1, 0});
  return P;
}

// Folded bit program over every node (eval_discrete, circuit.cpp:126-146):
// ~x and x are free on a 32-row word, so NOT/BUF nodes with a materialized
// operand become a mask on the reference instead of a row.
void build_folded_bits(Layout& L) {
  Lap lap;
  const int n = L.n_nodes;
  std::vector<uint8_t> virt(n, 0);
  for (int i = 0; i < n; ++i)
    if ((L.kind[i] == SGX_NOT || L.kind[i] == SGX_BUF) && !virt[L.a[i]]) virt[i] = 1;
  std::vector<int32_t> lev(n, 0);
  int max_level = 0;
  auto base = [&](int x) { return virt[x] ? L.a[x] : x; };
  for (int i = 0; i < n; ++i) {
    if (virt[i]) continue;
    const int oc = operand_count(L.kind[i]);
    if (oc >= 1) lev[i] = lev[base(L.a[i])] + 1;
    if (oc == 2) lev[i] = std::max(lev[i], lev[base(L.b[i])] + 1);
    max_level = std::max(max_level, lev[i]);
  }
  std::vector<std::vector<int32_t>> by_level(max_level + 1);
  for (int i = 0; i < n; ++i)
    if (!virt[i]) by_level[lev[i]].push_back(i);
  std::vector<int32_t> row(n, -1);
  int32_t next = 0;
  for (const auto& lv : by_level)
    for (int i : lv) row[i] = next++;
  L.fb_rows = next;
  auto enc = [&](int x) {  // row << 1 | negate, through at most one folded NOT
    const bool neg = virt[x] && L.kind[x] == SGX_NOT;
    return (row[base(x)] << 1) | (neg ? 1 : 0);
  };
  L.fb_ops.clear();
  L.fb_lvl_ptr.clear();
  for (const auto& lv : by_level) {
    L.fb_lvl_ptr.push_back(static_cast<int32_t>(L.fb_ops.size()));
    for (int i : lv) {
      if (L.kind[i] == SGX_INPUT) continue;
      const int oc = operand_count(L.kind[i]);
      L.fb_ops.push_back({L.kind[i], row[i], oc >= 1 ? enc(L.a[i]) : 0, oc == 2 ? enc(L.b[i]) : 0});
    }
  }
  L.fb_lvl_ptr.push_back(static_cast<int32_t>(L.fb_ops.size()));
  L.fb_cpi_row.clear();
  L.fb_ucpi_row.clear();
  for (int v : L.cpi) L.fb_cpi_row.push_back(row[L.node_of_var[v]]);
  for (int v : L.ucpi) L.fb_ucpi_row.push_back(row[L.node_of_var[v]]);
  L.fb_out_enc.clear();
  for (int o : L.out_node) L.fb_out_enc.push_back(enc(o));
  L.fb_key_enc.assign(static_cast<size_t>(L.key_words) * 64, -1);
  for (int v = 1; v <= L.num_vars; ++v) L.fb_key_enc[v - 1] = enc(L.node_of_var[v]);
  lap("fb ops");

  // CNF records (kCnfOpen): a literal is its row, bit-inverted when negated
  // (row = e ^ (e >> 31)); a clause of <= 4 literals is one record padded with
  // the always-zero row fb_rows; a longer one is a chain of open records of 3
  // literals + kCnfOpen, then a closing record.  Whole clauses dealt to
  // kCnfThreads threads, longest-first to the least loaded, then padded with
  // open all-zero records and transposed.
  const int64_t n_clauses = static_cast<int64_t>(L.hclause_ptr.size()) - 1;
  const int32_t zero_row = L.fb_rows;
  std::vector<I4> recs;                 // all clauses' records, flat
  std::vector<int64_t> rec_ptr(n_clauses + 1, 0);
  std::vector<int32_t> lits;
  for (int64_t c = 0; c < n_clauses; ++c) {
    lits.clear();
    for (int64_t l = L.hclause_ptr[c]; l < L.hclause_ptr[c + 1]; ++l) {
      const int32_t lit = L.hclause_lit[l];
      const int e = enc(L.node_of_var[lit < 0 ? -lit : lit]);
      const bool neg = ((e & 1) ^ (lit < 0 ? 1 : 0)) != 0;
      lits.push_back(neg ? ~(e >> 1) : (e >> 1));
    }
    size_t k = 0;
    for (; lits.size() - k > 4; k += 3) recs.push_back({lits[k], lits[k + 1], lits[k + 2], kCnfOpen});
    int32_t t[4] = {zero_row, zero_row, zero_row, zero_row};
    for (size_t u = 0; k + u < lits.size(); ++u) t[u] = lits[k + u];
    recs.push_back({t[0], t[1], t[2], t[3]});
    rec_ptr[c + 1] = static_cast<int64_t>(recs.size());
  }
  auto nrec = [&](int64_t c) { return rec_ptr[c + 1] - rec_ptr[c]; };
  lap("cnf recs");
  // Longest first, stable (a bucket sort on the record count).
  int64_t maxr = 0;
  for (int64_t c = 0; c < n_clauses; ++c) maxr = std::max(maxr, nrec(c));
  std::vector<int64_t> bstart(maxr + 2, 0);
  for (int64_t c = 0; c < n_clauses; ++c) ++bstart[maxr - nrec(c) + 1];
  for (int64_t r = 1; r <= maxr + 1; ++r) bstart[r] += bstart[r - 1];
  std::vector<int64_t> order(n_clauses);
  for (int64_t c = 0; c < n_clauses; ++c) order[bstart[maxr - nrec(c)]++] = c;
  // Least-loaded thread, lowest index on ties (a min-heap of (load, thread)).
  std::vector<std::vector<I4>> per(kCnfThreads);
  std::priority_queue<std::pair<int64_t, int>, std::vector<std::pair<int64_t, int>>, std::greater<>> heap;
  for (int t = 0; t < kCnfThreads; ++t) heap.push({0, t});
  for (int64_t c : order) {
    auto [ld, best] = heap.top();
    heap.pop();
    per[best].insert(per[best].end(), recs.begin() + rec_ptr[c], recs.begin() + rec_ptr[c + 1]);
    heap.push({ld + nrec(c), best});
  }
  lap("cnf deal");
  size_t steps = 0;
  for (const auto& p : per) steps = std::max(steps, p.size());
  L.fb_cnf_steps = static_cast<int32_t>(steps);
  L.fb_cnf4.assign(steps * kCnfThreads, I4{zero_row, zero_row, zero_row, kCnfOpen});
  for (int t = 0; t < kCnfThreads; ++t)
    for (size_t j = 0; j < per[t].size(); ++j) L.fb_cnf4[j * kCnfThreads + t] = per[t][j];
}

}  // namespace

// Liveness-allocated harvest program (Layout::lb_*; k_harvest_live).
void build_live_bits(Layout& L) {
  const int n = L.n_nodes;
  std::vector<uint8_t> virt(n, 0);
  for (int i = 0; i < n; ++i)
    if ((L.kind[i] == SGX_NOT || L.kind[i] == SGX_BUF) && !virt[L.a[i]]) virt[i] = 1;
  auto base = [&](int x) { return virt[x] ? L.a[x] : x; };
  auto negv = [&](int x) { return virt[x] && L.kind[x] == SGX_NOT; };
  std::vector<int32_t> lev(n, 0);
  int max_level = 0;
  for (int i = 0; i < n; ++i) {
    if (virt[i]) continue;
    const int oc = operand_count(L.kind[i]);
    if (oc >= 1) lev[i] = lev[base(L.a[i])] + 1;
    if (oc == 2) lev[i] = std::max(lev[i], lev[base(L.b[i])] + 1);
    max_level = std::max(max_level, lev[i]);
  }
  const int P = max_level + 2;  // checks of the last level run in the extra phase
  // last phase reading each row
  std::vector<int32_t> last(n, -1);
  for (int i = 0; i < n; ++i) {
    if (virt[i]) continue;
    last[i] = std::max(last[i], lev[i]);
    const int oc = operand_count(L.kind[i]);
    if (oc >= 1) last[base(L.a[i])] = std::max(last[base(L.a[i])], lev[i]);
    if (oc == 2) last[base(L.b[i])] = std::max(last[base(L.b[i])], lev[i]);
  }
  const int64_t n_clauses = static_cast<int64_t>(L.hclause_ptr.size()) - 1;
  std::vector<int32_t> cl_phase(n_clauses);
  for (int64_t c = 0; c < n_clauses; ++c) {
    int m = 0;
    for (int64_t l = L.hclause_ptr[c]; l < L.hclause_ptr[c + 1]; ++l) {
      const int32_t lit = L.hclause_lit[l];
      m = std::max(m, lev[base(L.node_of_var[lit < 0 ? -lit : lit])]);
    }
    cl_phase[c] = m + 1;
    for (int64_t l = L.hclause_ptr[c]; l < L.hclause_ptr[c + 1]; ++l) {
      const int32_t lit = L.hclause_lit[l];
      const int r = base(L.node_of_var[lit < 0 ? -lit : lit]);
      last[r] = std::max(last[r], m + 1);
    }
  }
  for (int o : L.out_node) last[base(o)] = std::max(last[base(o)], lev[base(o)] + 1);
  // linear-scan slot allocation (slot 0 is the always-zero row)
  std::vector<std::vector<int32_t>> def_at(P), free_at(P + 1);
  for (int i = 0; i < n; ++i)
    if (!virt[i]) {
      def_at[lev[i]].push_back(i);
      free_at[last[i] + 1].push_back(i);
    }
  std::vector<int32_t> slot(n, -1);
  std::priority_queue<int32_t, std::vector<int32_t>, std::greater<>> freeq;
  int32_t nslots = 1;
  for (int ph = 0; ph < P; ++ph) {
    for (int r : free_at[ph]) freeq.push(slot[r]);
    for (int r : def_at[ph]) {
      if (freeq.empty()) {
        slot[r] = nslots++;
      } else {
        slot[r] = freeq.top();
        freeq.pop();
      }
    }
  }
  L.lb_slots = nslots;
  L.lb_levels = P;
  // spill rows: bases of CNF-variable nodes
  std::vector<int32_t> spill(n, -1);
  int32_t nsp = 0;
  for (int v = 1; v <= L.num_vars; ++v) {
    const int r = base(L.node_of_var[v]);
    if (spill[r] < 0) spill[r] = nsp++;
  }
  L.lb_n_spill = nsp;
  auto enc = [&](int x) { return (slot[base(x)] << 1) | (negv(x) ? 1 : 0); };
  L.lb_ops.clear();
  L.lb_op_ptr.clear();
  for (int ph = 0; ph < P; ++ph) {
    L.lb_op_ptr.push_back(static_cast<int32_t>(L.lb_ops.size()));
    for (int i : def_at[ph]) {
      if (L.kind[i] == SGX_INPUT) continue;
      const int oc = operand_count(L.kind[i]);
      L.lb_ops.push_back({L.kind[i] | (slot[i] << 4), oc >= 1 ? enc(L.a[i]) : 0, oc == 2 ? enc(L.b[i]) : 0,
                          spill[i]});
    }
  }
  L.lb_op_ptr.push_back(static_cast<int32_t>(L.lb_ops.size()));
  // checks by phase: output targets (one-literal checks), then clauses
  std::vector<std::vector<I4>> chk(P);
  auto lit_of = [&](int x, bool negate) {  // slot, or ~slot when the value is complemented
    const int32_t sl = slot[base(x)];
    return (negv(x) != negate) ? ~sl : sl;
  };
  for (size_t m = 0; m < L.out_node.size(); ++m) {
    const int o = L.out_node[m];
    chk[lev[base(o)] + 1].push_back({lit_of(o, L.out_tgt[m] == 0), 0, 0, 0});
  }
  L.lb_big_lits.clear();
  for (int64_t c = 0; c < n_clauses; ++c) {
    const int64_t k = L.hclause_ptr[c + 1] - L.hclause_ptr[c];
    std::vector<int32_t> lits;
    for (int64_t l = L.hclause_ptr[c]; l < L.hclause_ptr[c + 1]; ++l) {
      const int32_t lit = L.hclause_lit[l];
      lits.push_back(lit_of(L.node_of_var[lit < 0 ? -lit : lit], lit < 0));
    }
    if (k <= 4) {
      int32_t t[4] = {0, 0, 0, 0};
      for (int64_t u = 0; u < k; ++u) t[u] = lits[u];
      chk[cl_phase[c]].push_back({t[0], t[1], t[2], t[3]});
    } else {
      chk[cl_phase[c]].push_back({static_cast<int32_t>(L.lb_big_lits.size()), static_cast<int32_t>(k), 0, kLbBig});
      L.lb_big_lits.insert(L.lb_big_lits.end(), lits.begin(), lits.end());
    }
  }
  L.lb_chk.clear();
  L.lb_chk_ptr.clear();
  for (int ph = 0; ph < P; ++ph) {
    L.lb_chk_ptr.push_back(static_cast<int32_t>(L.lb_chk.size()));
    L.lb_chk.insert(L.lb_chk.end(), chk[ph].begin(), chk[ph].end());
  }
  L.lb_chk_ptr.push_back(static_cast<int32_t>(L.lb_chk.size()));
  // warp-synchronous cut: 32 records per iteration, >= 1 iteration per phase
  if (nslots >= (1 << 24)) throw std::invalid_argument("circuit too large for the live harvest");
  L.lw_ops.clear();
  for (int ph = 0; ph < P; ++ph) {
    const int32_t ob = L.lb_op_ptr[ph], no = L.lb_op_ptr[ph + 1] - ob;
    const int32_t iters = std::max<int32_t>(1, (no + 31) / 32);
    const bool has_chk = L.lb_chk_ptr[ph + 1] > L.lb_chk_ptr[ph];
    for (int32_t it = 0; it < iters; ++it)
      for (int32_t ln = 0; ln < 32; ++ln) {
        const int32_t k = it * 32 + ln;
        I4 r{nslots << 4, 0, 0, -1};  // padding: sink <- 0 (ANF all zero)
        if (k < no) {  // the gate with its operand negations as the ANF of f(X, Y) over raw slots
          const I4 o = L.lb_ops[ob + k];
          r = {(o.x & ~0xf) | anf_of(o.x & 0xf, o.y & 1, o.z & 1), o.y >> 1, o.z >> 1, o.w};
        }
        if (it + 1 == iters) r.x |= kLwEnd | (has_chk ? kLwChk : 0);
        L.lw_ops.push_back(r);
      }
  }
  while ((L.lw_ops.size() / 32) % kLwChunk) L.lw_ops.push_back({nslots << 4, 0, 0, -1});  // whole ring chunks
  L.lw_iters = static_cast<int32_t>(L.lw_ops.size() / 32);
  L.lb_cpi.clear();
  L.lb_ucpi.clear();
  for (int v : L.cpi) {
    const int r = L.node_of_var[v];
    L.lb_cpi.insert(L.lb_cpi.end(), {slot[r], spill[r]});
  }
  for (int v : L.ucpi) {
    const int r = L.node_of_var[v];
    L.lb_ucpi.insert(L.lb_ucpi.end(), {slot[r], spill[r]});
  }
  L.lb_key_enc.assign(static_cast<size_t>(L.key_words) * 64, -1);
  for (int v = 1; v <= L.num_vars; ++v) {
    const int x = L.node_of_var[v];
    L.lb_key_enc[v - 1] = (spill[base(x)] << 1) | (negv(x) ? 1 : 0);
  }
  if (getenv("SGX_TRACE")) {
    fprintf(stderr, "[sgx] live harvest: %d phases, %d slots, %d spill rows, %zu ops, %zu checks, %d warp iterations\n", P,
            nslots, nsp, L.lb_ops.size(), L.lb_chk.size(), L.lw_iters);
    std::vector<int> no, nc;
    for (int ph = 0; ph < P; ++ph) {
      no.push_back(L.lb_op_ptr[ph + 1] - L.lb_op_ptr[ph]);
      nc.push_back(L.lb_chk_ptr[ph + 1] - L.lb_chk_ptr[ph]);
    }
    auto pct = [](std::vector<int> v, double q) { std::sort(v.begin(), v.end()); return v[static_cast<size_t>(q * (v.size() - 1))]; };
    fprintf(stderr, "[sgx] live harvest per phase: ops p50 %d p90 %d p99 %d max %d; checks p50 %d p90 %d p99 %d max %d\n",
            pct(no, .5), pct(no, .9), pct(no, .99), pct(no, 1), pct(nc, .5), pct(nc, .9), pct(nc, .99), pct(nc, 1));
  }
}

Layout build_layout(const sgx_circuit_desc& d) {
  Layout L;
  const bool trace = getenv("SGX_TRACE") != nullptr;
  auto tp = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!trace) return;
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[sgx] layout %-12s %.2f ms\n", what, std::chrono::duration<double, std::milli>(t - tp).count());
    tp = t;
  };
  if (d.n_nodes < 0 || d.num_vars < 0 || d.n_outputs < 0 || d.n_cpi < 0 || d.n_ucpi < 0 ||
      d.n_clauses < 0)
    throw std::invalid_argument("negative size in circuit descriptor");
  L.n_nodes = d.n_nodes;
  L.num_vars = d.num_vars;
  L.unsat = d.unsat != 0;
  const int n = d.n_nodes;
  L.kind.assign(d.kind, d.kind + n);
  L.a.assign(d.a, d.a + n);
  L.b.assign(d.b, d.b + n);
  L.var.assign(d.var, d.var + n);

  L.max_var = d.num_vars;
  for (int i = 0; i < n; ++i) {
    if (L.kind[i] < SGX_INPUT || L.kind[i] > SGX_XNOR2)
      throw std::invalid_argument("unknown gate kind at node " + std::to_string(i));
    int oc = operand_count(L.kind[i]);
    if ((oc >= 1 && (L.a[i] < 0 || L.a[i] >= i)) || (oc == 2 && (L.b[i] < 0 || L.b[i] >= i)))
      throw std::invalid_argument("operands must reference earlier gates (node " +
                                  std::to_string(i) + ")");
    if (oc < 1) L.a[i] = -1;
    if (oc < 2) L.b[i] = -1;
    if (L.var[i] < 0) throw std::invalid_argument("gate var must be positive");
    L.max_var = std::max(L.max_var, L.var[i]);
  }
  L.node_of_var.assign(L.max_var + 1, -1);
  for (int i = 0; i < n; ++i) {
    if (L.var[i] == 0) continue;
    if (L.node_of_var[L.var[i]] != -1) throw std::invalid_argument(xv(L.var[i]) + " mapped to two gates");
    L.node_of_var[L.var[i]] = i;
  }
  auto node_of = [&](int v) {  // Circuit::node_of, circuit.cpp:52-58
    if (v <= 0 || v > L.max_var || L.node_of_var[v] < 0)
      throw std::invalid_argument(xv(v) + " has no circuit node");
    return L.node_of_var[v];
  };

  for (int m = 0; m < d.n_outputs; ++m) {
    L.out_var.push_back(d.out_var[m]);
    L.out_tgt.push_back(d.out_target[m] ? 1 : 0);
    L.out_node.push_back(node_of(d.out_var[m]));
  }
  // map_input_columns (autodiff.cpp:38-53)
  std::vector<uint8_t> bound(n, 0);
  for (int j = 0; j < d.n_cpi; ++j) {
    int v = d.cpi[j];
    int node = node_of(v);
    if (L.kind[node] != SGX_INPUT) throw std::invalid_argument(xv(v) + " is not a circuit input");
    if (bound[node]) throw std::invalid_argument(xv(v) + " bound to two columns");
    bound[node] = 1;
    L.cpi.push_back(v);
  }
  for (int k = 0; k < d.n_ucpi; ++k) {
    int v = d.ucpi[k];
    int node = node_of(v);
    if (L.kind[node] != SGX_INPUT) throw std::invalid_argument(xv(v) + " is not a circuit input");
    if (bound[node]) throw std::invalid_argument(xv(v) + " bound to two columns");
    bound[node] = 2;
    L.ucpi.push_back(v);
  }
  // eval_discrete needs every INPUT assigned (circuit.cpp:129-135).
  for (int i = 0; i < n; ++i)
    if (L.kind[i] == SGX_INPUT && !bound[i])
      throw std::invalid_argument("input " + xv(L.var[i]) + " is unassigned");
  // eval_cnf / dedupe_key need every CNF variable (cnf.cpp:130-134, sampler.cpp:20-22).
  for (int v = 1; v <= L.num_vars; ++v) node_of(v);

  L.clause_ptr.assign(d.clause_ptr, d.clause_ptr + d.n_clauses + 1);
  if (L.clause_ptr[0] != 0) throw std::invalid_argument("clause_ptr must start at 0");
  for (int64_t c = 0; c < d.n_clauses; ++c) {
    if (L.clause_ptr[c + 1] <= L.clause_ptr[c]) throw std::invalid_argument("empty clause");
  }
  int64_t nl = L.clause_ptr[d.n_clauses];
  if (nl > INT32_MAX) throw std::invalid_argument("too many literals");
  L.clause_lit.assign(d.clause_lit, d.clause_lit + nl);
  for (int32_t lit : L.clause_lit) {
    int v = lit < 0 ? -lit : lit;
    if (v == 0 || v > L.num_vars) throw std::invalid_argument("variable " + std::to_string(v) + " is unassigned");
  }

  lap("validate");
  // ASAP levels.
  L.level.assign(n, 0);
  for (int i = 0; i < n; ++i) {
    int oc = operand_count(L.kind[i]);
    if (oc >= 1) L.level[i] = L.level[L.a[i]] + 1;
    if (oc == 2) L.level[i] = std::max(L.level[i], L.level[L.b[i]] + 1);
  }

  // Primary-output cone: transitive fan-in of the outputs.
  std::vector<uint8_t> cone(n, 0), all(n, 1);
  for (int o : L.out_node) cone[o] = 1;
  for (int i = n - 1; i >= 0; --i) {
    if (!cone[i]) continue;
    int oc = operand_count(L.kind[i]);
    if (oc >= 1) cone[L.a[i]] = 1;
    if (oc == 2) cone[L.b[i]] = 1;
  }
  // The soft program, the live harvest program and the bit / folded bit
  // programs below read the validated inputs only and write disjoint fields:
  // the first two are compiled on their own threads.
  L.key_words = (L.num_vars + 63) / 64;
  // (inline below 4096 nodes: there, three thread spawns cost more than the work)
  const bool par = n >= 4096;
  auto spawn = [par](auto&& f) { return par ? std::thread(f) : (f(), std::thread()); };
  std::exception_ptr err_soft, err_live;
  std::thread t_soft = spawn([&] {
    try {
      L.cone = build_soft(L, cone);
    } catch (...) {
      err_soft = std::current_exception();
    }
  });
  // The harvest clause set (harvest_clauses) feeds the three harvest
  // programs; it runs first on the live-program thread, overlapping the
  // soft program, and the other two wait for it.
  std::promise<void> clauses_done;
  std::shared_future<void> clauses = clauses_done.get_future().share();
  std::thread t_live = spawn([&] {
    try {
      try {
        harvest_clauses(L);
        clauses_done.set_value();
      } catch (...) {
        clauses_done.set_exception(std::current_exception());
        throw;
      }
      build_live_bits(L);
    } catch (...) {
      err_live = std::current_exception();
    }
  });
  std::exception_ptr err_fold;
  std::thread t_fold = spawn([&] {
    try {
      clauses.get();
      build_folded_bits(L);
    } catch (...) {
      err_fold = std::current_exception();
    }
  });
  struct Join {  // joined on every path out (exceptions included)
    std::thread &a, &b, &c;
    ~Join() {
      for (std::thread* t : {&a, &b, &c})
        if (t->joinable()) t->join();
    }
  } join{t_soft, t_live, t_fold};
  (void)all;  // the all-node program for the parity taps is built on demand

  // Bit program: every node, level-sorted; INPUT rows come from the harden
  // kernel, everything else from bit ops.
  std::vector<int32_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int x, int y) { return L.level[x] < L.level[y]; });
  L.n_bit_rows = n;
  L.bit_row_of_node.assign(n, -1);
  for (int r = 0; r < n; ++r) L.bit_row_of_node[order[r]] = r;
  int nlev = 0;
  for (int i = 0; i < n; ++i) nlev = std::max(nlev, L.level[i] + 1);
  L.bit_lvl_ptr.assign(nlev + 1, 0);
  int cur = 0;
  for (int l = 0; l < nlev; ++l) {
    L.bit_lvl_ptr[l] = static_cast<int32_t>(L.bit_ops.size());
    while (cur < n && L.level[order[cur]] == l) {
      int i = order[cur++];
      if (L.kind[i] == SGX_INPUT) continue;
      int oc = operand_count(L.kind[i]);
      L.bit_ops.push_back({L.kind[i], L.bit_row_of_node[i], oc >= 1 ? L.bit_row_of_node[L.a[i]] : 0,
                           oc == 2 ? L.bit_row_of_node[L.b[i]] : 0});
    }
  }
  L.bit_lvl_ptr[nlev] = static_cast<int32_t>(L.bit_ops.size());
  for (int v : L.cpi) L.cpi_bit_row.push_back(L.bit_row_of_node[L.node_of_var[v]]);
  for (int v : L.ucpi) L.ucpi_bit_row.push_back(L.bit_row_of_node[L.node_of_var[v]]);
  for (int o : L.out_node) L.out_bit_row.push_back(L.bit_row_of_node[o]);
  clauses.get();
  L.clause_ptr32.resize(L.hclause_ptr.size());
  for (size_t c = 0; c < L.hclause_ptr.size(); ++c) L.clause_ptr32[c] = static_cast<int32_t>(L.hclause_ptr[c]);
  for (int64_t c = 0; c + 1 < static_cast<int64_t>(L.hclause_ptr.size()); ++c) {
    for (int64_t l = L.hclause_ptr[c]; l < L.hclause_ptr[c + 1]; ++l) {
      int32_t lit = L.hclause_lit[l];
      int v = lit < 0 ? -lit : lit;
      bool last = l + 1 == L.hclause_ptr[c + 1];
      L.clause_enc.push_back((L.bit_row_of_node[L.node_of_var[v]] << 2) | (last ? 2 : 0) |
                             (lit < 0 ? 1 : 0));
    }
  }
  L.key_bit_row.assign(static_cast<size_t>(L.key_words) * 64, -1);
  for (int v = 1; v <= L.num_vars; ++v) L.key_bit_row[v - 1] = L.bit_row_of_node[L.node_of_var[v]];
  lap("bits");
  if (t_soft.joinable()) t_soft.join();
  if (t_live.joinable()) t_live.join();
  if (t_fold.joinable()) t_fold.join();
  lap("threads join");
  if (err_soft) std::rethrow_exception(err_soft);
  if (err_live) std::rethrow_exception(err_live);
  if (err_fold) std::rethrow_exception(err_fold);
  return L;
}

void build_full_program(Layout& L) {
  if (!L.full.row_of_node.empty() || L.n_nodes == 0) return;
  L.full = build_soft(L, std::vector<uint8_t>(L.n_nodes, 1));
}

void layout_info(const Layout& L, int64_t* info) {
  info[0] = L.n_nodes;
  info[1] = L.cone.n_set;   // cone nodes (SURVEY 8(d) N_c)
  info[2] = L.cone.n_edges;
  info[3] = L.cone.n_levels;
  info[4] = static_cast<int64_t>(L.bit_lvl_ptr.size()) - 1;
  info[5] = L.cone.n_rows;  // materialized (tape) rows after NOT/BUF folding
  info[6] = static_cast<int64_t>(L.cone.rec.size());  // backward edge records
  info[7] = static_cast<int64_t>(L.bit_ops.size());
  info[8] = static_cast<int64_t>(L.clause_ptr.size()) - 1;
  info[9] = L.n_lits();
  info[10] = L.key_words;
  info[11] = static_cast<int64_t>(L.cpi.size());
  info[12] = static_cast<int64_t>(L.ucpi.size());
  info[13] = static_cast<int64_t>(L.out_node.size());
  info[14] = L.num_vars;
  info[15] = L.unsat ? 1 : 0;
}

}  // namespace sgx
