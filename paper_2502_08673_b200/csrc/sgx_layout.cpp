#include "sgx_layout.hpp"

#include <algorithm>
#include <numeric>
#include <stdexcept>

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

void pad_chunk(std::vector<I4>& ops) {
  while (ops.size() % kU) ops.push_back({kNop, -1, -1, -1});
}

// Soft program over the nodes with in_set[i] != 0 (closed under operands).
SoftProgram build_soft(const Layout& L, const std::vector<uint8_t>& in_set) {
  SoftProgram P;
  const int n = L.n_nodes;
  P.row_of_node.assign(n, -1);
  std::vector<int32_t> order;
  for (int i = 0; i < n; ++i)
    if (in_set[i]) order.push_back(i);
  std::stable_sort(order.begin(), order.end(),
                   [&](int x, int y) { return L.level[x] < L.level[y]; });
  P.node_of_row = order;
  P.n_rows = static_cast<int32_t>(order.size());
  for (int r = 0; r < P.n_rows; ++r) P.row_of_node[order[r]] = r;
  int max_level = -1;
  for (int i : order) max_level = std::max(max_level, L.level[i]);
  P.n_levels = max_level + 1;

  std::vector<int32_t> col_of_node(n, -1);
  for (size_t j = 0; j < L.cpi.size(); ++j) col_of_node[L.node_of_var[L.cpi[j]]] = static_cast<int32_t>(j);
  P.col_row.assign(L.cpi.size(), -1);
  for (size_t j = 0; j < L.cpi.size(); ++j) P.col_row[j] = P.row_of_node[L.node_of_var[L.cpi[j]]];

  std::vector<int32_t> seed_of_node(n, -1);
  for (size_t m = 0; m < L.out_node.size(); ++m)
    if (in_set[L.out_node[m]]) seed_of_node[L.out_node[m]] = static_cast<int32_t>(m);
  P.out_row.resize(L.out_node.size());
  for (size_t m = 0; m < L.out_node.size(); ++m) P.out_row[m] = P.row_of_node[L.out_node[m]];

  // Level buckets (rows are level-sorted, so buckets are row ranges).
  std::vector<int32_t> lvl_begin(P.n_levels + 1, P.n_rows);
  for (int r = P.n_rows - 1; r >= 0; --r) lvl_begin[L.level[order[r]]] = r;
  lvl_begin[P.n_levels] = P.n_rows;
  for (int l = P.n_levels - 1; l >= 0; --l)
    if (lvl_begin[l] > lvl_begin[l + 1]) lvl_begin[l] = lvl_begin[l + 1];

  // Forward ops, level by level.
  for (int l = 0; l < P.n_levels; ++l) {
    for (int r = lvl_begin[l]; r < lvl_begin[l + 1]; ++r) {
      int i = order[r];
      int32_t k = L.kind[i];
      I4 op{k, r, -1, -1};
      if (k == SGX_INPUT) op.z = col_of_node[i];
      if (operand_count(k) >= 1) op.z = P.row_of_node[L.a[i]];
      if (operand_count(k) == 2) op.w = P.row_of_node[L.b[i]];
      P.fwd.push_back(op);
    }
    pad_chunk(P.fwd);
  }

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

  // Backward micro-ops, levels high to low.
  for (int l = P.n_levels - 1; l >= 0; --l) {
    for (int r = lvl_begin[l + 1] - 1; r >= lvl_begin[l]; --r) {
      int i = order[r];
      int32_t k = L.kind[i];
      bool is_col_input = k == SGX_INPUT && col_of_node[i] >= 0;
      bool has_operands = operand_count(k) > 0;
      if (!is_col_input && !has_operands) continue;  // CONST / 0.5-input: adjoint unused
      int32_t m = seed_of_node[i];
      int32_t begin_code = kBegin;
      if (m >= 0) begin_code |= kSeedBit | (L.out_tgt[m] ? kTargetBit : 0);
      P.bwd.push_back({begin_code, r, 0, 0});
      for (int64_t e = fo_ptr[i]; e < fo_ptr[i + 1]; ++e) {
        int32_t ck = L.kind[fo[e].consumer];
        P.bwd.push_back({kEdge | (ck << kKindShift), P.row_of_node[fo[e].consumer],
                         fo[e].other >= 0 ? P.row_of_node[fo[e].other] : -1, 0});
      }
      P.bwd.push_back({kEnd, has_operands ? r : -1, is_col_input ? col_of_node[i] : -1, 0});
    }
    pad_chunk(P.bwd);
  }
  return P;
}

}  // namespace

Layout build_layout(const sgx_circuit_desc& d) {
  Layout L;
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
  L.cone = build_soft(L, cone);
  L.full = build_soft(L, all);

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
  L.clause_ptr32.resize(L.clause_ptr.size());
  for (size_t c = 0; c < L.clause_ptr.size(); ++c) L.clause_ptr32[c] = static_cast<int32_t>(L.clause_ptr[c]);
  for (int64_t c = 0; c + 1 < static_cast<int64_t>(L.clause_ptr.size()); ++c) {
    for (int64_t l = L.clause_ptr[c]; l < L.clause_ptr[c + 1]; ++l) {
      int32_t lit = L.clause_lit[l];
      int v = lit < 0 ? -lit : lit;
      bool last = l + 1 == L.clause_ptr[c + 1];
      L.clause_enc.push_back((L.bit_row_of_node[L.node_of_var[v]] << 2) | (last ? 2 : 0) |
                             (lit < 0 ? 1 : 0));
    }
  }
  L.key_words = (L.num_vars + 63) / 64;
  L.key_bit_row.assign(static_cast<size_t>(L.key_words) * 64, -1);
  for (int v = 1; v <= L.num_vars; ++v) L.key_bit_row[v - 1] = L.bit_row_of_node[L.node_of_var[v]];
  return L;
}

void layout_info(const Layout& L, int64_t* info) {
  info[0] = L.n_nodes;
  info[1] = L.cone.n_rows;
  info[2] = L.cone.n_edges;
  info[3] = L.cone.n_levels;
  info[4] = static_cast<int64_t>(L.bit_lvl_ptr.size()) - 1;
  info[5] = static_cast<int64_t>(L.cone.fwd.size());
  info[6] = static_cast<int64_t>(L.cone.bwd.size());
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
