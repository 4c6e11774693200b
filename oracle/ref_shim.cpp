// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference library (satgrad, compiled
// in place from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libsatgrad_ref.so). It exists so that Python tests, the fixture
// generator (tests/golden/make_fixtures.py) and bench.py's reference arm can
// drive the reference's own code path:
//   parse_dimacs / extract / build / classify_paths   (cnf.cpp, extract.cpp, circuit.cpp)
//   embed / forward / loss / backward / gd_step / harden  (autodiff.cpp:57-297)
//   init_soft_inputs / run                              (sampler.cpp:54-64, 89-203)
//   testgen::random_circuit / encode                    (tests/gen.cpp:117-124, 283-345)
// The or-chain generator below restates acceptance_main.cpp:101-138
// (or50_fixture) with its constants as parameters; the planted 3-SAT generator
// is new and uses the reference hash.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <sstream>
#include <string>
#include <vector>

#include "gen.hpp"
#include "satgrad/autodiff.hpp"
#include "satgrad/circuit.hpp"
#include "satgrad/cnf.hpp"
#include "satgrad/extract.hpp"
#include "satgrad/rng.hpp"
#include "satgrad/sampler.hpp"

using namespace satgrad;

namespace {

thread_local std::string g_err;

struct RefInst {
  CnfFormula cnf;
  ExtractionResult res;
  Circuit circuit;
  PathClassification paths;
  std::vector<int> node_of_var;  // dense var -> node map (-1 = none)
  std::string scratch;
  RunResult run;
  bool has_run = false;
};

RefInst* finish(CnfFormula cnf, const ExtractorConfig& cfg = {}) {
  auto inst = std::make_unique<RefInst>();
  inst->cnf = std::move(cnf);
  inst->res = extract(inst->cnf, cfg);
  inst->circuit = build(inst->res);
  inst->paths = classify_paths(inst->res);
  int max_var = inst->circuit.num_vars;
  for (const auto& [v, n] : inst->circuit.var_to_node) max_var = std::max(max_var, v);
  inst->node_of_var.assign(max_var + 1, -1);
  for (const auto& [v, n] : inst->circuit.var_to_node) inst->node_of_var[v] = n;
  return inst.release();
}

// acceptance_main.cpp:101-138 with (seed, inputs, levels, gpl, arity, outs)
// as parameters; (424242, 50, 5, 10, 4, 4) reproduces or50_fixture exactly.
testgen::TCircuit or_chain(uint64_t seed, int inputs, int levels, int gpl,
                           int arity, int outs) {
  uint64_t ctr = 0;
  auto next = [&] { return hash_stream({seed, 0x6f723530, ctr++}); };
  auto rnd = [&](int n) { return static_cast<int>(next() % n); };
  testgen::TCircuit tc;
  tc.num_inputs = inputs;
  tc.num_vars = inputs;
  std::vector<int> prev, all;
  for (int v = 1; v <= inputs; ++v) all.push_back(v);
  prev = all;
  for (int lvl = 0; lvl < levels; ++lvl) {
    std::vector<int> o;
    for (int g = 0; g < gpl; ++g) {
      testgen::TGate gate;
      gate.kind = testgen::TKind::Or;
      for (int i = 0; i < arity; ++i) {
        const std::vector<int>& pool = rnd(10) < 7 ? prev : all;
        int var = pool[rnd(static_cast<int>(pool.size()))];
        gate.args.push_back(rnd(2) ? -var : var);
      }
      gate.out = ++tc.num_vars;
      o.push_back(gate.out);
      tc.gates.push_back(gate);
    }
    all.insert(all.end(), o.begin(), o.end());
    prev = std::move(o);
  }
  Assignment witness(inputs + 1, 0xFF);
  for (int v = 1; v <= inputs; ++v) witness[v] = next() & 1;
  Assignment full = testgen::eval_netlist(tc, witness);
  for (int i = 0; i < outs && i < static_cast<int>(prev.size()); ++i) {
    int j = i + rnd(static_cast<int>(prev.size()) - i);
    std::swap(prev[i], prev[j]);
    tc.outputs.push_back({prev[i], full[prev[i]] != 0});
  }
  return tc;
}

// Planted 3-SAT: a hidden witness; every clause draws 3 distinct variables and
// random signs, redrawn until the witness satisfies it.
CnfFormula planted_3sat(uint64_t seed, int vars, int clauses) {
  uint64_t ctr = 0;
  auto next = [&] { return hash_stream({seed, 0x33736174, ctr++}); };
  std::vector<int> w(vars + 1);
  for (int v = 1; v <= vars; ++v) w[v] = next() & 1;
  CnfFormula cnf;
  cnf.num_vars = vars;
  for (int c = 0; c < clauses; ++c) {
    int x[3];
    for (int i = 0; i < 3; ++i) {
      for (;;) {
        x[i] = 1 + static_cast<int>(next() % vars);
        bool dup = false;
        for (int k = 0; k < i; ++k) dup |= x[k] == x[i];
        if (!dup) break;
      }
    }
    for (;;) {
      Clause cl;
      bool sat = false;
      for (int i = 0; i < 3; ++i) {
        bool neg = next() & 1;
        cl.push_back(Literal{x[i], neg});
        sat |= (w[x[i]] != 0) != neg;
      }
      if (sat) {
        cnf.clauses.push_back(cl);
        break;
      }
    }
  }
  return cnf;
}

template <typename S>
Mat<S> to_mat(const S* data, int rows, int cols) {
  Mat<S> m(rows, cols);
  if (static_cast<size_t>(rows) * cols != 0) std::memcpy(m.a.data(), data, sizeof(S) * m.a.size());
  return m;
}

#define GUARD_BEGIN try {
#define GUARD_END(ret)              \
  }                                 \
  catch (const std::exception& e) { \
    g_err = e.what();               \
    return ret;                     \
  }

template <typename S>
int forward_t(RefInst* h, const int32_t* cols, int ncols, const S* p, int batch,
              S* tape, S* y, int threads) {
  GUARD_BEGIN
  std::vector<int> c(cols, cols + ncols);
  ForwardResult<S> f = forward(h->circuit, c, to_mat(p, batch, ncols), threads);
  if (tape) std::memcpy(tape, f.tape.values.data(), sizeof(S) * f.tape.values.size());
  if (y) std::memcpy(y, f.y.a.data(), sizeof(S) * f.y.a.size());
  return 0;
  GUARD_END(-1)
}

template <typename S>
int backward_t(RefInst* h, const int32_t* cols, int ncols, const S* tape,
               int batch, const uint8_t* targets, const S* v, S* dv, S* dp,
               int threads) {
  GUARD_BEGIN
  std::vector<int> c(cols, cols + ncols);
  ForwardTape<S> t;
  t.batch = batch;
  t.values.assign(tape, tape + h->circuit.nodes.size() * static_cast<size_t>(batch));
  std::vector<uint8_t> tg(targets, targets + h->circuit.outputs.size());
  BackwardResult<S> b = backward(h->circuit, c, t, tg, to_mat(v, batch, ncols), threads);
  if (dv) std::memcpy(dv, b.dv.a.data(), sizeof(S) * b.dv.a.size());
  if (dp) std::memcpy(dp, b.dp.a.data(), sizeof(S) * b.dp.a.size());
  return 0;
  GUARD_END(-1)
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_from_dimacs(const char* text) {
  GUARD_BEGIN
  return finish(parse_dimacs(text));
  GUARD_END(nullptr)
}

// The same with a non-default ExtractorConfig (extract.hpp:14-17).
void* ref_from_dimacs_cfg(const char* text, int complement_cap, int minimize_cap) {
  GUARD_BEGIN
  ExtractorConfig cfg;
  cfg.complement_cap = complement_cap;
  cfg.minimize_cap = minimize_cap;
  return finish(parse_dimacs(text), cfg);
  GUARD_END(nullptr)
}

// kind: 0 = encode(random_circuit(p0..p4)), 1 = encode(or_chain(p0..p5)),
//       2 = planted_3sat(p0, p1, p2),
//       3 = encode(single gate signature (TKind p0, arity p1)) exactly as the
//           acceptance corpus builds it (acceptance_main.cpp:66-83)
void* ref_generate(int kind, const int64_t* p) {
  GUARD_BEGIN
  switch (kind) {
    case 0:
      return finish(testgen::encode(testgen::random_circuit(
          static_cast<uint64_t>(p[0]), static_cast<int>(p[1]), static_cast<int>(p[2]),
          static_cast<int>(p[3]), static_cast<int>(p[4]))));
    case 1:
      return finish(testgen::encode(or_chain(static_cast<uint64_t>(p[0]), static_cast<int>(p[1]),
                                             static_cast<int>(p[2]), static_cast<int>(p[3]),
                                             static_cast<int>(p[4]), static_cast<int>(p[5]))));
    case 2:
      return finish(planted_3sat(static_cast<uint64_t>(p[0]), static_cast<int>(p[1]),
                                 static_cast<int>(p[2])));
    case 3: {
      int n = static_cast<int>(p[1]);
      testgen::TCircuit tc;
      tc.num_inputs = n;
      tc.num_vars = n + 1;
      testgen::TGate g;
      g.kind = static_cast<testgen::TKind>(p[0]);
      g.out = n + 1;
      for (int i = 1; i <= n; ++i) g.args.push_back(i);
      tc.gates.push_back(g);
      Assignment witness(n + 1, 0xFF);
      for (int i = 1; i <= n; ++i)
        witness[i] = static_cast<uint8_t>(hash_stream({7u, uint64_t(n), uint64_t(i)}) & 1);
      Assignment full = testgen::eval_netlist(tc, witness);
      tc.outputs.push_back({g.out, full[g.out] != 0});
      return finish(testgen::encode(tc));
    }
  }
  throw std::invalid_argument("unknown generator");
  GUARD_END(nullptr)
}

void ref_free(void* h) { delete static_cast<RefInst*>(h); }

const char* ref_dimacs(void* hv, int64_t* len) {
  RefInst* h = static_cast<RefInst*>(hv);
  h->scratch = write_dimacs(h->cnf);
  *len = static_cast<int64_t>(h->scratch.size());
  return h->scratch.c_str();
}

const char* ref_circuit_json(void* hv, int64_t* len) {
  RefInst* h = static_cast<RefInst*>(hv);
  h->scratch = export_json(h->circuit, h->res);
  *len = static_cast<int64_t>(h->scratch.size());
  return h->scratch.c_str();
}

const char* ref_unsat_note(void* hv) {
  return static_cast<RefInst*>(hv)->res.unsat_note.c_str();
}

// out[0..9] = num_vars, clauses, literals, nodes, inputs, outputs, cpi, ucpi,
//             unsat, max_var
void ref_sizes(void* hv, int64_t* out) {
  RefInst* h = static_cast<RefInst*>(hv);
  int64_t lits = 0;
  for (const Clause& c : h->cnf.clauses) lits += static_cast<int64_t>(c.size());
  out[0] = h->cnf.num_vars;
  out[1] = static_cast<int64_t>(h->cnf.clauses.size());
  out[2] = lits;
  out[3] = static_cast<int64_t>(h->circuit.nodes.size());
  out[4] = static_cast<int64_t>(h->circuit.inputs.size());
  out[5] = static_cast<int64_t>(h->circuit.outputs.size());
  out[6] = static_cast<int64_t>(h->paths.constrained_pi.size());
  out[7] = static_cast<int64_t>(h->paths.unconstrained_pi.size());
  out[8] = h->res.unsat ? 1 : 0;
  out[9] = static_cast<int64_t>(h->node_of_var.size()) - 1;
}

void ref_export(void* hv, int32_t* kind, int32_t* a, int32_t* b, int32_t* var,
                int32_t* inputs, int32_t* out_var, uint8_t* out_tgt, int32_t* cpi,
                int32_t* ucpi, int64_t* clause_ptr, int32_t* clause_lit,
                int32_t* node_of_var) {
  RefInst* h = static_cast<RefInst*>(hv);
  const Circuit& c = h->circuit;
  for (size_t i = 0; i < c.nodes.size(); ++i) {
    kind[i] = static_cast<int32_t>(c.nodes[i].kind);
    a[i] = c.nodes[i].a;
    b[i] = c.nodes[i].b;
    var[i] = c.nodes[i].var;
  }
  for (size_t i = 0; i < c.inputs.size(); ++i) inputs[i] = c.inputs[i];
  for (size_t i = 0; i < c.outputs.size(); ++i) {
    out_var[i] = c.outputs[i].var;
    out_tgt[i] = c.outputs[i].target ? 1 : 0;
  }
  for (size_t i = 0; i < h->paths.constrained_pi.size(); ++i) cpi[i] = h->paths.constrained_pi[i];
  for (size_t i = 0; i < h->paths.unconstrained_pi.size(); ++i)
    ucpi[i] = h->paths.unconstrained_pi[i];
  int64_t k = 0;
  clause_ptr[0] = 0;
  for (size_t i = 0; i < h->cnf.clauses.size(); ++i) {
    for (const Literal& l : h->cnf.clauses[i]) clause_lit[k++] = to_dimacs(l);
    clause_ptr[i + 1] = k;
  }
  for (size_t v = 0; v < h->node_of_var.size(); ++v) node_of_var[v] = h->node_of_var[v];
}

int ref_init_soft_inputs(int batch, int cols, uint64_t seed, int restart, double* out) {
  GUARD_BEGIN
  Mat<double> v = init_soft_inputs(batch, cols, seed, restart);
  if (!v.a.empty()) std::memcpy(out, v.a.data(), sizeof(double) * v.a.size());
  return 0;
  GUARD_END(-1)
}

uint64_t ref_hash_stream(const uint64_t* xs, int n) {
  uint64_t h = 0x243f6a8885a308d3ull;
  // hash_stream takes an initializer_list; this loop is the same fold
  // (rng.hpp:21-25) over an arbitrary-length tuple.
  for (int i = 0; i < n; ++i) h = mix64(h ^ mix64(xs[i]));
  return h;
}

uint64_t ref_hash5(uint64_t a, uint64_t b, uint64_t c, uint64_t d, uint64_t e) {
  return hash_stream({a, b, c, d, e});
}

uint64_t ref_hash6(uint64_t a, uint64_t b, uint64_t c, uint64_t d, uint64_t e, uint64_t f) {
  return hash_stream({a, b, c, d, e, f});
}

int ref_embed_f32(const float* v, int64_t n, float* p) {
  Mat<float> m = to_mat(v, 1, static_cast<int>(n));
  Mat<float> r = embed(m);
  std::memcpy(p, r.a.data(), sizeof(float) * n);
  return 0;
}

int ref_forward_f32(void* h, const int32_t* cols, int ncols, const float* p, int batch,
                    float* tape, float* y, int threads) {
  return forward_t<float>(static_cast<RefInst*>(h), cols, ncols, p, batch, tape, y, threads);
}
int ref_forward_f64(void* h, const int32_t* cols, int ncols, const double* p, int batch,
                    double* tape, double* y, int threads) {
  return forward_t<double>(static_cast<RefInst*>(h), cols, ncols, p, batch, tape, y, threads);
}
int ref_backward_f32(void* h, const int32_t* cols, int ncols, const float* tape, int batch,
                     const uint8_t* targets, const float* v, float* dv, float* dp, int threads) {
  return backward_t<float>(static_cast<RefInst*>(h), cols, ncols, tape, batch, targets, v, dv,
                           dp, threads);
}
int ref_backward_f64(void* h, const int32_t* cols, int ncols, const double* tape, int batch,
                     const uint8_t* targets, const double* v, double* dv, double* dp,
                     int threads) {
  return backward_t<double>(static_cast<RefInst*>(h), cols, ncols, tape, batch, targets, v, dv,
                            dp, threads);
}

int ref_loss_f32(const float* y, int rows, int cols, const uint8_t* targets, float* per_row,
                 float* total) {
  GUARD_BEGIN
  LossResult<float> l = loss(to_mat(y, rows, cols), std::vector<uint8_t>(targets, targets + cols));
  if (per_row) std::memcpy(per_row, l.per_row.data(), sizeof(float) * rows);
  *total = l.total;
  return 0;
  GUARD_END(-1)
}

int ref_gd_step_f32(float* v, const float* g, int64_t n, float lr) {
  Mat<float> m = to_mat(v, 1, static_cast<int>(n));
  gd_step(m, to_mat(g, 1, static_cast<int>(n)), lr);
  std::memcpy(v, m.a.data(), sizeof(float) * n);
  return 0;
}

int ref_harden_f32(const float* v, int64_t n, uint8_t* bits) {
  std::vector<uint8_t> b = harden(to_mat(v, 1, static_cast<int>(n)));
  std::memcpy(bits, b.data(), n);
  return 0;
}

// eval_discrete (circuit.cpp:124-152) for one row: pi_values indexed by var.
int ref_eval_discrete(void* hv, const uint8_t* pi_values, int64_t len, uint8_t* out,
                      int64_t out_len) {
  GUARD_BEGIN
  RefInst* h = static_cast<RefInst*>(hv);
  Assignment a(pi_values, pi_values + len);
  Assignment full = eval_discrete(h->circuit, a);
  for (int64_t i = 0; i < out_len; ++i) out[i] = i < static_cast<int64_t>(full.size()) ? full[i] : 0xFF;
  return 0;
  GUARD_END(-1)
}

int ref_eval_cnf(void* hv, const uint8_t* a, int64_t len) {
  GUARD_BEGIN
  RefInst* h = static_cast<RefInst*>(hv);
  return eval_cnf(h->cnf, Assignment(a, a + len)) ? 1 : 0;
  GUARD_END(-1)
}

// satgrad::run (sampler.cpp:198-203). restart: 0 None, 1 ReinitOnExhaust.
int ref_run(void* hv, int batch, int iterations, double lr, uint64_t seed,
            int64_t max_solutions, double timeout_s, int restart, int threads,
            int use_f32) {
  GUARD_BEGIN
  RefInst* h = static_cast<RefInst*>(hv);
  SamplerConfig cfg;
  cfg.batch = batch;
  cfg.iterations = iterations;
  cfg.learning_rate = lr;
  cfg.seed = seed;
  cfg.max_solutions = max_solutions;
  cfg.timeout_s = timeout_s;
  cfg.restart = restart ? RestartPolicy::ReinitOnExhaust : RestartPolicy::None;
  cfg.threads = threads;
  cfg.use_f32 = use_f32 != 0;
  h->run = run(h->cnf, h->circuit, h->res, h->paths, cfg);
  h->has_run = true;
  return 0;
  GUARD_END(-1)
}

// out: unique, attempts, restarts, timed_out, n_loss, n_new_unique, key_words
void ref_run_stats(void* hv, int64_t* out, double* wall_and_tput) {
  RefInst* h = static_cast<RefInst*>(hv);
  const RunStats& s = h->run.stats;
  out[0] = s.unique_count;
  out[1] = s.attempts;
  out[2] = s.restarts;
  out[3] = s.timed_out ? 1 : 0;
  out[4] = static_cast<int64_t>(s.loss_trace.size());
  out[5] = static_cast<int64_t>(s.new_unique.size());
  out[6] = (h->cnf.num_vars + 63) / 64;
  wall_and_tput[0] = s.wall_time_s;
  wall_and_tput[1] = s.throughput;
}

void ref_run_traces(void* hv, double* loss, int64_t* new_unique) {
  RefInst* h = static_cast<RefInst*>(hv);
  const RunStats& s = h->run.stats;
  for (size_t i = 0; i < s.loss_trace.size(); ++i) loss[i] = s.loss_trace[i];
  for (size_t i = 0; i < s.new_unique.size(); ++i) new_unique[i] = s.new_unique[i];
}

const char* ref_run_note(void* hv) { return static_cast<RefInst*>(hv)->run.stats.note.c_str(); }

// Insertion-ordered dedupe keys (sampler.cpp:18-26) of every solution.
void ref_run_keys(void* hv, uint64_t* keys) {
  RefInst* h = static_cast<RefInst*>(hv);
  int nv = h->cnf.num_vars;
  size_t words = (nv + 63) / 64;
  for (long long i = 0; i < h->run.solutions.size(); ++i) {
    std::vector<uint64_t> k = dedupe_key(h->run.solutions.assignment(i), nv);
    std::memcpy(keys + i * words, k.data(), words * sizeof(uint64_t));
  }
}

// format_solutions (sampler.cpp:78-85) of n keys [n][words] (dedupe_key
// layout) inserted in order into a SolutionSet; returns the text length and
// copies min(len, cap) bytes into out (out may be null to size it).
long long ref_format_keys(const uint64_t* keys, long long n, int num_vars, char* out, long long cap) {
  GUARD_BEGIN
  SolutionSet s(num_vars);
  const int words = (num_vars + 63) / 64;
  Assignment a(num_vars + 1, 0);
  for (long long i = 0; i < n; ++i) {
    for (int v = 1; v <= num_vars; ++v) a[v] = (keys[i * words + (v - 1) / 64] >> ((v - 1) % 64)) & 1;
    s.insert(a);
  }
  const std::string t = format_solutions(s);
  if (out) std::memcpy(out, t.data(), std::min<long long>(cap, static_cast<long long>(t.size())));
  return static_cast<long long>(t.size());
  GUARD_END(-1)
}

// Extraction timing and lists: parse once, then time
// satgrad::extract and satgrad::build separately; out_s = {extract, build}.
int ref_extract_seconds(const char* text, int repeats, double* out_s) {
  GUARD_BEGIN
  CnfFormula cnf = parse_dimacs(text);
  double te = 0, tb = 0;
  for (int r = 0; r < std::max(1, repeats); ++r) {
    auto t0 = std::chrono::steady_clock::now();
    ExtractionResult res = extract(cnf);
    auto t1 = std::chrono::steady_clock::now();
    Circuit c = build(res);
    auto t2 = std::chrono::steady_clock::now();
    te += std::chrono::duration<double>(t1 - t0).count();
    tb += std::chrono::duration<double>(t2 - t1).count();
  }
  out_s[0] = te / std::max(1, repeats);
  out_s[1] = tb / std::max(1, repeats);
  return 0;
  GUARD_END(-1)
}

// ExtractionResult list sizes {pi, po, iv, aux, be} and the iv / aux lists.
void ref_extraction_lists(void* hv, int64_t* sizes, int32_t* iv, int32_t* aux) {
  const ExtractionResult& r = static_cast<RefInst*>(hv)->res;
  sizes[0] = static_cast<int64_t>(r.pi.size());
  sizes[1] = static_cast<int64_t>(r.po.size());
  sizes[2] = static_cast<int64_t>(r.iv.size());
  sizes[3] = static_cast<int64_t>(r.aux.size());
  sizes[4] = static_cast<int64_t>(r.be.size());
  if (iv) std::copy(r.iv.begin(), r.iv.end(), iv);
  if (aux) std::copy(r.aux.begin(), r.aux.end(), aux);
}

// The verify subcommand's per-line checks (cmd_verify, tools/satgrad_main.cpp:
// 242-302; the tool itself needs CLI11, absent here) restated over the
// reference's own parse_dimacs / eval_cnf / SolutionSet, with istream token
// semantics.  out = {checked, err_line, err_var, err_kind, wall_ns}; kinds as
// sgx_verify_solutions.  TEST INFRASTRUCTURE: the checker and CPU baseline.
int ref_verify_text(void* hv, const char* text, int64_t len, int64_t* out) {
  GUARD_BEGIN
  const CnfFormula& cnf = static_cast<RefInst*>(hv)->cnf;
  const auto t0 = std::chrono::steady_clock::now();
  std::istringstream in(std::string(text, static_cast<size_t>(len)));
  SolutionSet seen(cnf.num_vars);
  std::string row;
  int64_t lineno = 0, checked = 0, err_line = 0, err_var = 0, kind = 0;
  while (kind == 0 && std::getline(in, row)) {
    ++lineno;
    std::istringstream tok(row);
    Assignment a(cnf.num_vars + 1, 0xFF);
    bool done = false, nonblank = false;
    long long x;
    while (tok >> x) {
      nonblank = true;
      if (x == 0) {
        done = true;
        break;
      }
      const long long v = x < 0 ? -x : x;
      if (v > cnf.num_vars) {
        kind = 1;
        err_var = v;
        break;
      }
      const uint8_t b = x > 0 ? 1 : 0;
      if (a[v] != 0xFF && a[v] != b) {
        kind = 2;
        err_var = v;
        break;
      }
      a[v] = b;
    }
    if (kind) break;
    if (!nonblank) continue;
    if (!done) {
      kind = 3;
      break;
    }
    for (int v = 1; v <= cnf.num_vars && !kind; ++v)
      if (a[v] == 0xFF) {
        kind = 4;
        err_var = v;
      }
    if (kind) break;
    if (!eval_cnf(cnf, a)) {
      kind = 5;
      break;
    }
    if (!seen.insert(a)) {
      kind = 6;
      break;
    }
    ++checked;
  }
  if (kind) err_line = lineno;
  out[0] = checked;
  out[1] = err_line;
  out[2] = err_var;
  out[3] = kind;
  out[4] = std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
  return 0;
  GUARD_END(-1)
}

}  // extern "C"
