// Reference-side binding: satgrad::run on a B200 through the C-ABI.
//
// Header-only and templated on nothing but the reference's own public types
// (include/satgrad/{cnf,circuit,extract,sampler}.hpp), so a satgrad
// maintainer drops it in and replaces
//
//     satgrad::RunResult r = satgrad::run(cnf, circuit, res, paths, cfg);
//
// with
//
//     satgrad::RunResult r = satgrad_b200::run(cnf, circuit, res, paths, cfg);
//
// Semantics are the reference's f32 instantiation (cfg.use_f32 = true): the
// same solutions in the same insertion order, the same attempts / restarts /
// new_unique / timed_out, loss_trace within f32 summation error
// (sampler.cpp:89-203).  Errors come back as the exceptions the reference
// throws: std::invalid_argument for bad inputs, std::runtime_error for device
// failures.  Link with libsatgrad_b200.so.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "satgrad/circuit.hpp"
#include "satgrad/cnf.hpp"
#include "satgrad/extract.hpp"
#include "satgrad/sampler.hpp"
#include "satgrad_b200.h"

namespace satgrad_b200 {

inline void check(int rc) {
  if (rc == SGX_OK) return;
  if (rc == SGX_E_INVALID) throw std::invalid_argument(sgx_last_error());
  throw std::runtime_error(std::string("satgrad_b200: ") + sgx_last_error());
}

// One context per device, opened on first use, kept for the process lifetime.
inline sgx_ctx* context(int device = 0) {
  static std::vector<std::pair<int, sgx_ctx*>> ctxs;
  for (auto& dc : ctxs)
    if (dc.first == device) return dc.second;
  sgx_ctx* ctx = nullptr;
  check(sgx_open(device, &ctx));
  ctxs.emplace_back(device, ctx);
  return ctx;
}

// Circuit + CnfFormula + PathClassification -> sgx_circuit_desc arrays.
struct Desc {
  std::vector<int32_t> kind, a, b, var, out_var, cpi, ucpi, lits;
  std::vector<uint8_t> out_tgt;
  std::vector<int64_t> ptr;
  sgx_circuit_desc d{};

  Desc(const satgrad::CnfFormula& cnf, const satgrad::Circuit& c, const satgrad::ExtractionResult& res,
       const satgrad::PathClassification& paths) {
    for (const satgrad::GateNode& n : c.nodes) {  // circuit.hpp:25-29
      kind.push_back(static_cast<int32_t>(n.kind));
      a.push_back(n.a);
      b.push_back(n.b);
      var.push_back(n.var);
    }
    for (const satgrad::PoEntry& p : c.outputs) {
      out_var.push_back(p.var);
      out_tgt.push_back(p.target ? 1 : 0);
    }
    cpi.assign(paths.constrained_pi.begin(), paths.constrained_pi.end());
    ucpi.assign(paths.unconstrained_pi.begin(), paths.unconstrained_pi.end());
    ptr.push_back(0);
    for (const satgrad::Clause& cl : cnf.clauses) {
      for (const satgrad::Literal& l : cl) lits.push_back(satgrad::to_dimacs(l));
      ptr.push_back(static_cast<int64_t>(lits.size()));
    }
    d.n_nodes = static_cast<int32_t>(kind.size());
    d.kind = kind.data();
    d.a = a.data();
    d.b = b.data();
    d.var = var.data();
    d.num_vars = cnf.num_vars;
    d.n_outputs = static_cast<int32_t>(out_var.size());
    d.out_var = out_var.data();
    d.out_target = out_tgt.data();
    d.n_cpi = static_cast<int32_t>(cpi.size());
    d.cpi = cpi.data();
    d.n_ucpi = static_cast<int32_t>(ucpi.size());
    d.ucpi = ucpi.data();
    d.n_clauses = static_cast<int64_t>(cnf.clauses.size());
    d.clause_ptr = ptr.data();
    d.clause_lit = lits.data();
    d.unsat = res.unsat ? 1 : 0;
  }
};

// satgrad::extract + satgrad::build + satgrad::classify_paths (extract.hpp:53,
// 65; circuit.hpp:42) through sgx_extract: the same Circuit node for node,
// the same ExtractionResult lists (pi, iv, po, aux, unsat, unsat_note).
// res.be is left empty -- the definitions live in the circuit's nodes -- so
// paths are classified on the node graph (an input is constrained iff it is
// in the fan-in of an output node), which equals classify_paths(res).
struct Extracted {
  satgrad::ExtractionResult res;
  satgrad::Circuit circuit;
  satgrad::PathClassification paths;
};

inline Extracted extract(const satgrad::CnfFormula& cnf, const satgrad::ExtractorConfig& cfg = {}) {
  std::vector<int32_t> ptr{0}, lits;
  for (const satgrad::Clause& cl : cnf.clauses) {
    for (const satgrad::Literal& l : cl) lits.push_back(satgrad::to_dimacs(l));
    ptr.push_back(static_cast<int32_t>(lits.size()));
  }
  sgx_extraction* x = nullptr;
  check(sgx_extract(cnf.num_vars, ptr.data(), lits.data(), static_cast<int64_t>(cnf.clauses.size()),
                    cfg.complement_cap, cfg.minimize_cap, &x));
  std::unique_ptr<sgx_extraction, void (*)(sgx_extraction*)> hold(x, sgx_extraction_free);
  int64_t sz[7];
  check(sgx_extraction_sizes(x, sz));
  std::vector<int32_t> kind(sz[0]), a(sz[0]), b(sz[0]), var(sz[0]), pi(sz[1]), ov(sz[2]), iv(sz[3]), aux(sz[4]);
  std::vector<uint8_t> ot(sz[2]);
  check(sgx_extraction_export(x, kind.data(), a.data(), b.data(), var.data(), pi.data(), ov.data(), ot.data(),
                              iv.data(), aux.data()));
  Extracted e;
  e.res.num_vars = cnf.num_vars;
  e.res.pi.assign(pi.begin(), pi.end());
  e.res.iv.assign(iv.begin(), iv.end());
  e.res.aux.assign(aux.begin(), aux.end());
  for (size_t i = 0; i < ov.size(); ++i) e.res.po.push_back({ov[i], ot[i] != 0});
  e.res.unsat = sz[6] != 0;
  e.res.unsat_note = sgx_extraction_note(x);
  satgrad::Circuit& c = e.circuit;
  c.num_vars = cnf.num_vars;
  c.inputs = e.res.pi;
  c.outputs = e.res.po;
  for (int64_t i = 0; i < sz[0]; ++i) {
    c.nodes.push_back({static_cast<satgrad::GateKind>(kind[i]), a[i], b[i], var[i]});
    if (var[i] != 0) c.var_to_node.emplace(var[i], static_cast<int>(i));
  }
  std::vector<char> reach(c.nodes.size(), 0);
  for (const satgrad::PoEntry& p : c.outputs) reach[c.node_of(p.var)] = 1;
  for (int64_t i = static_cast<int64_t>(c.nodes.size()) - 1; i >= 0; --i) {
    if (!reach[i]) continue;
    if (c.nodes[i].a >= 0) reach[c.nodes[i].a] = 1;
    if (c.nodes[i].b >= 0) reach[c.nodes[i].b] = 1;
  }
  for (int v : c.inputs) (reach[c.node_of(v)] ? e.paths.constrained_pi : e.paths.unconstrained_pi).push_back(v);
  return e;
}

// `satgrad verify` (cmd_verify, tools/satgrad_main.cpp:242-302) of a
// solution text: the CNF checks run on the GPU.  Returns 0 when every line
// is a distinct satisfying assignment; otherwise the reference's message
// ("<line>: <what>") in *message and the error kind (sgx_verify_solutions).
inline int verify(const satgrad::CnfFormula& cnf, const std::string& text, std::string* message = nullptr,
                  long long* checked = nullptr, int device = 0) {
  std::vector<int64_t> ptr{0};
  std::vector<int32_t> lits;
  for (const satgrad::Clause& cl : cnf.clauses) {
    for (const satgrad::Literal& l : cl) lits.push_back(satgrad::to_dimacs(l));
    ptr.push_back(static_cast<int64_t>(lits.size()));
  }
  int64_t out[5];
  check(sgx_verify_cnf(context(device), cnf.num_vars, ptr.data(), lits.data(),
                       static_cast<int64_t>(cnf.clauses.size()), text.data(), static_cast<int64_t>(text.size()), out));
  static const char* what[7] = {"", "exceeds the variable count", "assigned both ways", "missing 0 terminator",
                                "unassigned", "assignment does not satisfy the formula", "duplicate assignment"};
  if (checked) *checked = out[0];
  if (message) {
    const int k = static_cast<int>(out[3]);
    *message = k == 0 ? "" : std::to_string(out[1]) + ": " + ((k == 1 || k == 2 || k == 4) ? "x" + std::to_string(out[2]) + " " : "") + what[k];
  }
  return static_cast<int>(out[3]);
}

namespace detail {
inline sgx_sampler_cfg sampler_cfg(const satgrad::SamplerConfig& cfg) {
  if (!cfg.use_f32)
    throw std::invalid_argument("satgrad_b200 implements the f32 instantiation (use_f32 = true)");
  sgx_sampler_cfg sc{};
  sc.batch = cfg.batch;
  sc.iterations = cfg.iterations;
  sc.learning_rate = cfg.learning_rate;
  sc.seed = cfg.seed;
  sc.max_solutions = cfg.max_solutions;
  sc.timeout_s = cfg.timeout_s;
  sc.restart_policy = cfg.restart == satgrad::RestartPolicy::ReinitOnExhaust ? SGX_RESTART_REINIT_ON_EXHAUST
                                                                              : SGX_RESTART_NONE;
  return sc;
}

inline void fill_stats(satgrad::RunResult& out, const sgx_run_stats& st, const satgrad::ExtractionResult& res) {
  out.stats.unique_count = st.unique_count;
  out.stats.attempts = st.attempts;
  out.stats.wall_time_s = st.wall_time_s;
  out.stats.throughput = st.throughput;
  out.stats.restarts = st.restarts;
  out.stats.timed_out = st.timed_out != 0;
  if (st.unsat) out.stats.note = res.unsat_note.empty() ? "unsatisfiable by construction" : res.unsat_note;
}

// Keys [first, first + n) of the packed [rows][words] block -> SolutionSet.
inline void insert_keys(satgrad::RunResult& out, const uint64_t* keys, int64_t first, int64_t n, int words,
                        int num_vars) {
  satgrad::Assignment a(num_vars + 1, 0);
  for (int64_t i = first; i < first + n; ++i) {
    for (int v = 1; v <= num_vars; ++v)
      a[v] = (keys[static_cast<size_t>(i) * words + (v - 1) / 64] >> ((v - 1) % 64)) & 1;
    out.solutions.insert(a);
  }
}

struct HostKeys {
  uint64_t* p = nullptr;
  int64_t n = 0, bytes = 0;
  HostKeys() = default;
  HostKeys(const HostKeys&) = delete;
  HostKeys& operator=(const HostKeys&) = delete;
  ~HostKeys() {
    if (p) sgx_host_free(p, bytes);
  }
};
}  // namespace detail

// satgrad::run (sampler.hpp:79-81) on device `device`.
inline satgrad::RunResult run(const satgrad::CnfFormula& cnf, const satgrad::Circuit& c,
                              const satgrad::ExtractionResult& res,
                              const satgrad::PathClassification& paths,
                              const satgrad::SamplerConfig& cfg, int device = 0) {
  sgx_sampler_cfg sc = detail::sampler_cfg(cfg);
  Desc desc(cnf, c, res, paths);
  sgx_circuit* circ = nullptr;
  check(sgx_circuit_upload(context(device), &desc.d, &circ));
  std::unique_ptr<sgx_circuit, int (*)(sgx_circuit*)> circ_guard(circ, sgx_circuit_free);
  sgx_sampler* s = nullptr;
  check(sgx_sampler_create(circ, &sc, &s));
  std::unique_ptr<sgx_sampler, int (*)(sgx_sampler*)> s_guard(s, sgx_sampler_free);
  // The result streams to host memory while the run samples (sgx_drain).
  check(sgx_set_host_stream(s, 1));
  sgx_run_stats st{};
  check(sgx_run(s, &st));

  satgrad::RunResult out;
  out.solutions = satgrad::SolutionSet(cnf.num_vars);
  detail::fill_stats(out, st, res);
  out.stats.loss_trace.resize(st.n_loss);
  std::vector<int64_t> nu(st.n_harvest);
  check(sgx_run_traces(s, out.stats.loss_trace.data(), nu.data()));
  out.stats.new_unique.assign(nu.begin(), nu.end());

  // Solutions in insertion order -> SolutionSet (dedupe_key layout).  The
  // keys are already on the host: take them without a copy.
  const int32_t words = sgx_key_words(s);
  detail::HostKeys hk;
  check(sgx_solutions_take(s, &hk.p, &hk.n, &hk.bytes));
  detail::insert_keys(out, hk.p, 0, hk.n, words, cnf.num_vars);
  return out;
}

// satgrad::run sample-sharded over several GPUs: one host
// thread per entry of `devices` (entries may repeat: {0, 0} runs two ranks on
// one GPU).  Rank g samples global rows [g*b, (g+1)*b) with
// b = cfg.batch / devices.size(), and the ranks exchange 64-bit fingerprints
// once per harvest (sgx_run_sharded over the library's in-process exchange),
// so the result -- the same solutions in the same order, the same counters --
// is satgrad::run at cfg.batch.  The loss trace is the mean over ranks of
// each rank's mean row loss, i.e. the union's mean.
inline satgrad::RunResult run(const satgrad::CnfFormula& cnf, const satgrad::Circuit& c,
                              const satgrad::ExtractionResult& res,
                              const satgrad::PathClassification& paths,
                              const satgrad::SamplerConfig& cfg, const std::vector<int>& devices) {
  const int R = static_cast<int>(devices.size());
  if (R < 1) throw std::invalid_argument("run: empty device list");
  if (R == 1) return run(cnf, c, res, paths, cfg, devices[0]);
  if (cfg.batch % R != 0) throw std::invalid_argument("run: batch must divide evenly over the devices");
  sgx_sampler_cfg sc = detail::sampler_cfg(cfg);
  sc.batch = cfg.batch / R;
  Desc desc(cnf, c, res, paths);
  std::vector<sgx_exchange> ex(R);
  check(sgx_exchange_local_create(R, ex.data()));
  struct Rank {
    sgx_circuit* circ = nullptr;
    sgx_sampler* s = nullptr;
    sgx_run_stats st{};
    int rc = 0;
    std::string err;
  };
  std::vector<Rank> rk(R);
  auto cleanup = [&] {
    for (Rank& r : rk) {
      if (r.s) sgx_sampler_free(r.s);
      if (r.circ) sgx_circuit_free(r.circ);
    }
    sgx_exchange_local_destroy(&ex[0]);
  };
  try {
    for (int g = 0; g < R; ++g) {
      check(sgx_circuit_upload(context(devices[g]), &desc.d, &rk[g].circ));
      sgx_sampler_cfg cg = sc;
      cg.row_offset = static_cast<int64_t>(g) * sc.batch;
      check(sgx_sampler_create(rk[g].circ, &cg, &rk[g].s));
    }
    std::vector<std::thread> th;
    for (int g = 0; g < R; ++g)
      th.emplace_back([&, g] {
        rk[g].rc = sgx_run_sharded(rk[g].s, &ex[g], &rk[g].st);
        if (rk[g].rc) rk[g].err = sgx_last_error();
      });
    for (auto& t : th) t.join();
    for (Rank& r : rk)
      if (r.rc) throw std::runtime_error("satgrad_b200 sharded run: " + r.err);

    satgrad::RunResult out;
    out.solutions = satgrad::SolutionSet(cnf.num_vars);
    detail::fill_stats(out, rk[0].st, res);
    const int nh = rk[0].st.n_harvest, nl = rk[0].st.n_loss;
    out.stats.loss_trace.assign(nl, 0.0);
    std::vector<std::vector<int64_t>> added(R, std::vector<int64_t>(nh));
    std::vector<std::unique_ptr<detail::HostKeys>> keys(R);
    for (int g = 0; g < R; ++g) {
      std::vector<double> lt(nl);
      std::vector<int64_t> nu(nh);
      check(sgx_run_traces(rk[g].s, lt.data(), nu.data()));
      for (int i = 0; i < nl; ++i) out.stats.loss_trace[i] += lt[i] / R;
      if (g == 0) out.stats.new_unique.assign(nu.begin(), nu.end());
      check(sgx_run_local_added(rk[g].s, added[g].data()));
      keys[g] = std::make_unique<detail::HostKeys>();
      check(sgx_solutions_take(rk[g].s, &keys[g]->p, &keys[g]->n, &keys[g]->bytes));
    }
    // insertion order over the union: harvest by harvest, ranks in order
    const int32_t words = sgx_key_words(rk[0].s);
    std::vector<int64_t> at(R, 0);
    for (int h = 0; h < nh; ++h)
      for (int g = 0; g < R; ++g) {
        detail::insert_keys(out, keys[g]->p, at[g], added[g][h], words, cnf.num_vars);
        at[g] += added[g][h];
      }
    keys.clear();
    cleanup();
    return out;
  } catch (...) {
    cleanup();
    throw;
  }
}

}  // namespace satgrad_b200
