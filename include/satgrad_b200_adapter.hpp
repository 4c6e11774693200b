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

// satgrad::run (sampler.hpp:79-81) on device `device`.
inline satgrad::RunResult run(const satgrad::CnfFormula& cnf, const satgrad::Circuit& c,
                              const satgrad::ExtractionResult& res,
                              const satgrad::PathClassification& paths,
                              const satgrad::SamplerConfig& cfg, int device = 0) {
  if (!cfg.use_f32)
    throw std::invalid_argument("satgrad_b200 implements the f32 instantiation (use_f32 = true)");
  Desc desc(cnf, c, res, paths);
  sgx_circuit* circ = nullptr;
  check(sgx_circuit_upload(context(device), &desc.d, &circ));
  std::unique_ptr<sgx_circuit, int (*)(sgx_circuit*)> circ_guard(circ, sgx_circuit_free);
  sgx_sampler_cfg sc{};
  sc.batch = cfg.batch;
  sc.iterations = cfg.iterations;
  sc.learning_rate = cfg.learning_rate;
  sc.seed = cfg.seed;
  sc.max_solutions = cfg.max_solutions;
  sc.timeout_s = cfg.timeout_s;
  sc.restart_policy = cfg.restart == satgrad::RestartPolicy::ReinitOnExhaust ? SGX_RESTART_REINIT_ON_EXHAUST
                                                                              : SGX_RESTART_NONE;
  sgx_sampler* s = nullptr;
  check(sgx_sampler_create(circ, &sc, &s));
  std::unique_ptr<sgx_sampler, int (*)(sgx_sampler*)> s_guard(s, sgx_sampler_free);
  // The result streams to host memory while the run samples (sgx_drain).
  check(sgx_set_host_stream(s, 1));
  sgx_run_stats st{};
  check(sgx_run(s, &st));

  satgrad::RunResult out;
  out.solutions = satgrad::SolutionSet(cnf.num_vars);
  out.stats.unique_count = st.unique_count;
  out.stats.attempts = st.attempts;
  out.stats.wall_time_s = st.wall_time_s;
  out.stats.throughput = st.throughput;
  out.stats.restarts = st.restarts;
  out.stats.timed_out = st.timed_out != 0;
  if (st.unsat) out.stats.note = res.unsat_note.empty() ? "unsatisfiable by construction" : res.unsat_note;
  out.stats.loss_trace.resize(st.n_loss);
  std::vector<int64_t> nu(st.n_harvest);
  check(sgx_run_traces(s, out.stats.loss_trace.data(), nu.data()));
  out.stats.new_unique.assign(nu.begin(), nu.end());

  // Solutions in insertion order -> SolutionSet (dedupe_key layout).  The
  // keys are already on the host: take them without a copy.
  const int32_t words = sgx_key_words(s);
  uint64_t* kp = nullptr;
  int64_t n = 0, map_bytes = 0;
  check(sgx_solutions_take(s, &kp, &n, &map_bytes));
  struct HostKeys {
    uint64_t* p;
    int64_t bytes;
    ~HostKeys() { sgx_host_free(p, bytes); }
  } hold{kp, map_bytes};
  const uint64_t* keys = kp;
  satgrad::Assignment a(cnf.num_vars + 1, 0);
  for (int64_t i = 0; i < n; ++i) {
    for (int v = 1; v <= cnf.num_vars; ++v)
      a[v] = (keys[static_cast<size_t>(i) * words + (v - 1) / 64] >> ((v - 1) % 64)) & 1;
    out.solutions.insert(a);
  }
  return out;
}

}  // namespace satgrad_b200
