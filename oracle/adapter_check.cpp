// TEST INFRASTRUCTURE ONLY.  Proves the reference-side binding
// (include/satgrad_b200_adapter.hpp) is a drop-in: the UNMODIFIED reference
// pipeline (parse_dimacs -> extract -> build -> classify_paths) feeds both
// satgrad::run (CPU, f32) and satgrad_b200::run (B200), and the two
// RunResults must agree: same solutions in the same order (format_solutions
// byte-identical), same counters, loss traces within f32 summation error.
// Built by `make -C oracle adapter` into oracle/_ref/adapter_check; run by
// tests/test_gpu_parity.py::test_reference_adapter_drop_in.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>

#include "satgrad/sampler.hpp"
#include "satgrad_b200_adapter.hpp"

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: adapter_check <cnf> [batch iters seed quota restart]\n");
    return 2;
  }
  std::ifstream in(argv[1], std::ios::binary);
  std::stringstream ss;
  ss << in.rdbuf();
  satgrad::CnfFormula cnf = satgrad::parse_dimacs(ss.str());
  satgrad::ExtractionResult res = satgrad::extract(cnf);
  satgrad::Circuit c = satgrad::build(res);
  satgrad::PathClassification paths = satgrad::classify_paths(res);
  if (argc > 2 && std::string(argv[2]) == "--extract-only") {
    // satgrad_b200::extract against the reference's extract + build + classify_paths
    satgrad_b200::Extracted x = satgrad_b200::extract(cnf);
    int bad = 0;
    auto same = [&](bool ok, const char* what) {
      if (!ok) {
        std::printf("MISMATCH %s\n", what);
        ++bad;
      }
    };
    same(x.circuit.nodes.size() == c.nodes.size(), "node count");
    for (size_t i = 0; i < c.nodes.size() && i < x.circuit.nodes.size(); ++i) {
      const auto &p = c.nodes[i], &q = x.circuit.nodes[i];
      if (p.kind != q.kind || p.a != q.a || p.b != q.b || p.var != q.var) {
        same(false, "node");
        break;
      }
    }
    same(x.circuit.inputs == c.inputs, "inputs");
    same(x.circuit.var_to_node == c.var_to_node, "var_to_node");
    same(x.res.po.size() == res.po.size(), "po count");
    for (size_t i = 0; i < res.po.size() && i < x.res.po.size(); ++i)
      same(x.res.po[i].var == res.po[i].var && x.res.po[i].target == res.po[i].target, "po");
    same(x.res.iv == res.iv && x.res.aux == res.aux && x.res.pi == res.pi, "iv / aux / pi");
    same(x.res.unsat == res.unsat && x.res.unsat_note == res.unsat_note, "unsat");
    same(x.paths.constrained_pi == paths.constrained_pi && x.paths.unconstrained_pi == paths.unconstrained_pi, "paths");
    std::printf("%s: %zu nodes\n", bad ? "extract MISMATCH" : "extract ok", x.circuit.nodes.size());
    return bad ? 1 : 0;
  }
  satgrad::SamplerConfig cfg;
  cfg.use_f32 = true;
  if (argc > 2) cfg.batch = std::atoi(argv[2]);
  if (argc > 3) cfg.iterations = std::atoi(argv[3]);
  if (argc > 4) cfg.seed = std::strtoull(argv[4], nullptr, 10);
  if (argc > 5) cfg.max_solutions = std::atoll(argv[5]);
  if (argc > 6 && std::atoi(argv[6])) cfg.restart = satgrad::RestartPolicy::ReinitOnExhaust;

  satgrad::RunResult cpu = satgrad::run(cnf, c, res, paths, cfg);
  satgrad::RunResult gpu = satgrad_b200::run(cnf, c, res, paths, cfg);

  int bad = 0;
  auto expect = [&](bool ok, const char* what) {
    if (!ok) {
      std::printf("MISMATCH %s\n", what);
      ++bad;
    }
  };
  expect(satgrad::format_solutions(cpu.solutions) == satgrad::format_solutions(gpu.solutions), "solutions");
  expect(cpu.stats.unique_count == gpu.stats.unique_count, "unique_count");
  expect(cpu.stats.attempts == gpu.stats.attempts, "attempts");
  expect(cpu.stats.new_unique == gpu.stats.new_unique, "new_unique");
  expect(cpu.stats.restarts == gpu.stats.restarts, "restarts");
  expect(cpu.stats.timed_out == gpu.stats.timed_out, "timed_out");
  expect(cpu.stats.loss_trace.size() == gpu.stats.loss_trace.size(), "loss_trace length");
  for (size_t i = 0; i < cpu.stats.loss_trace.size() && i < gpu.stats.loss_trace.size(); ++i) {
    double a = cpu.stats.loss_trace[i], b = gpu.stats.loss_trace[i];
    expect(std::fabs(a - b) <= 1e-4 * std::fmax(std::fabs(a), 1e-30), "loss_trace value");
  }
  // satgrad_b200::run over two ranks (sgx_run_sharded, in-process exchange,
  // both on device 0): the union of the shards is the reference's run
  if (cfg.batch % 2 == 0) {
    satgrad::RunResult sh = satgrad_b200::run(cnf, c, res, paths, cfg, std::vector<int>{0, 0});
    expect(satgrad::format_solutions(cpu.solutions) == satgrad::format_solutions(sh.solutions), "sharded solutions");
    expect(cpu.stats.unique_count == sh.stats.unique_count, "sharded unique_count");
    expect(cpu.stats.attempts == sh.stats.attempts, "sharded attempts");
    expect(cpu.stats.new_unique == sh.stats.new_unique, "sharded new_unique");
    expect(cpu.stats.restarts == sh.stats.restarts, "sharded restarts");
    expect(cpu.stats.loss_trace.size() == sh.stats.loss_trace.size(), "sharded loss_trace length");
    for (size_t i = 0; i < cpu.stats.loss_trace.size() && i < sh.stats.loss_trace.size(); ++i) {
      double a = cpu.stats.loss_trace[i], b = sh.stats.loss_trace[i];
      expect(std::fabs(a - b) <= 1e-4 * std::fmax(std::fabs(a), 1e-30), "sharded loss_trace value");
    }
  }
  // satgrad_b200::verify (cmd_verify on the GPU) on the reference's own text:
  // all lines pass; a repeated first line is a duplicate one line past the end
  {
    const std::string text = satgrad::format_solutions(cpu.solutions);
    std::string msg;
    long long checked = -1;
    const int k = satgrad_b200::verify(cnf, text, &msg, &checked);
    expect(k == 0 && checked == cpu.stats.unique_count, "verify of the reference's solutions");
    if (cpu.stats.unique_count > 0) {
      const std::string dup = text + text.substr(0, text.find('\n') + 1);
      const int k2 = satgrad_b200::verify(cnf, dup, &msg, &checked);
      expect(k2 == 6 && checked == cpu.stats.unique_count &&
                 msg == std::to_string(cpu.stats.unique_count + 1) + ": duplicate assignment",
             "verify duplicate");
    }
  }
  std::printf("%s: %lld unique (cpu %.3f s, b200 %.3f s)\n", bad ? "adapter MISMATCH" : "adapter ok",
              static_cast<long long>(gpu.stats.unique_count), cpu.stats.wall_time_s, gpu.stats.wall_time_s);
  return bad ? 1 : 0;
}
