"""satgrad_b200: the data-parallel SAT sampling loop of arXiv 2502.08673
(reference: satgrad) rebuilt for B200 (sm_100a).

The host API mirrors the reference's C++ headers (cnf.hpp, circuit.hpp,
sampler.hpp, autodiff.hpp); the sampling loop itself runs in
``libsatgrad_b200.so`` behind the C-ABI of ``include/satgrad_b200.h``.
"""
from .cnf import CnfFormula, ParseError, eval_cnf, parse_dimacs, verify_keys, write_dimacs
from .circuit import (Circuit, Instance, PathClassification, SchemaError, classify_paths,
                      export_json, import_json, load_instance)
from .extract import ExtractionResult, extract_circuit, instance_from_cnf
from .sampler import (DeviceCircuit, Optimizer, RestartPolicy, SoftKernel, jit_source, RunResult, RunStats, Sampler, SamplerConfig,
                      SolutionSet, jit_quiesce, layout_digest, layout_stats, run, run_instance, set_layout_cache_dir,
                      verify_solutions)

__all__ = [
    "CnfFormula", "ParseError", "eval_cnf", "parse_dimacs", "verify_keys", "write_dimacs",
    "Circuit", "Instance", "PathClassification", "SchemaError", "classify_paths", "export_json",
    "import_json", "load_instance", "DeviceCircuit", "RestartPolicy", "RunResult", "RunStats",
    "Sampler", "SamplerConfig", "SolutionSet", "layout_digest", "layout_stats", "run", "run_instance",
    "set_layout_cache_dir", "jit_quiesce",
    "ExtractionResult", "extract_circuit", "instance_from_cnf", "verify_solutions",
]
