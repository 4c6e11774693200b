"""ctypes binding of ``libsatgrad_b200.so`` (C-ABI in include/satgrad_b200.h).

There is no fallback: if the library is missing or a call fails, this module
raises.  The sm_100a library is the only implementation of the sampling loop.
"""
from __future__ import annotations

import ctypes as C
import atexit
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libsatgrad_b200.so")

SGX_OK, SGX_E_INVALID, SGX_E_CUDA, SGX_E_NOMEM, SGX_E_STATE = 0, -1, -2, -3, -4

# Every symbol include/satgrad_b200.h declares (tests check the export table).
EXPORTS = [
    "sgx_last_error", "sgx_version", "sgx_open", "sgx_close", "sgx_circuit_upload",
    "sgx_circuit_info", "sgx_circuit_free", "sgx_set_layout_cache_dir", "sgx_layout_digest", "sgx_jit_quiesce", "sgx_layout_stats", "sgx_harvest_clause_mask", "sgx_sampler_create",
    "sgx_sampler_free", "sgx_init", "sgx_step", "sgx_harvest", "sgx_run", "sgx_run_traces",
    "sgx_solution_count", "sgx_key_words", "sgx_fetch_solutions", "sgx_phase_times",
    "sgx_forward", "sgx_backward", "sgx_embed", "sgx_expf", "sgx_fingerprint_stride",
    "sgx_harvest_local", "sgx_harvest_merge", "sgx_harvest_commit", "sgx_read_logits",
    "sgx_set_host_stream", "sgx_solutions_take", "sgx_host_free", "sgx_step_async", "sgx_step_loss",
    "sgx_format_solutions", "sgx_launch_count", "sgx_extract", "sgx_extraction_sizes",
    "sgx_extraction_export", "sgx_extraction_note", "sgx_extraction_free", "sgx_verify_solutions",
    "sgx_verify_cnf", "sgx_jit_source", "sgx_sampler_soft_info", "sgx_verify_keys",
    "sgx_run_sharded", "sgx_nccl_unique_id", "sgx_exchange_nccl_create", "sgx_exchange_nccl_destroy",
    "sgx_exchange_local_create", "sgx_exchange_local_destroy", "sgx_run_local_added",
]


class SgxError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"satgrad_b200 error {code}: {msg}")
        self.code = code


class CircuitDesc(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_int32), ("kind", C.POINTER(C.c_int32)), ("a", C.POINTER(C.c_int32)),
        ("b", C.POINTER(C.c_int32)), ("var", C.POINTER(C.c_int32)), ("num_vars", C.c_int32),
        ("n_outputs", C.c_int32), ("out_var", C.POINTER(C.c_int32)),
        ("out_target", C.POINTER(C.c_uint8)), ("n_cpi", C.c_int32),
        ("cpi", C.POINTER(C.c_int32)), ("n_ucpi", C.c_int32), ("ucpi", C.POINTER(C.c_int32)),
        ("n_clauses", C.c_int64), ("clause_ptr", C.POINTER(C.c_int64)),
        ("clause_lit", C.POINTER(C.c_int32)), ("unsat", C.c_int32),
    ]


class SamplerCfg(C.Structure):
    _fields_ = [
        ("batch", C.c_int32), ("iterations", C.c_int32), ("learning_rate", C.c_double),
        ("seed", C.c_uint64), ("max_solutions", C.c_int64), ("timeout_s", C.c_double),
        ("restart_policy", C.c_int32), ("row_offset", C.c_int64),
        ("solution_capacity", C.c_int64), ("max_restarts", C.c_int32), ("soft_kernel", C.c_int32),
        ("optimizer", C.c_int32), ("adam_beta1", C.c_double), ("adam_beta2", C.c_double),
        ("adam_eps", C.c_double), ("reinit_age", C.c_int32),
    ]


class RunStatsC(C.Structure):
    _fields_ = [
        ("unique_count", C.c_int64), ("attempts", C.c_int64), ("wall_time_s", C.c_double),
        ("throughput", C.c_double), ("restarts", C.c_int32), ("timed_out", C.c_int32),
        ("n_loss", C.c_int32), ("n_harvest", C.c_int32), ("unsat", C.c_int32),
        ("reserved", C.c_int32), ("device_ms", C.c_double), ("launches", C.c_int64),
    ]


ALLGATHER_DEVICE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)
ALLGATHER_HOST = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.c_int32)


class Exchange(C.Structure):
    """sgx_exchange: the collectives of sgx_run_sharded."""
    _fields_ = [("user", C.c_void_p), ("rank", C.c_int32), ("nranks", C.c_int32),
                ("allgather_device", ALLGATHER_DEVICE), ("allgather_host", ALLGATHER_HOST)]


_lib = None


def library_path() -> str:
    return LIB_PATH


def load() -> C.CDLL:
    """Load the sm_100a library; raise if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: run `python -m paper_2502_08673_b200.build` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    pvp = C.POINTER(C.c_void_p)
    f32p, f64p = C.POINTER(C.c_float), C.POINTER(C.c_double)
    i64p, u64p = C.POINTER(C.c_int64), C.POINTER(C.c_uint64)
    sigs = {
        "sgx_last_error": (C.c_char_p, []),
        "sgx_version": (C.c_char_p, []),
        "sgx_open": (C.c_int, [C.c_int, pvp]),
        "sgx_close": (C.c_int, [vp]),
        "sgx_circuit_upload": (C.c_int, [vp, C.POINTER(CircuitDesc), pvp]),
        "sgx_circuit_info": (C.c_int, [vp, i64p]),
        "sgx_circuit_free": (C.c_int, [vp]),
        "sgx_set_layout_cache_dir": (C.c_int, [C.c_char_p]),
        "sgx_jit_quiesce": (C.c_int, []),
        "sgx_layout_digest": (C.c_int, [C.POINTER(CircuitDesc), C.POINTER(C.c_uint64), C.POINTER(C.c_int32)]),
        "sgx_layout_stats": (C.c_int, [C.POINTER(CircuitDesc), i64p]),
        "sgx_harvest_clause_mask": (C.c_int, [C.POINTER(CircuitDesc), C.POINTER(C.c_uint8)]),
        "sgx_sampler_create": (C.c_int, [vp, C.POINTER(SamplerCfg), pvp]),
        "sgx_sampler_free": (C.c_int, [vp]),
        "sgx_init": (C.c_int, [vp, i32]),
        "sgx_step": (C.c_int, [vp, f64p]),
        "sgx_harvest": (C.c_int, [vp, i32, i32, i64p, i64p]),
        "sgx_run": (C.c_int, [vp, C.POINTER(RunStatsC)]),
        "sgx_run_traces": (C.c_int, [vp, f64p, i64p]),
        "sgx_solution_count": (i64, [vp]),
        "sgx_key_words": (i32, [vp]),
        "sgx_fetch_solutions": (C.c_int, [vp, i64, i64, u64p]),
        "sgx_phase_times": (C.c_int, [vp, f64p]),
        "sgx_forward": (C.c_int, [vp, f32p, i32, f32p, f32p]),
        "sgx_backward": (C.c_int, [vp, f32p, i32, f32p, f32p, f32p]),
        "sgx_embed": (C.c_int, [vp, f32p, i64, f32p]),
        "sgx_expf": (C.c_int, [vp, f32p, i64, f32p]),
        "sgx_fingerprint_stride": (C.c_int, [vp]),
        "sgx_harvest_local": (C.c_int, [vp, i32, i32, i64p, C.POINTER(C.c_void_p)]),
        "sgx_harvest_merge": (C.c_int, [vp, C.c_void_p, i64p, i32, i32, i64, i64p]),
        "sgx_harvest_commit": (C.c_int, [vp, i64, i64p, i64p]),
        "sgx_read_logits": (C.c_int, [vp, f32p]),
        "sgx_set_host_stream": (C.c_int, [vp, i32]),
        "sgx_solutions_take": (C.c_int, [vp, C.POINTER(C.c_void_p), i64p, i64p]),
        "sgx_host_free": (C.c_int, [C.c_void_p, i64]),
        "sgx_step_async": (C.c_int, [vp, C.POINTER(i32)]),
        "sgx_step_loss": (C.c_int, [vp, i32, f64p]),
        "sgx_format_solutions": (C.c_int, [vp, i64, i64, C.c_void_p, i64, i64p]),
        "sgx_launch_count": (i64, [vp]),
        "sgx_extract": (C.c_int, [i32, C.POINTER(i32), C.POINTER(i32), i64, i32, i32, pvp]),
        "sgx_extraction_sizes": (C.c_int, [vp, i64p]),
        "sgx_extraction_export": (C.c_int, [vp] + [C.POINTER(i32)] * 6 + [C.POINTER(C.c_uint8)]
                                  + [C.POINTER(i32)] * 2),
        "sgx_extraction_note": (C.c_char_p, [vp]),
        "sgx_extraction_free": (None, [vp]),
        "sgx_verify_solutions": (C.c_int, [vp, C.c_char_p, i64, i64p]),
        "sgx_verify_cnf": (C.c_int, [vp, i32, i64p, C.POINTER(i32), i64, C.c_char_p, i64, i64p]),
        "sgx_jit_source": (C.c_int, [C.POINTER(CircuitDesc), C.c_char_p, i64, i64p]),
        "sgx_sampler_soft_info": (C.c_int, [vp, i64p]),
        "sgx_verify_keys": (C.c_int, [vp, u64p, i64, i64p]),
        "sgx_run_sharded": (C.c_int, [vp, C.POINTER(Exchange), C.POINTER(RunStatsC)]),
        "sgx_nccl_unique_id": (C.c_int, [C.c_char_p]),
        "sgx_exchange_nccl_create": (C.c_int, [i32, C.c_char_p, i32, i32, C.POINTER(Exchange)]),
        "sgx_exchange_nccl_destroy": (C.c_int, [C.POINTER(Exchange)]),
        "sgx_exchange_local_create": (C.c_int, [i32, C.POINTER(Exchange)]),
        "sgx_exchange_local_destroy": (C.c_int, [C.POINTER(Exchange)]),
        "sgx_run_local_added": (C.c_int, [vp, i64p]),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    # Background NVRTC compiles (the circuit-specialised soft pass) must end
    # before the interpreter and the C++ runtime tear down (sgx_jit_quiesce).
    atexit.register(L.sgx_jit_quiesce)
    return L


def check(code: int) -> None:
    if code != SGX_OK:
        msg = load().sgx_last_error().decode(errors="replace")
        if code == SGX_E_INVALID:
            raise ValueError(msg)
        raise SgxError(code, msg)


def ptr(a: np.ndarray, ctype):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))
