"""TEST INFRASTRUCTURE ONLY -- ctypes front ends for the two parity checkers.

* ``RefLib`` drives the UNMODIFIED reference library (satgrad) compiled in place
  from /root/reference/proj by ``oracle/Makefile`` into ``oracle/_ref/``
  (through ``oracle/ref_shim.cpp``).
* ``PortLib`` drives ``oracle/sgx_oracle.c``, our plain-C restatement of the
  reference hot path (autodiff.cpp:12-297, sampler.cpp:18-194), pinned
  bit-for-bit against ``RefLib`` by tests/test_oracle.py.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline leg may
import this module; the product library never links or calls it.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libsatgrad_ref.so")
PORT_SO = os.path.join(HERE, "libsgx_oracle.so")

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def port_available() -> bool:
    return os.path.exists(PORT_SO)


@dataclass
class RunOut:
    unique: int
    attempts: int
    restarts: int
    timed_out: bool
    wall: float
    loss_trace: list = field(default_factory=list)
    new_unique: list = field(default_factory=list)
    keys: np.ndarray | None = None  # [unique, words] uint64, insertion order
    note: str = ""


class RefLib:
    _lib = None

    def __init__(self):
        if RefLib._lib is None:
            if not ref_available():
                raise FileNotFoundError(f"{REF_SO} not built (make -C oracle ref)")
            L = C.CDLL(REF_SO)
            L.ref_last_error.restype = C.c_char_p
            L.ref_from_dimacs.restype = C.c_void_p
            L.ref_from_dimacs.argtypes = [C.c_char_p]
            L.ref_from_dimacs_cfg.restype = C.c_void_p
            L.ref_from_dimacs_cfg.argtypes = [C.c_char_p, C.c_int, C.c_int]
            L.ref_generate.restype = C.c_void_p
            L.ref_generate.argtypes = [C.c_int, _i64p]
            L.ref_free.argtypes = [C.c_void_p]
            L.ref_dimacs.restype = C.c_void_p
            L.ref_dimacs.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
            L.ref_circuit_json.restype = C.c_void_p
            L.ref_circuit_json.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
            L.ref_unsat_note.restype = C.c_char_p
            L.ref_unsat_note.argtypes = [C.c_void_p]
            L.ref_sizes.argtypes = [C.c_void_p, _i64p]
            L.ref_export.argtypes = [C.c_void_p, _i32p, _i32p, _i32p, _i32p, _i32p, _i32p,
                                     _u8p, _i32p, _i32p, _i64p, _i32p, _i32p]
            L.ref_init_soft_inputs.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, _f64p]
            L.ref_hash5.restype = C.c_uint64
            L.ref_hash5.argtypes = [C.c_uint64] * 5
            L.ref_hash6.restype = C.c_uint64
            L.ref_hash6.argtypes = [C.c_uint64] * 6
            L.ref_embed_f32.argtypes = [_f32p, C.c_int64, _f32p]
            L.ref_forward_f32.argtypes = [C.c_void_p, _i32p, C.c_int, _f32p, C.c_int, _f32p,
                                          _f32p, C.c_int]
            L.ref_forward_f64.argtypes = [C.c_void_p, _i32p, C.c_int, _f64p, C.c_int, _f64p,
                                          _f64p, C.c_int]
            L.ref_backward_f32.argtypes = [C.c_void_p, _i32p, C.c_int, _f32p, C.c_int, _u8p,
                                           _f32p, _f32p, _f32p, C.c_int]
            L.ref_backward_f64.argtypes = [C.c_void_p, _i32p, C.c_int, _f64p, C.c_int, _u8p,
                                           _f64p, _f64p, _f64p, C.c_int]
            L.ref_loss_f32.argtypes = [_f32p, C.c_int, C.c_int, _u8p, _f32p,
                                       C.POINTER(C.c_float)]
            L.ref_gd_step_f32.argtypes = [_f32p, _f32p, C.c_int64, C.c_float]
            L.ref_harden_f32.argtypes = [_f32p, C.c_int64, _u8p]
            L.ref_eval_discrete.argtypes = [C.c_void_p, _u8p, C.c_int64, _u8p, C.c_int64]
            L.ref_eval_cnf.argtypes = [C.c_void_p, _u8p, C.c_int64]
            L.ref_run.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_uint64,
                                  C.c_int64, C.c_double, C.c_int, C.c_int, C.c_int]
            L.ref_run_stats.argtypes = [C.c_void_p, _i64p, _f64p]
            L.ref_run_traces.argtypes = [C.c_void_p, _f64p, _i64p]
            L.ref_run_note.restype = C.c_char_p
            L.ref_run_note.argtypes = [C.c_void_p]
            L.ref_run_keys.argtypes = [C.c_void_p, _u64p]
            L.ref_format_keys.restype = C.c_longlong
            L.ref_format_keys.argtypes = [_u64p, C.c_longlong, C.c_int, C.c_void_p, C.c_longlong]
            L.ref_extract_seconds.argtypes = [C.c_char_p, C.c_int, _f64p]
            L.ref_extraction_lists.argtypes = [C.c_void_p, _i64p, _i32p, _i32p]
            L.ref_verify_text.argtypes = [C.c_void_p, C.c_char_p, C.c_int64, _i64p]
            RefLib._lib = L
        self.L = RefLib._lib

    def extract_seconds(self, dimacs: str, repeats: int = 1) -> tuple[float, float]:
        """Reference extract / build wall time on this host (one thread)."""
        out = np.zeros(2, np.float64)
        if self.L.ref_extract_seconds(dimacs.encode(), repeats, out) != 0:
            raise ValueError(self.error())
        return float(out[0]), float(out[1])

    def error(self) -> str:
        return self.L.ref_last_error().decode()

    def hash5(self, *xs) -> int:
        return int(self.L.ref_hash5(*[int(x) for x in xs]))

    def format_keys(self, keys: np.ndarray, num_vars: int) -> bytes:
        """satgrad::format_solutions (sampler.cpp:78-85) of keys inserted in order."""
        keys = np.ascontiguousarray(keys, np.uint64).reshape(-1, (num_vars + 63) // 64 or 1)
        n = len(keys) if num_vars else 0
        ln = self.L.ref_format_keys(keys.ravel() if keys.size else np.zeros(1, np.uint64), n, num_vars, None, 0)
        if ln < 0:
            raise ValueError(self.error())
        buf = C.create_string_buffer(max(1, ln))
        self.L.ref_format_keys(keys.ravel() if keys.size else np.zeros(1, np.uint64), n, num_vars, buf, ln)
        return buf.raw[:ln]

    def hash6(self, *xs) -> int:
        return int(self.L.ref_hash6(*[int(x) for x in xs]))

    def init_soft_inputs(self, batch, cols, seed, restart=0) -> np.ndarray:
        out = np.zeros(max(1, batch * cols), np.float64)
        assert self.L.ref_init_soft_inputs(batch, cols, seed, restart, out) == 0
        return out[: batch * cols].reshape(batch, cols)

    def embed_f32(self, v: np.ndarray) -> np.ndarray:
        v = np.ascontiguousarray(v, np.float32).ravel()
        p = np.zeros_like(v)
        self.L.ref_embed_f32(v, v.size, p)
        return p

    def loss_f32(self, y: np.ndarray, targets) -> tuple[np.ndarray, float]:
        y = np.ascontiguousarray(y, np.float32)
        t = np.ascontiguousarray(targets, np.uint8)
        per = np.zeros(max(1, y.shape[0]), np.float32)
        tot = C.c_float()
        assert self.L.ref_loss_f32(y, y.shape[0], y.shape[1], t, per, C.byref(tot)) == 0
        return per[: y.shape[0]], float(tot.value)

    def gd_step_f32(self, v, g, lr) -> np.ndarray:
        v = np.ascontiguousarray(v, np.float32).copy()
        g = np.ascontiguousarray(g, np.float32)
        self.L.ref_gd_step_f32(v.ravel(), g.ravel(), v.size, lr)
        return v

    def harden_f32(self, v) -> np.ndarray:
        v = np.ascontiguousarray(v, np.float32)
        out = np.zeros(v.size, np.uint8)
        self.L.ref_harden_f32(v.ravel(), v.size, out)
        return out.reshape(v.shape)


class RefInstance:
    """One CNF pushed through the reference pipeline: parse_dimacs (or a
    generator) -> extract -> build -> classify_paths."""

    def __init__(self, handle: int):
        self.lib = RefLib()
        if not handle:
            raise ValueError(self.lib.error())
        self.h = handle
        s = np.zeros(10, np.int64)
        self.lib.L.ref_sizes(self.h, s)
        (self.num_vars, self.n_clauses, self.n_lits, self.n_nodes, self.n_inputs,
         self.n_out, self.n_cpi, self.n_ucpi, unsat, self.max_var) = [int(x) for x in s]
        self.unsat = bool(unsat)
        self.unsat_note = self.lib.L.ref_unsat_note(self.h).decode()
        n = max(1, self.n_nodes)
        self.kind = np.zeros(n, np.int32)
        self.a = np.zeros(n, np.int32)
        self.b = np.zeros(n, np.int32)
        self.var = np.zeros(n, np.int32)
        self.inputs = np.zeros(max(1, self.n_inputs), np.int32)
        self.out_var = np.zeros(max(1, self.n_out), np.int32)
        self.out_tgt = np.zeros(max(1, self.n_out), np.uint8)
        self.cpi = np.zeros(max(1, self.n_cpi), np.int32)
        self.ucpi = np.zeros(max(1, self.n_ucpi), np.int32)
        self.clause_ptr = np.zeros(self.n_clauses + 1, np.int64)
        self.clause_lit = np.zeros(max(1, self.n_lits), np.int32)
        self.node_of_var = np.zeros(self.max_var + 1, np.int32)
        self.lib.L.ref_export(self.h, self.kind, self.a, self.b, self.var, self.inputs,
                              self.out_var, self.out_tgt, self.cpi, self.ucpi, self.clause_ptr,
                              self.clause_lit, self.node_of_var)
        self.kind = self.kind[: self.n_nodes]
        self.a = self.a[: self.n_nodes]
        self.b = self.b[: self.n_nodes]
        self.var = self.var[: self.n_nodes]
        self.inputs = self.inputs[: self.n_inputs]
        self.out_var = self.out_var[: self.n_out]
        self.out_tgt = self.out_tgt[: self.n_out]
        self.cpi = self.cpi[: self.n_cpi]
        self.ucpi = self.ucpi[: self.n_ucpi]
        self.clause_lit = self.clause_lit[: self.n_lits]
        self.out_node = self.node_of_var[self.out_var] if self.n_out else np.zeros(0, np.int32)

    @classmethod
    def from_dimacs(cls, text: str) -> "RefInstance":
        return cls(RefLib().L.ref_from_dimacs(text.encode()))

    @classmethod
    def from_dimacs_cfg(cls, text: str, complement_cap: int, minimize_cap: int) -> "RefInstance":
        return cls(RefLib().L.ref_from_dimacs_cfg(text.encode(), complement_cap, minimize_cap))

    @classmethod
    def random_circuit(cls, seed, inputs, levels, gpl, outs) -> "RefInstance":
        return cls(RefLib().L.ref_generate(0, np.array([seed, inputs, levels, gpl, outs], np.int64)))

    @classmethod
    def or_chain(cls, seed, inputs, levels, gpl, arity, outs) -> "RefInstance":
        return cls(RefLib().L.ref_generate(
            1, np.array([seed, inputs, levels, gpl, arity, outs], np.int64)))

    @classmethod
    def gate_signature(cls, tkind, arity) -> "RefInstance":
        return cls(RefLib().L.ref_generate(3, np.array([tkind, arity], np.int64)))

    @classmethod
    def planted_3sat(cls, seed, nvars, nclauses) -> "RefInstance":
        return cls(RefLib().L.ref_generate(2, np.array([seed, nvars, nclauses], np.int64)))

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.L.ref_free(self.h)
            self.h = None

    def extraction_lists(self):
        """ExtractionResult sizes {pi, po, iv, aux, be} and the iv / aux lists."""
        sz = np.zeros(5, np.int64)
        n = self.num_vars + self.n_clauses + 1  # bounds |iv| (<= vars) and |aux| (<= clauses)
        iv = np.zeros(n, np.int32)
        aux = np.zeros(n, np.int32)
        self.lib.L.ref_extraction_lists(self.h, sz, iv, aux)
        return [int(x) for x in sz], iv[: sz[2]], aux[: sz[3]]

    def verify_text(self, text) -> dict:
        """cmd_verify's checks over the reference's eval_cnf / SolutionSet
        (ref_shim.cpp): {checked, line, var, kind, wall_s}."""
        data = text.encode() if isinstance(text, str) else bytes(text)
        out = np.zeros(5, np.int64)
        if self.lib.L.ref_verify_text(self.h, data, len(data), out) != 0:
            raise ValueError(self.lib.error())
        return {"checked": int(out[0]), "line": int(out[1]), "var": int(out[2]), "kind": int(out[3]),
                "wall_s": out[4] / 1e9}

    def dimacs(self) -> str:
        n = C.c_int64()
        p = self.lib.L.ref_dimacs(self.h, C.byref(n))
        return C.string_at(p, n.value).decode()

    def circuit_json(self) -> str:
        n = C.c_int64()
        p = self.lib.L.ref_circuit_json(self.h, C.byref(n))
        return C.string_at(p, n.value).decode()

    # autodiff.hpp:52-78 ------------------------------------------------------
    def forward(self, cols, p, dtype=np.float32, threads=1):
        cols = np.ascontiguousarray(cols, np.int32)
        p = np.ascontiguousarray(p, dtype)
        batch = p.shape[0]
        tape = np.zeros(max(1, self.n_nodes * batch), dtype)
        y = np.zeros(max(1, batch * self.n_out), dtype)
        fn = self.lib.L.ref_forward_f32 if dtype == np.float32 else self.lib.L.ref_forward_f64
        if fn(self.h, cols, len(cols), p.ravel() if p.size else np.zeros(1, dtype), batch, tape,
              y, threads) != 0:
            raise ValueError(self.lib.error())
        return (tape[: self.n_nodes * batch].reshape(self.n_nodes, batch),
                y[: batch * self.n_out].reshape(batch, self.n_out))

    def backward(self, cols, tape, targets, v, dtype=np.float32, threads=1):
        cols = np.ascontiguousarray(cols, np.int32)
        tape = np.ascontiguousarray(tape, dtype)
        v = np.ascontiguousarray(v, dtype)
        batch = tape.shape[1]
        dv = np.zeros(max(1, v.size), dtype)
        dp = np.zeros(max(1, v.size), dtype)
        fn = self.lib.L.ref_backward_f32 if dtype == np.float32 else self.lib.L.ref_backward_f64
        if fn(self.h, cols, len(cols), tape.ravel(), batch,
              np.ascontiguousarray(targets, np.uint8), v.ravel() if v.size else np.zeros(1, dtype),
              dv, dp, threads) != 0:
            raise ValueError(self.lib.error())
        return dv[: v.size].reshape(v.shape), dp[: v.size].reshape(v.shape)

    def eval_cnf_key(self, key: np.ndarray) -> bool:
        a = np.zeros(self.num_vars + 1, np.uint8)
        for v in range(1, self.num_vars + 1):
            a[v] = (int(key[(v - 1) // 64]) >> ((v - 1) % 64)) & 1
        r = self.lib.L.ref_eval_cnf(self.h, a, a.size)
        if r < 0:
            raise ValueError(self.lib.error())
        return bool(r)

    # sampler.hpp:79-81 --------------------------------------------------------
    def run(self, batch=1024, iterations=5, lr=10.0, seed=1, max_solutions=0, timeout_s=0.0,
            restart=False, threads=1, use_f32=True) -> RunOut:
        if self.lib.L.ref_run(self.h, batch, iterations, lr, seed, max_solutions, timeout_s,
                              1 if restart else 0, threads, 1 if use_f32 else 0) != 0:
            raise ValueError(self.lib.error())
        s = np.zeros(7, np.int64)
        w = np.zeros(2, np.float64)
        self.lib.L.ref_run_stats(self.h, s, w)
        loss = np.zeros(max(1, s[4]), np.float64)
        nu = np.zeros(max(1, s[5]), np.int64)
        self.lib.L.ref_run_traces(self.h, loss, nu)
        keys = np.zeros(max(1, s[0] * s[6]), np.uint64)
        self.lib.L.ref_run_keys(self.h, keys)
        return RunOut(unique=int(s[0]), attempts=int(s[1]), restarts=int(s[2]),
                      timed_out=bool(s[3]), wall=float(w[0]),
                      loss_trace=[float(x) for x in loss[: s[4]]],
                      new_unique=[int(x) for x in nu[: s[5]]],
                      keys=keys[: s[0] * s[6]].reshape(int(s[0]), int(s[6])),
                      note=self.lib.L.ref_run_note(self.h).decode())


class PortLib:
    """Our C restatement (oracle/sgx_oracle.c)."""

    _lib = None

    def __init__(self):
        if PortLib._lib is None:
            if not port_available():
                raise FileNotFoundError(f"{PORT_SO} not built (make -C oracle oracle)")
            L = C.CDLL(PORT_SO)
            L.so_mix64.restype = C.c_uint64
            L.so_mix64.argtypes = [C.c_uint64]
            L.so_hash_stream.restype = C.c_uint64
            L.so_hash_stream.argtypes = [_u64p, C.c_int]
            L.so_init_soft_inputs.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, _f64p]
            L.so_sigmoid.restype = C.c_float
            L.so_sigmoid.argtypes = [C.c_float]
            L.so_embed.argtypes = [_f32p, C.c_int64, _f32p]
            L.so_forward.argtypes = [C.c_int, _i32p, _i32p, _i32p, _i32p, C.c_int, _f32p, C.c_int,
                                     C.c_int, _i32p, _f32p, _f32p]
            L.so_loss.restype = C.c_float
            L.so_loss.argtypes = [_f32p, C.c_int, C.c_int, _u8p, _f32p]
            L.so_backward.argtypes = [C.c_int, _i32p, _i32p, _i32p, _i32p, C.c_int, _f32p,
                                      C.c_int, C.c_int, _i32p, _u8p, _f32p, _f32p, _f32p, _f32p]
            L.so_gd_step.argtypes = [_f32p, _f32p, C.c_int64, C.c_float]
            L.so_harden.argtypes = [_f32p, C.c_int64, _u8p]
            L.so_run.restype = C.c_void_p
            L.so_run.argtypes = [C.c_int, _i32p, _i32p, _i32p, _i32p, C.c_int, C.c_int, _i32p,
                                 C.c_int, _i32p, _u8p, C.c_int, _i32p, C.c_int, _i32p, C.c_int64,
                                 _i64p, _i32p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64,
                                 C.c_int64, C.c_double, C.c_int]
            L.so_run_stats.argtypes = [C.c_void_p, _i64p, C.POINTER(C.c_double)]
            L.so_run_traces.argtypes = [C.c_void_p, _f64p, _i64p]
            L.so_run_keys.argtypes = [C.c_void_p, _u64p]
            L.so_run_free.argtypes = [C.c_void_p]
            L.so_check_key.restype = C.c_int
            L.so_check_key.argtypes = [C.c_int64, _i64p, _i32p, _u64p]
            L.so_expf_range.argtypes = [_f32p, C.c_int64, _f32p]
            PortLib._lib = L
        self.L = PortLib._lib

    def hash_stream(self, *xs) -> int:
        return int(self.L.so_hash_stream(np.array(xs, np.uint64), len(xs)))

    def init_soft_inputs(self, batch, cols, seed, restart=0) -> np.ndarray:
        out = np.zeros(max(1, batch * cols), np.float64)
        self.L.so_init_soft_inputs(batch, cols, seed, restart, out)
        return out[: batch * cols].reshape(batch, cols)

    def embed(self, v) -> np.ndarray:
        v = np.ascontiguousarray(v, np.float32)
        p = np.zeros(max(1, v.size), np.float32)
        self.L.so_embed(v.ravel() if v.size else np.zeros(1, np.float32), v.size, p)
        return p[: v.size].reshape(v.shape)

    def expf(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros_like(x)
        self.L.so_expf_range(x.ravel(), x.size, out.ravel())
        return out

    @staticmethod
    def _col_of_node(inst, cols):
        con = np.full(max(1, inst.n_nodes), -1, np.int32)
        for j, v in enumerate(cols):
            con[inst.node_of_var[v]] = j
        return con

    def forward(self, inst, cols, p):
        p = np.ascontiguousarray(p, np.float32)
        batch = p.shape[0]
        tape = np.zeros(max(1, inst.n_nodes * batch), np.float32)
        y = np.zeros(max(1, batch * inst.n_out), np.float32)
        self.L.so_forward(inst.n_nodes, inst.kind, inst.a, inst.b, self._col_of_node(inst, cols),
                          len(cols), p.ravel() if p.size else np.zeros(1, np.float32), batch,
                          inst.n_out, np.ascontiguousarray(inst.out_node, np.int32), tape, y)
        return (tape[: inst.n_nodes * batch].reshape(inst.n_nodes, batch),
                y[: batch * inst.n_out].reshape(batch, inst.n_out))

    def loss(self, y, targets):
        y = np.ascontiguousarray(y, np.float32)
        per = np.zeros(max(1, y.shape[0]), np.float32)
        tot = self.L.so_loss(y.ravel(), y.shape[0], y.shape[1],
                             np.ascontiguousarray(targets, np.uint8), per)
        return per[: y.shape[0]], float(tot)

    def backward(self, inst, cols, tape, v):
        tape = np.ascontiguousarray(tape, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        batch = tape.shape[1]
        dv = np.zeros(max(1, v.size), np.float32)
        dp = np.zeros(max(1, v.size), np.float32)
        adj = np.zeros(max(1, inst.n_nodes * batch), np.float32)
        self.L.so_backward(inst.n_nodes, inst.kind, inst.a, inst.b, self._col_of_node(inst, cols),
                           len(cols), tape.ravel(), batch, inst.n_out,
                           np.ascontiguousarray(inst.out_node, np.int32),
                           np.ascontiguousarray(inst.out_tgt, np.uint8),
                           v.ravel() if v.size else np.zeros(1, np.float32), dv, dp, adj)
        return dv[: v.size].reshape(v.shape), dp[: v.size].reshape(v.shape)

    def run(self, inst, batch=1024, iterations=5, lr=10.0, seed=1, max_solutions=0,
            timeout_s=0.0, restart=False) -> RunOut:
        h = self.L.so_run(inst.n_nodes, inst.kind, inst.a, inst.b, inst.var, inst.num_vars,
                          inst.max_var, inst.node_of_var, inst.n_out, inst.out_var, inst.out_tgt,
                          len(inst.cpi), inst.cpi, len(inst.ucpi), inst.ucpi, inst.n_clauses,
                          inst.clause_ptr, inst.clause_lit, 1 if inst.unsat else 0, batch,
                          iterations, lr, seed, max_solutions, timeout_s, 1 if restart else 0)
        try:
            s = np.zeros(7, np.int64)
            w = C.c_double()
            self.L.so_run_stats(h, s, C.byref(w))
            loss = np.zeros(max(1, s[4]), np.float64)
            nu = np.zeros(max(1, s[5]), np.int64)
            self.L.so_run_traces(h, loss, nu)
            keys = np.zeros(max(1, s[0] * s[6]), np.uint64)
            self.L.so_run_keys(h, keys)
        finally:
            self.L.so_run_free(h)
        return RunOut(unique=int(s[0]), attempts=int(s[1]), restarts=int(s[2]),
                      timed_out=bool(s[3]), wall=float(w.value),
                      loss_trace=[float(x) for x in loss[: s[4]]],
                      new_unique=[int(x) for x in nu[: s[5]]],
                      keys=keys[: s[0] * s[6]].reshape(int(s[0]), int(s[6])))

    def check_key(self, inst, key) -> bool:
        return bool(self.L.so_check_key(inst.n_clauses, inst.clause_ptr, inst.clause_lit,
                                        np.ascontiguousarray(key, np.uint64)))
