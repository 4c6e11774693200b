"""``run`` and friends: the reference's sampler API over the sm_100a library.

Mirrors include/satgrad/sampler.hpp: ``SamplerConfig`` (:23-33),
``SolutionSet`` (:39-55), ``RunStats`` (:57-67), ``RunResult`` (:69-72) and
``run`` (:79-81, sampler.cpp:89-203).  Every call goes through the C-ABI of
``libsatgrad_b200.so``; nothing here computes a sample.

The device implements the reference's single-precision instantiation
(``use_f32 = true``) bit for bit; asking for the double-precision path raises.
"""
from __future__ import annotations

import ctypes as C
import weakref
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .circuit import Circuit, Instance, PathClassification
from .cnf import CnfFormula, format_solution_line, key_to_assignment


class SoftKernel(enum.IntEnum):
    """Soft-pass kernels (sgx_soft_kernel); all are bit-identical."""
    AUTO = 0  # circuit-specialised (NVRTC) kernel for small cones once compiled, else HBM tape
    HBM = 1   # level-synchronous HBM-tape kernels only
    JIT = 2   # compile the specialised kernel at sampler creation and wait for it


class Optimizer(enum.IntEnum):
    """Logit update (sgx_optimizer).  GD is the reference's gd_step; ADAM is an
    opt-in extension with no reference counterpart."""
    GD = 0
    ADAM = 1


class RestartPolicy(enum.IntEnum):
    NONE = 0
    REINIT_ON_EXHAUST = 1
    # extension (no reference counterpart): REINIT_ON_EXHAUST plus, after every
    # harvest, valid-but-duplicate rows redraw their logits (SGX_RESTART_REINIT_ROWS)
    REINIT_ROWS = 2
    # extension: REINIT_ROWS plus rows still invalid `reinit_age` GD steps after
    # their last draw redraw theirs (SGX_RESTART_REINIT_INVALID)
    REINIT_INVALID = 3


@dataclass
class SamplerConfig:
    batch: int = 1024
    iterations: int = 5
    learning_rate: float = 10.0
    seed: int = 1
    max_solutions: int = 0
    timeout_s: float = 0.0
    restart: RestartPolicy = RestartPolicy.NONE
    threads: int = 1          # accepted for API parity; the device ignores it
    use_f32: bool = True      # the device path is the f32 instantiation
    row_offset: int = 0       # global row of local row 0 (sample sharding)
    max_restarts: int = 1000  # sampler.cpp:180 safety valve
    solution_capacity: int = 0
    soft_kernel: SoftKernel = SoftKernel.AUTO
    optimizer: Optimizer = Optimizer.GD
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_eps: float = 1e-8
    reinit_age: int = 2       # RestartPolicy.REINIT_INVALID only


@dataclass
class RunStats:
    unique_count: int = 0
    attempts: int = 0
    wall_time_s: float = 0.0
    throughput: float = 0.0
    loss_trace: list = field(default_factory=list)
    new_unique: list = field(default_factory=list)
    restarts: int = 0
    timed_out: bool = False
    note: str = ""
    phase_ms: dict = field(default_factory=dict)
    device_ms: float = 0.0   # CUDA-event time of the run on the sampler stream
    launches: int = 0        # kernels the run launched


class SolutionSet:
    """Insertion-ordered unique solutions as packed dedupe keys."""

    def __init__(self, num_vars: int, keys: np.ndarray | None = None):
        self.num_vars = num_vars
        words = (num_vars + 63) // 64
        self.keys = keys if keys is not None else np.zeros((0, words), np.uint64)

    def size(self) -> int:
        return int(self.keys.shape[0])

    __len__ = size

    def assignment(self, i: int) -> np.ndarray:
        return key_to_assignment(self.keys[i], self.num_vars)

    def format(self) -> str:  # format_solutions, sampler.cpp:78-85
        return "".join(format_solution_line(k, self.num_vars) + "\n" for k in self.keys)


@dataclass
class RunResult:
    solutions: SolutionSet
    stats: RunStats


_ctx: dict[int, int] = {}


def device_context(device: int = 0) -> int:
    L = _lib.load()
    if device not in _ctx:
        h = C.c_void_p()
        _lib.check(L.sgx_open(device, C.byref(h)))
        _ctx[device] = h.value
    return _ctx[device]


def verify_solutions(cnf: CnfFormula, text, device: int = 0) -> dict:
    """``satgrad verify`` (cmd_verify, tools/satgrad_main.cpp:242-302) from the
    CNF alone: CNF checks on the GPU (sgx_verify_cnf).  Same result dict as
    DeviceCircuit.verify_solutions."""
    L = _lib.load()
    data = text.encode() if isinstance(text, str) else bytes(text)
    ptr = np.ascontiguousarray(cnf.clause_ptr, np.int64)
    lit = np.ascontiguousarray(cnf.clause_lit, np.int32)
    out = np.zeros(5, np.int64)
    _lib.check(L.sgx_verify_cnf(C.c_void_p(device_context(device)), int(cnf.num_vars), _lib.ptr(ptr, C.c_int64),
                                _lib.ptr(lit, C.c_int32), int(cnf.n_clauses), data, len(data),
                                _lib.ptr(out, C.c_int64)))
    checked, line, var, kind, launches = (int(x) for x in out)
    msg = (f"{line}: " + DeviceCircuit.VERIFY_MESSAGES[kind].format(var=var)) if kind else \
        f"verify: {checked} solutions, all satisfying and pairwise distinct"
    return {"checked": checked, "ok": kind == 0, "line": line, "kind": kind, "var": var, "message": msg,
            "launches": launches}


class DeviceCircuit:
    """A circuit + CNF uploaded and levelized on one GPU (sgx_circuit_upload)."""

    def __init__(self, cnf: CnfFormula, circuit: Circuit, paths: PathClassification,
                 unsat: bool = False, device: int = 0):
        self.L = _lib.load()
        self.num_vars = cnf.num_vars
        self.circuit = circuit
        self.paths = paths
        self._keep = [np.ascontiguousarray(x) for x in (
            circuit.kind, circuit.a, circuit.b, circuit.var, circuit.out_var, circuit.out_tgt,
            paths.constrained_pi, paths.unconstrained_pi, cnf.clause_ptr, cnf.clause_lit)]
        self.desc = make_desc(cnf, circuit, paths, unsat, self._keep)
        h = C.c_void_p()
        _lib.check(self.L.sgx_circuit_upload(device_context(device), C.byref(self.desc), C.byref(h)))
        self.h = h.value
        self.device = device

    @classmethod
    def from_instance(cls, inst: Instance, device: int = 0) -> "DeviceCircuit":
        return cls(inst.cnf, inst.circuit, inst.paths, inst.unsat, device)

    def info(self) -> dict:
        out = np.zeros(16, np.int64)
        _lib.check(self.L.sgx_circuit_info(self.h, _lib.ptr(out, C.c_int64)))
        keys = ["nodes", "cone_nodes", "cone_edges", "soft_levels", "bit_levels", "fwd_ops",
                "bwd_ops", "bit_ops", "clauses", "literals", "key_words", "cpi", "ucpi",
                "outputs", "num_vars", "unsat"]
        return dict(zip(keys, (int(x) for x in out)))

    # cmd_verify messages (tools/satgrad_main.cpp:265-295), by err_kind
    VERIFY_MESSAGES = {1: "x{var} exceeds the variable count", 2: "x{var} assigned both ways",
                       3: "missing 0 terminator", 4: "x{var} unassigned",
                       5: "assignment does not satisfy the formula", 6: "duplicate assignment"}

    def verify_solutions(self, text) -> dict:
        """``satgrad verify`` (cmd_verify, tools/satgrad_main.cpp:242-302) of a
        solution text against this circuit's CNF, CNF checks on the GPU.
        Returns {checked, ok, line, kind, var, message, launches}."""
        data = text.encode() if isinstance(text, str) else bytes(text)
        out = np.zeros(5, np.int64)
        _lib.check(self.L.sgx_verify_solutions(self.h, data, len(data), _lib.ptr(out, C.c_int64)))
        checked, line, var, kind, launches = (int(x) for x in out)
        msg = (f"{line}: " + self.VERIFY_MESSAGES[kind].format(var=var)) if kind else \
            f"verify: {checked} solutions, all satisfying and pairwise distinct"
        return {"checked": checked, "ok": kind == 0, "line": line, "kind": kind, "var": var,
                "message": msg, "launches": launches}

    def verify_keys(self, keys: np.ndarray) -> dict:
        """Device check of packed solution keys against the CNF: counts of keys
        that do not satisfy it, that are malformed, and that repeat an earlier key."""
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        out = np.zeros(5, np.int64)
        _lib.check(self.L.sgx_verify_keys(self.h, _lib.ptr(keys, C.c_uint64) if keys.size else None,
                                          keys.shape[0] if keys.ndim == 2 else 0, _lib.ptr(out, C.c_int64)))
        return {"checked": int(out[0]), "unsat": int(out[1]), "malformed": int(out[2]),
                "duplicate": int(out[3]), "invalid": int(out[1] + out[2] + out[3])}

    def close(self):
        if getattr(self, "h", None):
            self.L.sgx_circuit_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def make_desc(cnf, circuit, paths, unsat, keep) -> _lib.CircuitDesc:
    kind, a, b, var, out_var, out_tgt, cpi, ucpi, cptr, clit = keep
    d = _lib.CircuitDesc()
    d.n_nodes = len(kind)
    d.kind, d.a, d.b, d.var = (_lib.ptr(x, C.c_int32) for x in (kind, a, b, var))
    d.num_vars = cnf.num_vars
    d.n_outputs = len(out_var)
    d.out_var = _lib.ptr(out_var, C.c_int32)
    d.out_target = _lib.ptr(out_tgt, C.c_uint8)
    d.n_cpi, d.cpi = len(cpi), _lib.ptr(cpi, C.c_int32)
    d.n_ucpi, d.ucpi = len(ucpi), _lib.ptr(ucpi, C.c_int32)
    d.n_clauses = len(cptr) - 1
    d.clause_ptr = _lib.ptr(cptr, C.c_int64)
    d.clause_lit = _lib.ptr(clit, C.c_int32)
    d.unsat = 1 if unsat else 0
    return d


def layout_stats(cnf, circuit, paths, unsat=False) -> dict:
    """Host-only levelization (no GPU needed)."""
    L = _lib.load()
    keep = [np.ascontiguousarray(x) for x in (
        circuit.kind, circuit.a, circuit.b, circuit.var, circuit.out_var, circuit.out_tgt,
        paths.constrained_pi, paths.unconstrained_pi, cnf.clause_ptr, cnf.clause_lit)]
    d = make_desc(cnf, circuit, paths, unsat, keep)
    out = np.zeros(16, np.int64)
    _lib.check(L.sgx_layout_stats(C.byref(d), _lib.ptr(out, C.c_int64)))
    keys = ["nodes", "cone_nodes", "cone_edges", "soft_levels", "bit_levels", "fwd_ops",
            "bwd_ops", "bit_ops", "clauses", "literals", "key_words", "cpi", "ucpi", "outputs",
            "num_vars", "unsat"]
    return dict(zip(keys, (int(x) for x in out)))


def jit_quiesce() -> None:
    """Wait for background compiles of the circuit-specialised soft pass
    (sgx_jit_quiesce): afterwards every eligible sampler runs it."""
    _lib.check(_lib.load().sgx_jit_quiesce())


def set_layout_cache_dir(path: str | None) -> None:
    """On-disk layout cache for every later circuit upload (sgx_set_layout_cache_dir):
    <path>/<descriptor hash>.sgxlayout is read if valid, else compiled and written."""
    _lib.check(_lib.load().sgx_set_layout_cache_dir(path.encode() if path else None))


def layout_digest(cnf, circuit, paths, unsat=False) -> tuple[int, int]:
    """Host only: (digest of the layout an upload would use, source 0 compiled /
    1 in-process cache / 2 disk cache)."""
    L = _lib.load()
    keep = [np.ascontiguousarray(x) for x in (
        circuit.kind, circuit.a, circuit.b, circuit.var, circuit.out_var, circuit.out_tgt,
        paths.constrained_pi, paths.unconstrained_pi, cnf.clause_ptr, cnf.clause_lit)]
    d = make_desc(cnf, circuit, paths, unsat, keep)
    dig, src = C.c_uint64(), C.c_int32()
    _lib.check(L.sgx_layout_digest(C.byref(d), C.byref(dig), C.byref(src)))
    return int(dig.value), int(src.value)


def harvest_clause_mask(cnf, circuit, paths, unsat=False) -> np.ndarray:
    """Host only: uint8 per CNF clause, 1 = implied by the gate definitions or
    the output targets, so the harvest does not check it
    (sgx_harvest_clause_mask; SGX_ALL_CLAUSES=1 disables the pruning)."""
    L = _lib.load()
    keep = [np.ascontiguousarray(x) for x in (
        circuit.kind, circuit.a, circuit.b, circuit.var, circuit.out_var, circuit.out_tgt,
        paths.constrained_pi, paths.unconstrained_pi, cnf.clause_ptr, cnf.clause_lit)]
    d = make_desc(cnf, circuit, paths, unsat, keep)
    out = np.zeros(max(1, len(cnf.clause_ptr) - 1), np.uint8)
    _lib.check(L.sgx_harvest_clause_mask(C.byref(d), _lib.ptr(out, C.c_uint8)))
    return out[:len(cnf.clause_ptr) - 1]


def jit_source(cnf, circuit, paths, unsat=False) -> str:
    """CUDA source of the circuit-specialised soft pass (host only, no GPU)."""
    L = _lib.load()
    keep = [np.ascontiguousarray(x) for x in (
        circuit.kind, circuit.a, circuit.b, circuit.var, circuit.out_var, circuit.out_tgt,
        paths.constrained_pi, paths.unconstrained_pi, cnf.clause_ptr, cnf.clause_lit)]
    d = make_desc(cnf, circuit, paths, unsat, keep)
    n = C.c_int64()
    _lib.check(L.sgx_jit_source(C.byref(d), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value)
    _lib.check(L.sgx_jit_source(C.byref(d), buf, n.value, C.byref(n)))
    return buf.value.decode()


class Sampler:
    """sgx_sampler: device buffers for one batch shape + the run loop."""

    def __init__(self, dc: DeviceCircuit, cfg: SamplerConfig):
        if not cfg.use_f32:
            raise ValueError("the B200 path implements the reference's f32 instantiation "
                             "(SamplerConfig.use_f32 = True)")
        self.L = _lib.load()
        self.dc = dc
        self.cfg = cfg
        c = _lib.SamplerCfg()
        c.batch = cfg.batch
        c.iterations = cfg.iterations
        c.learning_rate = cfg.learning_rate
        c.seed = cfg.seed
        c.max_solutions = cfg.max_solutions
        c.timeout_s = cfg.timeout_s
        c.restart_policy = int(cfg.restart)
        c.row_offset = cfg.row_offset
        c.solution_capacity = cfg.solution_capacity
        c.max_restarts = cfg.max_restarts
        c.soft_kernel = int(cfg.soft_kernel)
        c.optimizer = int(cfg.optimizer)
        c.adam_beta1, c.adam_beta2, c.adam_eps = cfg.adam_beta1, cfg.adam_beta2, cfg.adam_eps
        c.reinit_age = cfg.reinit_age
        self._cfg = c
        h = C.c_void_p()
        _lib.check(self.L.sgx_sampler_create(dc.h, C.byref(c), C.byref(h)))
        self.h = h.value

    def run(self) -> RunStats:
        st = _lib.RunStatsC()
        _lib.check(self.L.sgx_run(self.h, C.byref(st)))
        loss = np.zeros(max(1, st.n_loss), np.float64)
        nu = np.zeros(max(1, st.n_harvest), np.int64)
        _lib.check(self.L.sgx_run_traces(self.h, _lib.ptr(loss, C.c_double),
                                         _lib.ptr(nu, C.c_int64)))
        ph = np.zeros(8, np.float64)
        _lib.check(self.L.sgx_phase_times(self.h, _lib.ptr(ph, C.c_double)))
        names = ["init", "step", "harvest", "forward", "backward", "eval", "keys", "commit"]
        note = ""
        if st.unsat:
            note = getattr(self.dc, "unsat_note", "") or "unsatisfiable by construction"
        return RunStats(unique_count=st.unique_count, attempts=st.attempts,
                        wall_time_s=st.wall_time_s, throughput=st.throughput,
                        loss_trace=[float(x) for x in loss[:st.n_loss]],
                        new_unique=[int(x) for x in nu[:st.n_harvest]], restarts=st.restarts,
                        timed_out=bool(st.timed_out), note=note,
                        phase_ms=dict(zip(names, (float(x) for x in ph))),
                        device_ms=st.device_ms, launches=st.launches)

    def soft_info(self) -> dict:
        """Which soft-pass kernel ran the last step ("hbm" / "jit" / "onchip"),
        steps run by the specialised kernel, its compile state and time, and
        the harvest kernel / words per CTA / samples per lane selected."""
        out = np.zeros(8, np.int64)
        _lib.check(self.L.sgx_sampler_soft_info(self.h, _lib.ptr(out, C.c_int64)))
        return {"last": ["hbm", "jit", "onchip"][int(out[0])], "jit_steps": int(out[1]),
                "jit_state": {-1: "none", 0: "compiling", 1: "ready", 2: "failed"}[int(out[2])],
                "jit_compile_ms": out[3] / 1000.0,
                "harvest": ["global", "smem", "live", "lw"][int(out[4])], "harvest_wpc": int(out[5]),
                "vec": int(out[6]), "padded_batch": int(out[7])}

    def launch_count(self) -> int:
        """Kernels launched since the last run() (or creation)."""
        return int(self.L.sgx_launch_count(self.h))

    def phase_times(self) -> dict:
        ph = np.zeros(8, np.float64)
        _lib.check(self.L.sgx_phase_times(self.h, _lib.ptr(ph, C.c_double)))
        names = ["init", "step", "harvest", "forward", "backward", "eval", "keys", "commit"]
        return dict(zip(names, (float(x) for x in ph)))

    def solution_count(self) -> int:
        return int(self.L.sgx_solution_count(self.h))

    def fetch(self, first: int = 0, count: int | None = None) -> np.ndarray:
        n = self.solution_count()
        if count is None:
            count = n - first
        words = int(self.L.sgx_key_words(self.h))
        out = np.zeros((count, words), np.uint64)
        _lib.check(self.L.sgx_fetch_solutions(self.h, first, count,
                                              _lib.ptr(out, C.c_uint64) if count else None))
        return out

    def set_host_stream(self, on: bool = True):
        """Copy each harvest's new solutions to host memory while sampling runs."""
        _lib.check(self.L.sgx_set_host_stream(self.h, 1 if on else 0))

    def take(self) -> np.ndarray:
        """Every solution key, [n][key_words] uint64 in insertion order, as an
        array that owns the library's host result memory (no copy when host
        streaming already landed it; released when the array is collected)."""
        words = int(self.L.sgx_key_words(self.h))
        p, rows, nbytes = C.c_void_p(), C.c_int64(), C.c_int64()
        _lib.check(self.L.sgx_solutions_take(self.h, C.byref(p), C.byref(rows), C.byref(nbytes)))
        if not p.value or rows.value == 0:
            return np.zeros((0, words), np.uint64)
        return _owned_keys(p.value, rows.value, words, nbytes.value)

    def format_solutions(self, first: int = 0, count: int | None = None) -> bytes:
        """format_solutions (sampler.cpp:78-85) rendered on the device: one
        "v1 -v2 ... vn 0" line per solution, insertion order."""
        n = self.solution_count()
        if count is None:
            count = n - first
        ln = C.c_int64()
        _lib.check(self.L.sgx_format_solutions(self.h, first, count, None, 0, C.byref(ln)))
        buf = np.empty(max(1, ln.value), np.uint8)
        _lib.check(self.L.sgx_format_solutions(self.h, first, count, buf.ctypes.data_as(C.c_void_p),
                                               ln.value, C.byref(ln)))
        return buf[: ln.value].tobytes()

    # building blocks ----------------------------------------------------------
    def logits(self) -> np.ndarray:
        """Current V, [batch][n_cpi] (trajectory parity tap)."""
        ncpi = len(self.dc.paths.constrained_pi)
        v = np.zeros((self.cfg.batch, ncpi), np.float32)
        if v.size:
            _lib.check(self.L.sgx_read_logits(self.h, _lib.ptr(v, C.c_float)))
        return v

    def init(self, restart: int):
        _lib.check(self.L.sgx_init(self.h, restart))

    def step(self) -> float:
        x = C.c_double()
        _lib.check(self.L.sgx_step(self.h, C.byref(x)))
        return x.value

    def harvest(self, restart: int, it: int) -> tuple[int, int]:
        att, add = C.c_int64(), C.c_int64()
        _lib.check(self.L.sgx_harvest(self.h, restart, it, C.byref(att), C.byref(add)))
        return att.value, add.value

    def close(self):
        if getattr(self, "h", None):
            self.L.sgx_sampler_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _owned_keys(addr: int, rows: int, words: int, map_bytes: int) -> np.ndarray:
    """A numpy view of library host memory that frees it (sgx_host_free) when
    the last view is collected."""
    buf = (C.c_uint64 * (rows * words)).from_address(addr)
    weakref.finalize(buf, _lib.load().sgx_host_free, C.c_void_p(addr), map_bytes)
    return np.frombuffer(buf, dtype=np.uint64).reshape(rows, words)


def run(cnf: CnfFormula, circuit: Circuit, paths: PathClassification, cfg: SamplerConfig,
        unsat: bool = False, unsat_note: str = "", device: int = 0) -> RunResult:
    """satgrad::run (sampler.hpp:79-81): upload, sample, fetch every solution."""
    import os
    import time
    trace = os.environ.get("SGX_E2E_TRACE")
    t = [time.perf_counter()]
    dc = DeviceCircuit(cnf, circuit, paths, unsat, device)
    dc.unsat_note = unsat_note
    t.append(time.perf_counter())
    s = Sampler(dc, cfg)
    t_s = time.perf_counter()
    try:
        s.set_host_stream(True)  # the result streams to the host while sampling runs
        t.append(time.perf_counter())
        stats = s.run()
        t.append(time.perf_counter())
        keys = s.take()
        t.append(time.perf_counter())
    finally:
        s.close()
        t.append(time.perf_counter())
        dc.close()
    t.append(time.perf_counter())
    if trace:
        d = [1000 * (b - a) for a, b in zip(t, t[1:])]
        print("[run] circuit %.1f sampler %.1f (create %.1f) run %.1f (device %.1f) take %.1f close sampler %.1f "
              "circuit %.1f ms" % (d[0], d[1], 1000 * (t_s - t[1]), d[2], stats.device_ms, d[3], d[4], d[5]), flush=True)
    return RunResult(SolutionSet(cnf.num_vars, keys), stats)


def run_instance(inst: Instance, cfg: SamplerConfig, device: int = 0) -> RunResult:
    return run(inst.cnf, inst.circuit, inst.paths, cfg, inst.unsat, inst.unsat_note, device)
