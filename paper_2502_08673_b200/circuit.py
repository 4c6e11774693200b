"""The reference's circuit netlist on the host, plus instance loading.

``Circuit`` mirrors include/satgrad/circuit.hpp:20-40: a topological node array
(operands always at lower ids), PI vars in classification order, PO entries
with targets, and var -> node.  ``import_json`` / ``export_json`` follow the
reference's lossless JSON schema (circuit.cpp:179-332), the on-disk cache a
reference user already has (``<cnf>.circuit.json``).

``classify_paths`` reproduces extract.cpp:174-193 from the circuit itself: a PI
is constrained iff its node lies in the transitive fan-in of some output node
(the circuit's gates reference exactly the support of each definition, so
node-level and definition-level reachability coincide; tests check this
against the reference on every fixture).  Both lists keep ``inputs`` order,
which keys the RNG columns.

``Instance`` bundles CNF + circuit + paths: what ``run`` consumes.
"""
from __future__ import annotations

import gzip
import json
import os
from dataclasses import dataclass, field

import numpy as np

from .cnf import CnfFormula, parse_dimacs

KINDS = ["INPUT", "CONST0", "CONST1", "BUF", "NOT", "AND2", "OR2", "XOR2", "XNOR2"]
INPUT, CONST0, CONST1, BUF, NOT, AND2, OR2, XOR2, XNOR2 = range(9)
_OPERANDS = [0, 0, 0, 1, 1, 2, 2, 2, 2]


class SchemaError(ValueError):
    """circuit.hpp:55-58."""


@dataclass
class Circuit:
    num_vars: int
    kind: np.ndarray       # int32[N]
    a: np.ndarray          # int32[N], -1 unused
    b: np.ndarray
    var: np.ndarray        # int32[N], 0 = internal
    inputs: np.ndarray     # int32, PI vars (res.pi order)
    out_var: np.ndarray    # int32
    out_tgt: np.ndarray    # uint8
    node_of_var: np.ndarray = field(default=None)  # int32[max_var + 1], -1 = none

    def __post_init__(self):
        for name in ("kind", "a", "b", "var", "inputs", "out_var"):
            setattr(self, name, np.ascontiguousarray(getattr(self, name), np.int32))
        self.out_tgt = np.ascontiguousarray(self.out_tgt, np.uint8)
        if self.node_of_var is None:
            max_var = max(int(self.num_vars), int(self.var.max()) if len(self.var) else 0)
            nov = np.full(max_var + 1, -1, np.int32)
            ids = np.nonzero(self.var)[0]
            nov[self.var[ids]] = ids
            self.node_of_var = nov

    @property
    def n_nodes(self) -> int:
        return len(self.kind)

    @property
    def max_var(self) -> int:
        return len(self.node_of_var) - 1

    def node_of(self, v: int) -> int:
        if v <= 0 or v > self.max_var or self.node_of_var[v] < 0:
            raise ValueError(f"x{v} has no circuit node")
        return int(self.node_of_var[v])

    @property
    def out_node(self) -> np.ndarray:
        return self.node_of_var[self.out_var] if len(self.out_var) else np.zeros(0, np.int32)


@dataclass
class PathClassification:
    constrained_pi: np.ndarray
    unconstrained_pi: np.ndarray


def classify_paths(c: Circuit) -> PathClassification:
    """extract.cpp:174-193 on the node graph."""
    reach = np.zeros(c.n_nodes, bool)
    reach[c.out_node] = True
    ops = np.array(_OPERANDS, np.int32)[c.kind]
    for i in range(c.n_nodes - 1, -1, -1):
        if reach[i]:
            if ops[i] >= 1:
                reach[c.a[i]] = True
            if ops[i] == 2:
                reach[c.b[i]] = True
    nodes = c.node_of_var[c.inputs]
    con = reach[nodes]
    return PathClassification(c.inputs[con].copy(), c.inputs[~con].copy())


def import_json(text: str) -> Circuit:
    """circuit.cpp:250-330 (structure checks included)."""
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise SchemaError(f"bad json: {e}") from None
    try:
        num_vars = int(j["num_vars"])
        if num_vars < 0 or int(j["aux_base"]) != num_vars:
            raise SchemaError("aux_base must equal num_vars")
        inputs = [int(v) for v in j["inputs"]]
        gates = j["gates"]
        n = len(gates)
        kind = np.zeros(n, np.int32)
        a = np.full(n, -1, np.int32)
        b = np.full(n, -1, np.int32)
        var = np.zeros(n, np.int32)
        seen = {}
        for i, g in enumerate(gates):
            if int(g["id"]) != i:
                raise SchemaError("gate ids must be consecutive from 0")
            try:
                k = KINDS.index(g["kind"])
            except ValueError:
                raise SchemaError(f"unknown gate kind '{g['kind']}'") from None
            args = [int(x) for x in g["args"]]
            if len(args) != _OPERANDS[k]:
                raise SchemaError(f"wrong operand count for {KINDS[k]}")
            if any(x >= i or x < -1 for x in args):
                raise SchemaError("operands must reference earlier gates")
            kind[i] = k
            if args:
                a[i] = args[0]
            if len(args) == 2:
                b[i] = args[1]
            if g["var"] is not None:
                v = int(g["var"])
                if v <= 0:
                    raise SchemaError("gate var must be positive")
                if v in seen:
                    raise SchemaError(f"x{v} mapped to two gates")
                seen[v] = i
                var[i] = v
        for v in inputs:
            if v not in seen or kind[seen[v]] != INPUT:
                raise SchemaError(f"input x{v} has no INPUT gate")
        in_set = set(inputs)
        for v, i in seen.items():
            if kind[i] == INPUT and v not in in_set:
                raise SchemaError(f"INPUT gate for x{v} missing from inputs")
        out_var, out_tgt, po = [], [], set()
        for o in j["outputs"]:
            v, t = int(o["var"]), int(o["target"])
            if t not in (0, 1):
                raise SchemaError("output target must be 0 or 1")
            if v not in seen:
                raise SchemaError(f"output x{v} has no gate")
            if v in po:
                raise SchemaError(f"duplicate output x{v}")
            po.add(v)
            out_var.append(v)
            out_tgt.append(t)
    except (KeyError, TypeError) as e:
        raise SchemaError(f"bad circuit json: {e}") from None
    return Circuit(num_vars, kind, a, b, var, np.asarray(inputs, np.int32),
                   np.asarray(out_var, np.int32), np.asarray(out_tgt, np.uint8))


def export_json(c: Circuit) -> str:
    """circuit.cpp:179-210 (same keys; serialised compactly)."""
    gates = []
    for i in range(c.n_nodes):
        k = int(c.kind[i])
        args = [int(c.a[i])] if _OPERANDS[k] >= 1 else []
        if _OPERANDS[k] == 2:
            args.append(int(c.b[i]))
        gates.append({"args": args, "id": i, "kind": KINDS[k],
                      "var": int(c.var[i]) if c.var[i] else None})
    j = {"aux_base": c.num_vars, "gates": gates, "inputs": [int(v) for v in c.inputs],
         "num_vars": c.num_vars,
         "outputs": [{"target": int(t), "var": int(v)} for v, t in zip(c.out_var, c.out_tgt)]}
    return json.dumps(j) + "\n"


@dataclass
class Instance:
    """CNF + extracted circuit + path classification (what run() takes)."""
    name: str
    cnf: CnfFormula
    circuit: Circuit
    paths: PathClassification
    unsat: bool = False
    unsat_note: str = ""

    # Flat views with the attribute names the C-ABI descriptor needs.
    @property
    def num_vars(self): return self.cnf.num_vars
    @property
    def n_nodes(self): return self.circuit.n_nodes
    @property
    def kind(self): return self.circuit.kind
    @property
    def a(self): return self.circuit.a
    @property
    def b(self): return self.circuit.b
    @property
    def var(self): return self.circuit.var
    @property
    def max_var(self): return self.circuit.max_var
    @property
    def node_of_var(self): return self.circuit.node_of_var
    @property
    def n_out(self): return len(self.circuit.out_var)
    @property
    def out_var(self): return self.circuit.out_var
    @property
    def out_tgt(self): return self.circuit.out_tgt
    @property
    def out_node(self): return self.circuit.out_node
    @property
    def cpi(self): return self.paths.constrained_pi
    @property
    def ucpi(self): return self.paths.unconstrained_pi
    @property
    def n_clauses(self): return self.cnf.n_clauses
    @property
    def clause_ptr(self): return self.cnf.clause_ptr
    @property
    def clause_lit(self): return self.cnf.clause_lit


DATA_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "data",
                        "instances")


def _read(path: str) -> str:
    if path.endswith(".gz"):
        with gzip.open(path, "rt") as f:
            return f.read()
    with open(path) as f:
        return f.read()


def load_instance(name_or_cnf: str, circuit_json: str | None = None) -> Instance:
    """Load ``data/instances/<name>.cnf.gz`` + ``<name>.circuit.json.gz``, or an
    explicit DIMACS path plus its reference circuit JSON cache."""
    if circuit_json is None:
        base = os.path.join(DATA_DIR, name_or_cnf)
        cnf_path, json_path = base + ".cnf.gz", base + ".circuit.json.gz"
        name = name_or_cnf
    else:
        cnf_path, json_path = name_or_cnf, circuit_json
        name = os.path.basename(name_or_cnf)
    cnf = parse_dimacs(_read(cnf_path))
    text = _read(json_path)
    meta = json.loads(text).get("satgrad_b200", {})
    circuit = import_json(text)
    return Instance(name, cnf, circuit, classify_paths(circuit), bool(meta.get("unsat", False)),
                    meta.get("unsat_note", ""))
