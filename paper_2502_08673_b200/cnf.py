"""DIMACS CNF I/O and the host-side clause checker.

Mirrors include/satgrad/cnf.hpp (reference): ``parse_dimacs`` follows
cnf.cpp:18-107 (duplicate literals dropped keeping first occurrences, clauses
may span lines, header/count mismatch is a warning, ``ParseError`` otherwise),
``write_dimacs`` follows cnf.cpp:109-127, and ``eval_cnf`` follows
cnf.cpp:129-147.  The clause list is held as CSR (``clause_ptr`` /
``clause_lit`` of signed DIMACS literals), the layout the C-ABI takes.

``verify_keys`` is the host re-verifier for solutions fetched from the device:
it evaluates every clause on packed dedupe keys (sampler.cpp:18-26 layout),
vectorised over solutions with numpy.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


class ParseError(ValueError):
    """cnf.hpp:40-43."""


@dataclass
class CnfFormula:
    num_vars: int = 0
    clause_ptr: np.ndarray = field(default_factory=lambda: np.zeros(1, np.int64))
    clause_lit: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    comments: list = field(default_factory=list)

    @property
    def n_clauses(self) -> int:
        return len(self.clause_ptr) - 1

    def clauses(self):
        for c in range(self.n_clauses):
            yield [int(x) for x in self.clause_lit[self.clause_ptr[c]:self.clause_ptr[c + 1]]]

    @classmethod
    def from_clauses(cls, num_vars: int, clauses, comments=()) -> "CnfFormula":
        ptr = [0]
        lits = []
        for cl in clauses:
            lits.extend(int(x) for x in cl)
            ptr.append(len(lits))
        return cls(num_vars, np.asarray(ptr, np.int64), np.asarray(lits, np.int32), list(comments))


def parse_dimacs(text: str, warnings: list | None = None) -> CnfFormula:
    """cnf.cpp:18-107."""
    comments: list[str] = []
    num_vars = 0
    declared = 0
    saw_header = False
    ptr = [0]
    lits: list[int] = []
    current: list[int] = []
    open_clause = False
    for line_no, line in enumerate(text.split("\n"), start=1):
        s = line.strip(" \t\r\v\f")
        if not s:
            continue
        if s[0] == "c" and (len(s) == 1 or s[1] in " \t\r\v\f"):
            body = line[line.index("c") + 1:]
            comments.append(body[1:] if body.startswith(" ") else body)
            continue
        if s[0] == "p":
            if saw_header:
                raise ParseError(f"line {line_no}: duplicate header")
            if open_clause:
                raise ParseError(f"line {line_no}: header inside a clause")
            parts = s.split()
            try:
                if len(parts) < 4 or parts[0] != "p" or parts[1] != "cnf":
                    raise ValueError
                num_vars, declared = int(parts[2]), int(parts[3])
                if num_vars < 0 or declared < 0:
                    raise ValueError
            except ValueError:
                raise ParseError(f"line {line_no}: malformed header") from None
            saw_header = True
            continue
        for tok in s.split():
            try:
                value = int(tok)
            except ValueError:
                raise ParseError(f"line {line_no}: unexpected token '{tok[0]}'") from None
            if not saw_header:
                raise ParseError(f"line {line_no}: clause data before header")
            if value == 0:
                if not current:
                    raise ParseError(f"line {line_no}: empty clause")
                seen = set()
                for l in current:  # keep first occurrences (cnf.cpp:37-42)
                    if l not in seen:
                        seen.add(l)
                        lits.append(l)
                ptr.append(len(lits))
                current = []
                open_clause = False
            else:
                if abs(value) > num_vars:
                    raise ParseError(f"line {line_no}: literal {value} exceeds declared "
                                     f"{num_vars} variables")
                current.append(value)
                open_clause = True
    if open_clause:
        raise ParseError("clause not 0-terminated at end of input")
    if not saw_header:
        raise ParseError("missing 'p cnf' header")
    n = len(ptr) - 1
    if n != declared and warnings is not None:
        warnings.append(f"header declares {declared} clauses, found {n}")
    return CnfFormula(num_vars, np.asarray(ptr, np.int64), np.asarray(lits, np.int32), comments)


def write_dimacs(cnf: CnfFormula) -> str:
    """cnf.cpp:109-127."""
    out = [f"c {c}" for c in cnf.comments]
    out.append(f"p cnf {cnf.num_vars} {cnf.n_clauses}")
    for cl in cnf.clauses():
        out.append(" ".join(str(x) for x in cl) + " 0")
    return "\n".join(out) + "\n"


def eval_cnf(cnf: CnfFormula, assignment) -> bool:
    """cnf.cpp:129-147 on an Assignment indexed by var (slot 0 unused)."""
    a = np.asarray(assignment)
    for cl in cnf.clauses():
        sat = False
        for l in cl:
            v = abs(l)
            if v >= len(a) or a[v] > 1:
                raise ValueError(f"variable {v} is unassigned")
            if (a[v] != 0) != (l < 0):
                sat = True
                break
        if not sat:
            return False
    return True


def verify_keys(cnf: CnfFormula, keys: np.ndarray) -> np.ndarray:
    """eval_cnf for every packed key row at once: bool[n]."""
    keys = np.asarray(keys, np.uint64)
    n = keys.shape[0]
    out = np.zeros(n, bool)
    if n == 0:
        return out
    lits = cnf.clause_lit.astype(np.int64)
    v = np.abs(lits) - 1
    word, shift, neg = v // 64, (v % 64).astype(np.uint64), (lits < 0)[None, :]
    step = max(1, 20_000_000 // max(1, len(lits)))
    for r0 in range(0, n, step):
        k = keys[r0:r0 + step]
        bits = (k[:, word] >> shift) & np.uint64(1)  # [rows, n_lits]
        lit_true = bits.astype(bool) != neg
        # OR within each clause via a cumulative count over the CSR.
        csum = np.concatenate([np.zeros((len(k), 1), np.int64), np.cumsum(lit_true, axis=1)], axis=1)
        per_clause = csum[:, cnf.clause_ptr[1:]] - csum[:, cnf.clause_ptr[:-1]]
        out[r0:r0 + step] = (per_clause > 0).all(axis=1)
    return out


def key_to_assignment(key: np.ndarray, num_vars: int) -> np.ndarray:
    """SolutionSet::assignment (sampler.cpp:46-52): uint8[num_vars + 1]."""
    a = np.full(num_vars + 1, 0xFF, np.uint8)
    v = np.arange(1, num_vars + 1)
    a[1:] = (np.asarray(key, np.uint64)[(v - 1) // 64] >> ((v - 1) % 64).astype(np.uint64)) & 1
    return a


def format_solution_line(key: np.ndarray, num_vars: int) -> str:
    """format_solution_line (sampler.cpp:66-76)."""
    a = key_to_assignment(key, num_vars)
    return " ".join(str(v) if a[v] else str(-v) for v in range(1, num_vars + 1)) + (" 0" if num_vars else "0")
