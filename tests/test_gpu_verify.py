"""Device-side `satgrad verify` (sgx_verify_solutions) against the reference's
checks (cmd_verify, tools/satgrad_main.cpp:242-302, restated over the
reference's eval_cnf / SolutionSet in oracle/ref_shim.cpp::ref_verify_text):
the same verdict, error line, error kind, variable and count of verified
solutions, on sampled solution texts and on every error the command reports.
"""
import numpy as np
import pytest

from oracle.oracle import RefInstance, ref_available
from paper_2502_08673_b200 import (DeviceCircuit, RestartPolicy, Sampler, SamplerConfig, load_instance,
                                   write_dimacs)

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")]

_CACHE = {}


def _setup(name, batch):
    if name not in _CACHE:
        inst = load_instance(name)
        dc = DeviceCircuit.from_instance(inst)
        s = Sampler(dc, SamplerConfig(batch=batch, iterations=5, seed=7,
                                      restart=RestartPolicy.REINIT_ON_EXHAUST, max_restarts=2))
        s.run()
        text = s.format_solutions().decode()
        s.close()
        _CACHE[name] = (inst, dc, RefInstance.from_dimacs(write_dimacs(inst.cnf)), text)
    return _CACHE[name]


def _same(dc, ref, text):
    got = dc.verify_solutions(text)
    want = ref.verify_text(text)
    assert (got["checked"], got["line"], got["kind"], got["var"]) == \
        (want["checked"], want["line"], want["kind"], want["var"]), (got, want)
    return got


def _mutations(lines, nv, rng):
    """Every cmd_verify error, plus the line shapes its tokenizer accepts."""
    n = len(lines)
    k = int(rng.integers(0, n))
    toks = lines[k].split()
    out = {"valid": lines}
    out["blank_and_garbage"] = lines[:k] + ["", "   ", "abc", "\t"] + lines[k:]
    out["crlf"] = [ln + "\r" for ln in lines]
    j = int(rng.integers(0, n))
    out["duplicate"] = lines[: j + 1] + [lines[min(j, k)]] + lines[j + 1:]
    flip = toks.copy()
    i = int(rng.integers(0, len(flip) - 1))
    flip[i] = str(-int(flip[i]))
    out["flipped_literal"] = lines[:k] + [" ".join(flip)] + lines[k + 1:]
    out["no_terminator"] = lines[:k] + [" ".join(toks[:-1])] + lines[k + 1:]
    out["exceeds"] = lines[:k] + [" ".join(toks[:-1] + [str(nv + 1), "0"])] + lines[k + 1:]
    both = toks[:-1] + [str(-int(toks[0])), "0"]
    out["both_ways"] = lines[:k] + [" ".join(both)] + lines[k + 1:]
    drop = toks[:i] + toks[i + 1:]
    out["unassigned"] = lines[:k] + [" ".join(drop)] + lines[k + 1:]
    plus = [("+" + t if not t.startswith("-") and t != "0" else t) for t in toks]
    out["plus_signs"] = lines[:k] + [" ".join(plus)] + lines[k + 1:]
    out["trailing_junk"] = lines[:k] + [" ".join(toks[:-1]) + " 0abc"] + lines[k + 1:]
    out["token_junk"] = lines[:k] + [" ".join(toks[:1]) + "x " + " ".join(toks[1:])] + lines[k + 1:]
    out["overflow"] = lines[:k] + [" ".join(toks[:-1] + ["99999999999999999999", "0"])] + lines[k + 1:]
    out["overflow_first"] = lines[:k] + ["99999999999999999999 " + lines[k]] + lines[k + 1:]
    out["repeat_literal"] = lines[:k] + [" ".join(toks[:1] + toks)] + lines[k + 1:]
    return out


@pytest.mark.parametrize("name,batch", [("c3a_or50", 4096), ("c1b_random", 2048), ("mux_chain14", 1024),
                                        ("c2_iscas", 256)])
def test_verify_matches_reference(gpu, name, batch):
    inst, dc, ref, text = _setup(name, batch)
    lines = text.rstrip("\n").split("\n")
    assert len(lines) > 1
    got = _same(dc, ref, text)
    assert got["ok"] and got["checked"] == len(lines)
    assert _same(dc, ref, text.rstrip("\n"))["ok"]  # no final newline
    rng = np.random.default_rng(len(lines))
    for trial in range(3):
        for what, ls in _mutations(lines, inst.cnf.num_vars, rng).items():
            _same(dc, ref, "\n".join(ls) + "\n")


def test_verify_empty_and_blank(gpu):
    inst, dc, ref, _ = _setup("mux_chain14", 1024)
    for t in ["", "\n", "\n\n  \n", "0\n"]:
        _same(dc, ref, t)


def test_verify_large_text_chunks(gpu):
    """A text above the one-chunk size (parsed on several host threads, checked
    in several device chunks): identical to the reference, errors late in the
    text included."""
    inst, dc, ref, text = _setup("c3a_or50", 4096)
    lines = text.rstrip("\n").split("\n")
    big = lines * max(1, (3 << 20) // max(1, len(text)) + 1)
    # distinct lines only up to the first repeat: the duplicate error lands at len(lines) + 1
    _same(dc, ref, "\n".join(big) + "\n")
    _same(dc, ref, "\n".join(lines) + "\n")


def test_verify_from_cnf_alone(gpu):
    """sgx_verify_cnf (the entry point for cmd_verify, which has no circuit)
    equals the circuit-bound call, error cases included."""
    from paper_2502_08673_b200 import verify_solutions
    inst, dc, ref, text = _setup("c1b_random", 2048)
    lines = text.rstrip("\n").split("\n")
    rng = np.random.default_rng(3)
    for what, ls in _mutations(lines, inst.cnf.num_vars, rng).items():
        t = "\n".join(ls) + "\n"
        a, b = verify_solutions(inst.cnf, t), dc.verify_solutions(t)
        assert (a["checked"], a["line"], a["kind"], a["var"]) == (b["checked"], b["line"], b["kind"], b["var"])


def test_full_size_format_verify_round_trip(gpu):
    """BASELINE's headline configuration (C2, B = 65,536, 5 iterations): every
    stored solution, rendered as the reference's text on the device, passes
    the device verify -- satisfying, complete, pairwise distinct -- and the
    count verified is the run's unique count (a size-independent property)."""
    from paper_2502_08673_b200 import verify_solutions
    inst = load_instance("c2_iscas")
    dc = DeviceCircuit.from_instance(inst)
    s = Sampler(dc, SamplerConfig(batch=65536, iterations=5, seed=1))
    try:
        st = s.run()
        text = s.format_solutions()
        v = verify_solutions(inst.cnf, text)
        assert v["ok"] and v["checked"] == st.unique_count > 10000, v
        # the last line repeated is reported one line past the end, like the reference
        last = text[text.rstrip(b"\n").rfind(b"\n") + 1:]
        v2 = dc.verify_solutions(text + last)
        assert v2["kind"] == 6 and v2["line"] == st.unique_count + 1 and v2["checked"] == st.unique_count
    finally:
        s.close()
        dc.close()
