"""Fuzz native extraction against the live reference: python tools/extract_fuzz.py FIRST LAST (seeds)."""
import sys; R=__import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))); sys.path.insert(0,R); sys.path.insert(0,R+'/tests')
import numpy as np
from test_extract import _random_cnf, _same
from oracle.oracle import RefInstance
from paper_2502_08673_b200 import extract_circuit, parse_dimacs, write_dimacs, CnfFormula
bad=0
import time
t0=time.time()
for seed in range(int(sys.argv[1]), int(sys.argv[2])):
    rng=np.random.default_rng(10000+seed)
    nv=int(rng.integers(3, 120 if seed%3 else 25))
    if seed % 5 == 0:
        # wide clauses / long residues to hit the 12 / 16 caps
        nv=min(nv,30); cls=[[int(v)*int(rng.choice([-1,1])) for v in rng.integers(1,nv+1,int(rng.integers(1,14)))] for _ in range(int(rng.integers(1,2*nv)))]
        cnf=CnfFormula.from_clauses(nv, cls)
    else:
        cnf=_random_cnf(rng,nv,int(rng.integers(1,4*nv)))
    text=write_dimacs(cnf)
    if seed%100==0: print('seed',seed,time.time()-t0,flush=True)
    ref=RefInstance.from_dimacs(text)
    r=extract_circuit(parse_dimacs(text))
    try:
        _same(r.circuit, ref); assert r.unsat==ref.unsat and r.unsat_note==ref.unsat_note
        sizes,iv,aux=ref.extraction_lists()
        assert [len(r.pi),len(r.po_var),len(r.iv),len(r.aux),r.n_defs]==sizes and np.array_equal(r.iv,iv)
    except AssertionError as e:
        bad+=1; print("seed",seed,"FAIL",e, nv)
        if bad>5: break
print("bad",bad, flush=True)
