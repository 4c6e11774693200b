import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SGX_REINIT_DEBUG"] = "1"
from paper_2502_08673_b200 import DeviceCircuit, RestartPolicy, Sampler, SamplerConfig, load_instance
dc = DeviceCircuit.from_instance(load_instance("c2_iscas"))
for pol in (RestartPolicy.REINIT_ROWS, RestartPolicy.REINIT_ON_EXHAUST):
    s = Sampler(dc, SamplerConfig(batch=8192, iterations=5, seed=1, restart=pol, max_restarts=1))
    st = s.run(); print(pol.name, st.unique_count, st.new_unique, flush=True); s.close()
