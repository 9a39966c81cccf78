import sys, time, pathlib
sys.path.insert(0, '.')
import numpy as np, paper_1004_0024_b200 as ib
from paper_1004_0024_b200 import workloads, instances as ins
wl = workloads.get("c5"); c = wl.make_csrs()[0]
model = ib.SpinModel.from_csr(c["n_spins"], c["h"], c["offsets"], c["targets"], c["couplings"], c["tau_counts"], c["layers"], c["per_layer"])
ts = []
for rep in range(8):
    t0 = time.perf_counter()
    st = ib.init_state(model, wl.betas, wl.n_ladders, base_seed=ins.CHAIN_SEED_BASE, swap_base_seed=ins.SWAP_SEED_BASE)
    st.sync()
    ts.append(1e3 * (time.perf_counter() - t0))
    st.close()
print("init_state ms:", " ".join(f"{t:.1f}" for t in ts))
