"""One launch of the coalesced kernel (148 chains of the C4 instance, 10 sweeps) for ncu."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, paper_1004_0024_b200 as ib
from paper_1004_0024_b200 import workloads, instances as ins
wl = workloads.get("c4")
c = wl.make_csrs()[0]
m = ib.SpinModel.from_csr(c["n_spins"], c["h"], c["offsets"], c["targets"], c["couplings"], c["tau_counts"], c["layers"], c["per_layer"])
st = ib.init_coalesced(m, np.resize(ins.geometric_betas(0.2, 5.0, 32), 148), base_seed=1000)
st.run(3)
st.run(10)
print(st.info())
