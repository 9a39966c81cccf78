import os, sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_1004_0024_b200 as ib
from helpers import ins, product_model
from oracle import pyoracle
pyoracle.build(ref=False)
port = pyoracle.Port()
P, h, edges = ins.layered_spec(32, ins.INSTANCE_SEED)
variants = {
    "path (band only)": [e for e in edges if abs(e[0] - e[1]) <= 2],
    "ring (+wrap far)": [e for e in edges if abs(e[0] - e[1]) <= 2 or abs(e[0] - e[1]) >= P - 2],
    "band + far>=16": [e for e in edges if abs(e[0] - e[1]) <= 2 or abs(e[0] - e[1]) >= 16],
    "full": edges,
}
betas = np.asarray([0.7], np.float32)
seeds = np.asarray([1234], np.uint32)
os.environ["ISING_B200_STRANDS"] = "1"
for name, ed in variants.items():
    csr = ins.build_layered_csr(P, h, ed, 8, 1.5)
    for sweeps in (1, 3):
        st = ib.init_state([product_model(csr)], betas, 1, seeds=seeds, kernel=ib.KERNEL_STRAND)
        st.run(sweeps, 0)
        spins = st.spins()[0]
        ch = port.chain(port.model(csr), 1234, 0.7, 1.0, 2)
        ch.sweep(sweeps)
        bad = np.nonzero(spins != ch.spins.astype(np.int8))[0]
        print(name, "sweeps", sweeps, "bad spins", bad[:10], bad.size)
        st.close()
