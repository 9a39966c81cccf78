import os, sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_1004_0024_b200 as ib
from helpers import ins, product_model
from oracle import pyoracle
pyoracle.build(ref=False)
port = pyoracle.Port()
P, h, edges = ins.layered_spec(32, ins.INSTANCE_SEED)
ed = [e for e in edges if abs(e[0] - e[1]) <= 2]
csr = ins.build_layered_csr(P, h, ed, 8, 1.5)
os.environ["ISING_B200_STRANDS"] = "1"
st = ib.init_state([product_model(csr)], np.asarray([0.7], np.float32), 1, seeds=np.asarray([1234], np.uint32), kernel=ib.KERNEL_STRAND)
h0, ht0 = st.fields(0)
st.run(1, 0)
st.sync()
ch = port.chain(port.model(csr), 1234, 0.7, 1.0, 2)
raw = port.mt_fill(1234, 16) if hasattr(port, "mt_fill") else None
print("raw", [hex(int(x)) for x in raw] if raw is not None else None)
print("oracle h0[:16]", ch.hs[:16], "ht", ch.ht[:16], "s0", ch.spins[:16])
ch.sweep(1)
print("oracle s1", ch.spins[:16])
