# quick parity probe of the strand family against the oracle (run on the GPU box from the repo root)
import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_1004_0024_b200 as ib
from helpers import assert_batch_matches, ins, oracle_batch, product_model
from oracle import pyoracle
pyoracle.build(ref=False)
port = pyoracle.Port()
def run(csrs, n_ladders, betas, sweeps, swap, tau=1.0, exp=2, chunks=None):
    betas = np.atleast_1d(np.asarray(betas, np.float32))
    chains = n_ladders * betas.size
    seeds = (ins.CHAIN_SEED_BASE + np.arange(chains)).astype(np.uint32)
    swap_seeds = (ins.SWAP_SEED_BASE + np.arange(n_ladders)).astype(np.uint32)
    want = oracle_batch(port, csrs, n_ladders, betas, seeds, swap_seeds, sweeps, swap, tau, exp, None, None)
    st = ib.init_state([product_model(c) for c in csrs], betas, n_ladders, seeds=seeds, swap_seeds=swap_seeds,
                       params=ib.SweepParams(tau, exp), kernel=ib.KERNEL_STRAND)
    for part in (chunks or [sweeps]):
        st.run(part, swap)
    print(st.info())
    assert_batch_matches(st, want, 1e-5)
    st.close()
csr = ins.build_layered_csr(*ins.layered_spec(32, ins.INSTANCE_SEED), 8, 1.5)
run([csr], 4, ins.geometric_betas(0.2, 5.0, 16), 1, 0)
print("1 sweep ok")
run([csr], 4, ins.geometric_betas(0.2, 5.0, 16), 40, 10)
print("40 sweeps ok")
csr = ins.build_layered_csr(*ins.layered_spec(40, 8), 5, 1.5)
run([csr], 45, ins.geometric_betas(0.3, 3.0, 3), 24, 4, chunks=[3, 9, 12])
print("ragged ok")
