# which spins differ first on the 64x4 chord graph (strand family vs oracle)
import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_1004_0024_b200 as ib
from helpers import ins, oracle_batch, product_model
from test_gpu_parity import chord_spec
from oracle import pyoracle
pyoracle.build(ref=False)
port = pyoracle.Port()
csr = ins.build_layered_csr(*chord_spec(64, 164, (3, 5, 6, 9, 13, 17, 26, 31)), 4, 0.8)
betas = ins.geometric_betas(0.25, 2.0, 5)
ladders = int(sys.argv[1]) if len(sys.argv) > 1 else 9
chains = ladders * 5
seeds = (ins.CHAIN_SEED_BASE + np.arange(chains)).astype(np.uint32)
swap_seeds = (ins.SWAP_SEED_BASE + np.arange(ladders)).astype(np.uint32)
for sweeps in (1, 2, 3):
    want = oracle_batch(port, [csr], ladders, betas, seeds, swap_seeds, sweeps, 0, 1.25, 2, None, None)
    st = ib.init_state([product_model(csr)], betas, ladders, seeds=seeds, swap_seeds=swap_seeds,
                       params=ib.SweepParams(1.25, 2), kernel=ib.KERNEL_STRAND)
    st.run(sweeps, 0)
    got = st.spins(0, chains)
    ws = want["spins"] if isinstance(want, dict) else want.spins
    bad = np.argwhere(got != ws)
    print("sweeps", sweeps, "info", {k: st.info()[k] for k in ("strands", "kernel")}, "mismatches", len(bad))
    if len(bad):
        print(bad[:20].tolist())
        ch = bad[0][0]
        print("chain", ch, "bad spins", [int(b[1]) for b in bad if b[0] == ch][:40])
        break
    st.close()
