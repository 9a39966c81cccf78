"""Throughput of the coalesced (intra-system) family on the C4 instance for a few chain counts,
beside the replica-parallel families on the same few-chain problem.  Run on a B200: python profiles/coalesced_bench.py"""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import time, numpy as np, paper_1004_0024_b200 as ib
from paper_1004_0024_b200 import workloads, instances as ins
wl = workloads.get("c4")
c = wl.make_csrs()[0]
m = ib.SpinModel.from_csr(c["n_spins"], c["h"], c["offsets"], c["targets"], c["couplings"], c["tau_counts"], c["layers"], c["per_layer"])
n = c["n_spins"]
for chains in (1, 16, 148, 592, 2048):
    betas = np.resize(ins.geometric_betas(0.2, 5.0, 32), chains)
    st = ib.init_coalesced(m, betas, base_seed=1000)
    st.run(5); st.info()
    sweeps = 50
    st.run(sweeps)
    ms = st.info()["last_run_ms"]
    fl, at = st.stats()
    print(f"coalesced chains={chains:5d}  {ms:9.2f} ms for {sweeps} sweeps  -> {chains*n*sweeps/ms*1e3:.3e} attempts/s  ({ms/sweeps*1e3:.1f} us/sweep)  flip rate {fl.sum()/at.sum():.4f}")
    st.close()
# lane = chain families on the same few-chain problem
for chains in (1, 32, 148):
    betas = np.resize(ins.geometric_betas(0.2, 5.0, 32), chains)
    st = ib.init_state(m, betas[:1] if chains == 1 else [1.0], chains, base_seed=1000)
    st.run(5); st.sync(); st.set_timing(True)
    st.run(20); ms = st.info()["last_run_ms"]
    print(f"layered  chains={chains:5d}  {ms:9.2f} ms for 20 sweeps -> {chains*n*20/ms*1e3:.3e} attempts/s")
    st.close()

# the reference's own coalesced engine on one host core (oracle/_ref), same instance
try:
    from oracle import pyoracle
    if pyoracle.Reference.available():
        ref = pyoracle.Reference()
        permuted, _ = ref.model(c).prepared_for(3)
        chain = ref.chain(permuted, 1000, 1.0, 1.0, 2, None, engine=3)
        chain.sweep(2)
        t0 = time.perf_counter(); chain.sweep(20); dt = time.perf_counter() - t0
        print(f"reference coalesced engine, 1 host thread: {20*n/dt:.3e} attempts/s ({dt/20*1e6:.0f} us/sweep)")
        basic = ref.chain(ref.model(c), 1000, 1.0, 1.0, 2, None, engine=1)
        basic.sweep(2)
        t0 = time.perf_counter(); basic.sweep(20); dt = time.perf_counter() - t0
        print(f"reference basic engine,     1 host thread: {20*n/dt:.3e} attempts/s ({dt/20*1e6:.0f} us/sweep)")
except Exception as exc:  # the reference library is optional on the GPU box
    print("reference timing skipped:", exc)
