"""One-off soak: the full c5 workload (16,384 chains x 32,768 spins, swap every 10) for 1,000 sweeps
through BOTH kernel families; every chain's checksum, flip count, slot and running energy must agree.
Run on a B200: python profiles/soak_c5.py [sweeps]"""
import sys, pathlib, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, paper_1004_0024_b200 as ib
from paper_1004_0024_b200 import workloads, instances as ins

sweeps = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
wl = workloads.get("c5")
c = wl.make_csrs()[0]
model = ib.SpinModel.from_csr(c["n_spins"], c["h"], c["offsets"], c["targets"], c["couplings"], c["tau_counts"],
                              c["layers"], c["per_layer"])
out = {}
for family in (ib.KERNEL_LAYERED, ib.KERNEL_GENERIC):
    t0 = time.perf_counter()
    with ib.init_state(model, wl.betas, wl.n_ladders, base_seed=ins.CHAIN_SEED_BASE, swap_base_seed=ins.SWAP_SEED_BASE,
                       kernel=family) as st:
        st.run(sweeps, wl.swap_interval)
        out[family] = (st.checksums(), st.stats()[0], st.slots(), st.running_energies().view(np.uint64),
                       st.swap_stats()[0])
    print(f"family {family}: {sweeps} sweeps in {time.perf_counter() - t0:.1f} s", flush=True)
for a, b in zip(out[ib.KERNEL_LAYERED], out[ib.KERNEL_GENERIC]):
    np.testing.assert_array_equal(a, b)
print("soak ok: checksums, flips, slots, running energies and swap counts of all",
      out[ib.KERNEL_LAYERED][0].size, "chains agree; checksum of checksums",
      hex(int(np.bitwise_xor.reduce(out[ib.KERNEL_LAYERED][0]))))
