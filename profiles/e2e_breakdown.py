"""Where the fixed cost of the end-to-end path goes (c5): model build, batch creation (graph analysis,
allocation, device init_state), stepping with per-step readouts, final readouts.  Run on a B200."""
import sys, pathlib, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, paper_1004_0024_b200 as ib
from paper_1004_0024_b200 import workloads, instances as ins

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
wl = workloads.get(name)
csrs = wl.make_csrs()
for rep in range(2):
    t = [time.perf_counter()]
    model = [ib.SpinModel.from_csr(c["n_spins"], c["h"], c["offsets"], c["targets"], c["couplings"], c["tau_counts"],
                                   c["layers"], c["per_layer"]) for c in csrs]
    model = model[0] if len(model) == 1 else model
    t.append(time.perf_counter())
    st = ib.init_state(model, wl.betas, wl.n_ladders, base_seed=ins.CHAIN_SEED_BASE, swap_base_seed=ins.SWAP_SEED_BASE)
    t.append(time.perf_counter())
    st.sync()
    t.append(time.perf_counter())
    for _ in range(20):
        st.run(10, 10)
        st.stats(); st.running_energies()
    t.append(time.perf_counter())
    en = st.energies()
    t.append(time.perf_counter())
    cs = st.checksums(); sp = st.spins(0, 16)
    t.append(time.perf_counter())
    st.close()
    t.append(time.perf_counter())
    names = ["model", "init_state (enqueue)", "init_state (device)", "20 steps + readouts", "energies", "checksums+spins", "close"]
    print(f"pass {rep}: " + ", ".join(f"{n} {1e3*(b-a):.1f} ms" for n, a, b in zip(names, t, t[1:])))
