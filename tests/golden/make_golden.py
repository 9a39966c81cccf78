"""Generates tests/golden/*.npz by running the UNMODIFIED reference (oracle/_ref/libisingref.so,
built from /root/reference by oracle/Makefile).  Run in the build container only:

    python tests/golden/make_golden.py

Each file stores the inputs (CSR arrays, seeds, parameters) next to the reference's outputs so
that the fixtures do not depend on regenerating the instance bit-for-bit elsewhere.
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import pyoracle as po  # noqa: E402
from paper_1004_0024_b200 import instances as ins  # noqa: E402

OUT = Path(__file__).resolve().parent


def primitives(ref):
    seeds = np.array([1, 5489, 123456789, 987654321, 42], np.uint32)
    # first outputs, the 624-block boundary and a late window of every stream
    windows = [(0, 8), (620, 632), (3 * 624, 3 * 624 + 8), (999_990, 1_000_000)]
    streams = {int(s): ref.mt_fill(int(s), 1_000_000) for s in seeds}
    mt = np.stack([np.concatenate([streams[int(s)][a:b] for a, b in windows]) for s in seeds])
    plain = ref.mt_next_stream(5489, 2000)
    assert (plain == streams[5489][:2000]).all()
    xor_fold = np.array([np.bitwise_xor.reduce(streams[int(s)]) for s in seeds], np.uint32)

    rng = np.random.default_rng(2024)
    raw = np.concatenate([
        np.array([0, 1, 2, 3, 2**23, 2**24 - 1, 2**24, 2**24 + 1, 2**25 + 3, 2**31 - 1, 2**31, 2**31 + 129,
                  2**32 - 257, 2**32 - 256, 2**32 - 129, 2**32 - 1], np.uint64),
        rng.integers(0, 2**32, 4000, dtype=np.uint64)]).astype(np.uint32)
    unit = np.array([ref.u32_to_unit(int(x)) for x in raw], np.float32)

    xs = np.concatenate([
        np.array([0.0, -0.0, np.log(2.0), -np.log(2.0), 1.0, -1.0, -21.834136, -21.834137, -21.9, -87.0, -87.4,
                  -90.0, -200.0, 22.0, 88.0, 88.8, 100.0, 1e-30, -1e-30, 1e-6, -1e-6], np.float64),
        rng.uniform(-30.0, 5.0, 3000), rng.uniform(-120.0, 120.0, 1000)]).astype(np.float32)
    exps = np.stack([np.array([ref.exp(k, float(x)) for x in xs], np.float32) for k in (1, 2, 3)])
    init = np.stack([ref.initial_spins(700, int(s)) for s in seeds])
    np.savez_compressed(OUT / "primitives.npz", seeds=seeds, mt_windows=np.array(windows), mt=mt,
                        mt_xor_fold=xor_fold, unit_in=raw, unit_out=unit, exp_in=xs, exp_out=exps,
                        initial_spins=init)


def run_case(ref, csr, seed, beta, tau_scale, kind, sweeps, initial=None):
    model = ref.model(csr)
    assert model.validate() is None, model.validate()
    chain = ref.chain(model, seed, beta, tau_scale, kind, initial)
    spins0 = chain.spins.copy()
    hs0, ht0 = chain.hs.copy(), chain.ht.copy()
    half = sweeps // 2
    chain.sweep(half)
    mid = chain.spins.copy()
    chain.sweep(sweeps - half)
    s = chain.spins
    # the reference engine (legacy graph, plain twist) must land on the same state
    twin = ref.chain(model, seed, beta, tau_scale, kind, initial, engine=0)
    twin.sweep(sweeps)
    assert (twin.spins == s).all() and twin.flips == chain.flips
    return dict(spins0=spins0.astype(np.int8), hs0=hs0, ht0=ht0, spins_mid=mid.astype(np.int8),
                spins=s.astype(np.int8), hs=chain.hs, ht=chain.ht, flips=np.uint64(chain.flips),
                attempts=np.uint64(chain.attempts), cost=np.float64(ref.total_cost(model, s)),
                checksum=np.uint64(ref.checksum(s)), coherence=np.uint64(chain.coherence()))


def trajectories(ref):
    cases = {
        "cubic4_pm1": (ins.cubic_pm1(4, 101, 0.0), 1.0, 1.0),
        "cubic6_gauss_h": (ins.cubic_pm1(6, 102, 0.5), 1.0, 1.0),
        "mixed6": (ins.cubic_mixed_degree(6, 103), 0.8, 1.0),
        "layered_24x8": (ins.build_layered_csr(*ins.layered_spec(24, 104), 8, 1.5), 0.6, 1.0),
        "layered_16x4_gamma": (ins.build_layered_csr(*ins.layered_spec(16, 105), 4, 0.75), 0.9, 0.5),
    }
    for name, (csr, beta, gamma) in cases.items():
        out = {f"csr_{k}": v for k, v in csr.items() if v is not None}
        meta = []
        for kind in (1, 2, 3):
            for seed in (7, 1234567):
                res = run_case(ref, csr, seed, beta, gamma, kind, 300)
                tag = f"k{kind}_s{seed}"
                meta.append((kind, seed))
                for k, v in res.items():
                    out[f"{tag}_{k}"] = v
        out["beta"], out["tau_scale"], out["sweeps"] = np.float32(beta), np.float32(gamma), np.int64(300)
        out["runs"] = np.array(meta, np.int64)
        np.savez_compressed(OUT / f"traj_{name}.npz", **out)

    # the reference's own hand traces (tests/test_sweep.cpp:122-145): explicit initial spins
    two = dict(n_spins=2, h=np.zeros(2, np.float32), offsets=np.array([0, 1, 2], np.uint32),
               targets=np.array([1, 0], np.uint32), couplings=np.ones(2, np.float32), tau_counts=None)
    res = run_case(ref, two, 1, 0.0, 1.0, 1, 2, initial=np.array([1, -1], np.int8))
    assert res["spins"].tolist() == [1, -1] and int(res["flips"]) == 4
    np.savez_compressed(OUT / "traj_two_spin.npz", **{k: v for k, v in res.items()})


def layered_builder(ref):
    positions, h, edges = ins.layered_spec(12, 55)
    model = ref.build_layered(positions, h, edges, 5, 1.5)
    csr = model.csr()
    np.savez_compressed(OUT / "layered_builder.npz", positions=np.int64(positions), h=h,
                        edges=np.array([(p, q) for p, q, _ in edges], np.uint32),
                        edge_j=np.array([c for _, _, c in edges], np.float32), n_layers=np.int64(5),
                        j_tau=np.float32(1.5), **{f"csr_{k}": v for k, v in csr.items()})


def model_documents(ref):
    """`ising-model v1` documents written by the reference's model_to_string (tests/test_model_text.py)."""
    sys.path.insert(0, str(OUT.parent))
    from test_model_text import sample_csrs
    for name, csr in sample_csrs().items():
        (OUT / f"model_{name}.txt").write_text(ref.model(csr).to_string())


if __name__ == "__main__":
    po.build()
    reference = po.Reference()
    if "--documents-only" not in sys.argv:
        primitives(reference)
        trajectories(reference)
        layered_builder(reference)
    model_documents(reference)
    print("golden vectors written to", OUT)
