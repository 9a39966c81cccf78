"""Shared helpers for the parity tests."""
import numpy as np

import paper_1004_0024_b200 as ib
from paper_1004_0024_b200 import instances as ins


def csr_from_npz(z, prefix="csr_"):
    keys = ("n_spins", "h", "offsets", "targets", "couplings", "tau_counts", "layers", "per_layer")
    out = {k: z[prefix + k] for k in keys if prefix + k in z.files}
    out["n_spins"] = int(out["n_spins"]) if "n_spins" in out else int(len(out["h"]))
    out.setdefault("tau_counts", None)
    out["layers"] = int(out.get("layers", 0))
    out["per_layer"] = int(out.get("per_layer", 0))
    return out


def product_model(csr) -> ib.SpinModel:
    return ib.SpinModel.from_csr(csr["n_spins"], csr["h"], csr["offsets"], csr["targets"], csr["couplings"],
                                 csr.get("tau_counts"), csr.get("layers", 0) or 0, csr.get("per_layer", 0) or 0)


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def oracle_batch(port, csrs, n_ladders, betas, seeds, swap_seeds, sweeps, swap_interval, tau_scale=1.0,
                 exp_kind=2, model_of_ladder=None, initial=None, threads=4):
    """Runs the plain-C oracle on the same batch description the product gets."""
    models = [port.model(c) for c in csrs]
    if model_of_ladder is None:
        model_of_ladder = list(range(n_ladders)) if len(models) == n_ladders and n_ladders > 1 else [0] * n_ladders
    per_ladder = [models[i] for i in model_of_ladder]
    return port.pt_run(per_ladder, n_ladders, betas, seeds, swap_seeds, sweeps, swap_interval, tau_scale,
                       exp_kind, threads, initial)


def assert_batch_matches(state, want, rel_energy=1e-5):
    """Bit-exact spins / flips / slots / running energies; energies within rel_energy."""
    got_spins = state.spins()
    assert got_spins.shape == want["spins"].shape
    bad = np.argwhere(got_spins != want["spins"])
    assert bad.size == 0, f"first spin mismatch at (chain, spin) = {bad[0].tolist()}"
    flips, attempts = state.stats()
    assert (flips == want["flips"]).all()
    np.testing.assert_array_equal(state.slots(), want["slot"])
    np.testing.assert_array_equal(state.running_energies().view(np.uint64), want["e_run"].view(np.uint64))
    e = state.energies()
    np.testing.assert_allclose(e, want["energy"], rtol=rel_energy, atol=1e-9)
    acc, att = state.swap_stats()
    nb = acc.shape[1]
    if nb > 1:
        np.testing.assert_array_equal(acc[:, : nb - 1], want["swap_acc"][:, : nb - 1])
        np.testing.assert_array_equal(att[:, : nb - 1], want["swap_att"][:, : nb - 1])
    return e


def random_graph(n, mean_degree, seed, repeats=0):
    """A seeded random multigraph: `mean_degree * n / 2` distinct edges plus `repeats` repeated ones,
    Gaussian couplings and fields (tests only: degrees well beyond eight, a ragged last chunk)."""
    rng = np.random.default_rng(seed)
    pairs = set()
    while len(pairs) < mean_degree * n // 2:
        a, b = (int(v) for v in rng.integers(0, n, 2))
        if a != b:
            pairs.add((min(a, b), max(a, b)))
    edges = sorted(pairs)
    edges += [edges[int(k)] for k in rng.integers(0, len(edges), repeats)]
    coup = rng.normal(0.0, 1.0, len(edges)).astype(np.float32)
    h = rng.normal(0.0, 0.3, n).astype(np.float32)
    return ins.csr_from_adjacency(h, ins._adjacency(n, np.array(edges, np.int64), coup))


# ---- a 12-spin model small enough to enumerate (statistical validation of the tempering sampler)
SMALL_N = 12
N = SMALL_N


def small_model(seed):
    """12 spins, ~degree 4, Gaussian couplings and fields (f32 values, exact in f64)."""
    rng = ins.MT19937(seed)
    edges = {}
    for i in range(N):
        edges[(i, (i + 1) % N)] = 0.0
    while len(edges) < 24:
        a, b = rng.below(N), rng.below(N)
        if a != b:
            edges.setdefault((min(a, b), max(a, b)), 0.0)
    js = rng.normals(len(edges), 0.8)
    h = rng.normals(N, 0.4).astype(np.float32)
    pairs = [(a, b, np.float32(j)) for (a, b), j in zip(sorted(edges), js)]
    adj = [[] for _ in range(N)]
    for a, b, j in pairs:
        adj[a].append((b, j))
        adj[b].append((a, j))
    offsets, targets, couplings = [0], [], []
    for i in range(N):
        for t, j in sorted(adj[i]):
            targets.append(t)
            couplings.append(j)
        offsets.append(len(targets))
    csr = dict(n_spins=N, h=h, offsets=np.array(offsets, np.uint32), targets=np.array(targets, np.uint32),
               couplings=np.array(couplings, np.float32), tau_counts=np.zeros(N, np.uint8), layers=0, per_layer=0)
    return csr, pairs, h


def enumerate_energies(pairs, h):
    """E(s) = -sum h_i s_i - sum_{i<j} J_ij s_i s_j for all 4096 states; bit i of the state index set
    <=> s_i = -1 (ref sign convention: total_cost, src/model.cpp:108-126)."""
    idx = np.arange(1 << N)
    s = 1.0 - 2.0 * ((idx[:, None] >> np.arange(N)[None, :]) & 1)
    e = -(s @ h.astype(np.float64))
    for a, b, j in pairs:
        e -= float(j) * s[:, a] * s[:, b]
    return e


__all__ = ["random_graph", "csr_from_npz", "product_model", "bits", "oracle_batch", "assert_batch_matches", "ins", "ib", "SMALL_N", "small_model", "enumerate_energies"]
