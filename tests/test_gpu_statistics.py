"""Statistical validation of the tempering sampler (SURVEY.md §8 f4, §8c "tempering swap: parity
unpinned"): the swap rule has no counterpart in the reference, so beyond CPU-vs-GPU parity it is
checked here against GROUND TRUTH — the exact Boltzmann distribution of a 12-spin model obtained
by enumerating its 4096 states (the approach of the reference's own validator, ref:
proj/src/oracle.cpp:64-109, restated with numpy).  With `exp_kind = exact` sequential-sweep
Metropolis plus replica exchange leaves every beta slot exactly Boltzmann distributed; checked are
the state histogram of every slot (chi-square), its mean energy, and the swap acceptance rate of
every neighbouring pair against its exact expectation under independent Boltzmann replicas."""
import numpy as np
import pytest

import paper_1004_0024_b200 as ib
from helpers import ins

pytestmark = pytest.mark.gpu

N = 12


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


def test_every_beta_slot_samples_the_exact_boltzmann_distribution(lib):
    csr, pairs, h = small_model(2024)
    energies = enumerate_energies(pairs, h)
    betas = np.array([0.15, 0.3, 0.5, 0.8, 1.2, 1.7], np.float32)
    nb, ladders = betas.size, 2048
    model = ib.SpinModel.from_csr(N, csr["h"], csr["offsets"], csr["targets"], csr["couplings"], csr["tau_counts"], 0, 0)
    # cross-check the enumeration against the product's own f64 energy on a few states
    for state_index in (0, 1, 2730, 4095):
        spins = (1 - 2 * ((state_index >> np.arange(N)) & 1)).astype(np.int8)
        assert abs(ib.total_cost(model, spins) - energies[state_index]) < 1e-9

    weights = np.exp(-betas.astype(np.float64)[:, None] * (energies[None, :] - energies.min()))
    prob = weights / weights.sum(axis=1, keepdims=True)

    snapshots, stride, burn_in = 48, 6, 300
    hist = np.zeros((nb, 1 << N))
    e_sum = np.zeros(nb)
    with ib.init_state(model, betas, ladders, base_seed=4242, swap_base_seed=777,
                       params=ib.SweepParams(1.0, ib.ExpKind.exact)) as st:
        st.run(burn_in, 1)
        acc0, att0 = st.swap_stats()
        for _ in range(snapshots):
            st.run(stride, 1)
            spins = st.spins()
            slots = st.slots()
            index = ((spins < 0).astype(np.int64) << np.arange(N)[None, :]).sum(axis=1)
            for k in range(nb):
                sel = index[slots == k]
                hist[k] += np.bincount(sel, minlength=1 << N)
                e_sum[k] += energies[sel].sum()
        acc1, att1 = st.swap_stats()
        # every ladder keeps exactly one chain per slot
        assert (np.sort(st.slots().reshape(ladders, nb), axis=1) == np.arange(nb)).all()

    samples = ladders * snapshots
    for k in range(nb):
        assert hist[k].sum() == samples
        expected = prob[k] * samples
        big = expected >= 8.0
        obs = np.append(hist[k][big], hist[k][~big].sum())
        exp = np.append(expected[big], expected[~big].sum())
        keep = exp > 0
        chi2 = (((obs - exp) ** 2)[keep] / exp[keep]).sum()
        dof = keep.sum() - 1
        z = (chi2 - dof) / np.sqrt(2.0 * dof)
        # snapshots of one ladder are a few sweeps apart, i.e. mildly correlated: generous bound
        assert z < 8.0, f"slot {k}: chi-square {chi2:.1f} for {dof} degrees of freedom (z = {z:.1f})"
        mean_exact = (prob[k] * energies).sum()
        var_exact = (prob[k] * (energies - mean_exact) ** 2).sum()
        z_mean = (e_sum[k] / samples - mean_exact) / np.sqrt(var_exact / samples)
        assert abs(z_mean) < 6.0, f"slot {k}: mean energy off by {z_mean:.1f} sigma"

    # swap acceptance of pair (k, k+1): E[min(1, exp((b_k - b_k+1) (E_a - E_b)))] over independent
    # Boltzmann states a ~ p_k, b ~ p_k+1 (exact, 4096^2 terms)
    acc = (acc1 - acc0).sum(axis=0).astype(np.float64)
    att = (att1 - att0).sum(axis=0).astype(np.float64)
    for k in range(nb - 1):
        delta = (float(betas[k]) - float(betas[k + 1])) * (energies[:, None] - energies[None, :])
        expect = (prob[k][:, None] * prob[k + 1][None, :] * np.minimum(1.0, np.exp(delta))).sum()
        rate = acc[k] / att[k]
        sigma = np.sqrt(expect * (1 - expect) / att[k])
        assert att[k] > 0 and abs(rate - expect) < 8.0 * sigma + 2e-3, \
            f"pair {k}: swap acceptance {rate:.4f}, exact expectation {expect:.4f}"


def test_a_wrong_temperature_is_detected(lib):
    """Power of the test above: the same statistics reject a ladder whose hottest slot is sampled at
    a beta 10 % off."""
    csr, pairs, h = small_model(2024)
    energies = enumerate_energies(pairs, h)
    model = ib.SpinModel.from_csr(N, csr["h"], csr["offsets"], csr["targets"], csr["couplings"], csr["tau_counts"], 0, 0)
    beta_run, beta_claimed = np.float32(0.55), 0.5
    weights = np.exp(-beta_claimed * (energies - energies.min()))
    prob = weights / weights.sum()
    ladders, snapshots = 2048, 24
    e_sum = 0.0
    with ib.init_state(model, [beta_run], ladders, base_seed=99, params=ib.SweepParams(1.0, ib.ExpKind.exact)) as st:
        st.run(200)
        for _ in range(snapshots):
            st.run(6)
            spins = st.spins()
            index = ((spins < 0).astype(np.int64) << np.arange(N)[None, :]).sum(axis=1)
            e_sum += energies[index].sum()
    samples = ladders * snapshots
    mean_exact = (prob * energies).sum()
    var_exact = (prob * (energies - mean_exact) ** 2).sum()
    assert abs((e_sum / samples - mean_exact) / np.sqrt(var_exact / samples)) > 6.0
