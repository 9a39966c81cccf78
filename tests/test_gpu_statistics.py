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
from helpers import SMALL_N, enumerate_energies, ins, small_model

pytestmark = pytest.mark.gpu

N = SMALL_N


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


def test_reference_z_test_bounds_on_the_device_ladder(lib):
    """The reference's chain_statistics_test (ref: proj/src/oracle.cpp:111-174) applied to the device
    sampler: every ladder is one replicate, its time-averaged cost and magnetization per beta slot are
    the replicate means, the standard error comes from their spread, and both observables must land
    within the reference's z threshold (4) of the exact values — which tests/test_oracle_vs_reference.py
    pins to the reference's own enumerate_boltzmann."""
    csr, pairs, h = small_model(2024)
    energies = enumerate_energies(pairs, h)
    states = np.arange(1 << N)
    magnet = (1.0 - 2.0 * ((states[:, None] >> np.arange(N)[None, :]) & 1)).mean(axis=1)
    betas = np.array([0.15, 0.3, 0.5, 0.8, 1.2, 1.7], np.float32)
    nb, ladders, sweeps, burn_in = betas.size, 64, 1500, 300
    model = ib.SpinModel.from_csr(N, csr["h"], csr["offsets"], csr["targets"], csr["couplings"], csr["tau_counts"], 0, 0)
    cost_sum = np.zeros((ladders, nb))
    mag_sum = np.zeros((ladders, nb))
    with ib.init_state(model, betas, ladders, base_seed=31337, swap_base_seed=4711,
                       params=ib.SweepParams(1.0, ib.ExpKind.exact)) as st:
        st.run(burn_in, 1)
        for _ in range(sweeps):
            st.run(1, 1)
            index = ((st.spins() < 0).astype(np.int64) << np.arange(N)[None, :]).sum(axis=1).reshape(ladders, nb)
            slots = st.slots().reshape(ladders, nb)
            rows = np.arange(ladders)[:, None]
            cost_sum[rows, slots] += energies[index]
            mag_sum[rows, slots] += magnet[index]
    for k in range(nb):
        w = np.exp(-float(betas[k]) * (energies - energies.min()))
        prob = w / w.sum()
        for name, sums, exact in (("cost", cost_sum, (prob * energies).sum()), ("magnetization", mag_sum, (prob * magnet).sum())):
            rep = sums[:, k] / sweeps
            se = rep.std(ddof=1) / np.sqrt(ladders)
            z = abs(rep.mean() - exact) / se
            assert z <= 4.0, f"slot {k}: {name} {rep.mean():.5f} vs exact {exact:.5f}, z = {z:.2f}"


def test_tempering_with_tau_scale_samples_the_scaled_energy(lib):
    """A layered model with gamma = 0.6: the sweeps sample exp(-beta (E_space + gamma E_tau)), and the swap
    compares running energies of exactly that quantity (oracle/ising_oracle.h), so every beta slot must
    be Boltzmann distributed in the SCALED energy.  16 spins (4 positions x 4 layers), exact exponential;
    mean scaled energy per slot and the swap acceptance of every pair against exact enumeration.  (With
    the unscaled energy in the swap rule the cold slots' means are off by many sigma.)"""
    positions, layers, gamma, j_tau = 4, 4, np.float32(0.6), np.float32(0.9)
    rng = ins.MT19937(77)
    h = rng.normals(positions, 0.5).astype(np.float32)
    edges = [(0, 1, 0.8), (1, 2, -1.1), (2, 3, 0.7), (0, 3, -0.5), (0, 2, 0.4)]
    csr = ins.build_layered_csr(positions, h, edges, layers, float(j_tau))
    n = positions * layers
    states = np.arange(1 << n)
    s = 1.0 - 2.0 * ((states[:, None] >> np.arange(n)[None, :]) & 1)
    e_space = -(s @ np.tile(h.astype(np.float64), layers))
    e_tau = np.zeros(1 << n)
    for l in range(layers):
        for a, b, j in edges:
            e_space -= float(np.float32(j)) * s[:, l * positions + a] * s[:, l * positions + b]
        for p in range(positions):
            e_tau -= float(j_tau) * s[:, l * positions + p] * s[:, ((l + 1) % layers) * positions + p]
    # the tempering energy scales every tau coupling by gamma in f32 (orc_tempering_cost)
    e_scaled = e_space + float(np.float32(gamma * j_tau)) / float(j_tau) * e_tau
    betas = np.array([0.2, 0.45, 0.8, 1.3], np.float32)
    nb, ladders, snapshots, stride = betas.size, 1024, 40, 5
    model = ib.SpinModel.from_csr(n, csr["h"], csr["offsets"], csr["targets"], csr["couplings"], csr["tau_counts"],
                                  csr["layers"], csr["per_layer"])
    e_sum = np.zeros(nb)
    with ib.init_state(model, betas, ladders, base_seed=5150, swap_base_seed=90210,
                       params=ib.SweepParams(float(gamma), ib.ExpKind.exact)) as st:
        st.run(300, 1)
        acc0, att0 = st.swap_stats()
        for _ in range(snapshots):
            st.run(stride, 1)
            index = ((st.spins() < 0).astype(np.int64) << np.arange(n)[None, :]).sum(axis=1)
            slots = st.slots()
            for k in range(nb):
                e_sum[k] += e_scaled[index[slots == k]].sum()
        acc1, att1 = st.swap_stats()
    samples = ladders * snapshots
    prob = []
    for k in range(nb):
        w = np.exp(-float(betas[k]) * (e_scaled - e_scaled.min()))
        prob.append(w / w.sum())
        mean_exact = (prob[k] * e_scaled).sum()
        var_exact = (prob[k] * (e_scaled - mean_exact) ** 2).sum()
        z = (e_sum[k] / samples - mean_exact) / np.sqrt(var_exact / samples)
        assert abs(z) < 6.0, f"slot {k}: mean scaled energy off by {z:.1f} sigma"
    acc = (acc1 - acc0).sum(axis=0).astype(np.float64)
    att = (att1 - att0).sum(axis=0).astype(np.float64)
    for k in range(nb - 1):
        # exact pair expectation from the energy histograms (65536^2 pairs is too many: bin by energy value)
        ea, inv_a = np.unique(np.round(e_scaled, 9), return_inverse=True)
        pa = np.bincount(inv_a, weights=prob[k])
        pb = np.bincount(inv_a, weights=prob[k + 1])
        delta = (float(betas[k]) - float(betas[k + 1])) * (ea[:, None] - ea[None, :])
        expect = (pa[:, None] * pb[None, :] * np.minimum(1.0, np.exp(delta))).sum()
        rate = acc[k] / att[k]
        sigma = np.sqrt(expect * (1 - expect) / att[k])
        assert abs(rate - expect) < 8.0 * sigma + 3e-3, f"pair {k}: swap acceptance {rate:.4f}, exact {expect:.4f}"
