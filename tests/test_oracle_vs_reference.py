"""Differential tests: the plain-C oracle against the reference's own code run in-process
(oracle/_ref/libisingref.so).  Skipped where the reference sources are absent (the GPU box);
tests/test_oracle_golden.py covers the same ground there from committed vectors."""
import numpy as np
import pytest

from helpers import bits, ins


def models():
    yield "cubic8", ins.cubic_pm1(8, 7, 0.5)
    yield "cubic5_h0", ins.cubic_pm1(5, 8, 0.0)
    yield "mixed6", ins.cubic_mixed_degree(6, 9)
    yield "layered", ins.build_layered_csr(*ins.layered_spec(24, 3), 8, 1.5)
    yield "layered_small_jt", ins.build_layered_csr(*ins.layered_spec(10, 4, degree_max=5), 6, 0.37)


def test_streams_and_maps_agree(port, ref):
    for seed in (1, 5489, 987654321, 0, 0xFFFFFFFF):
        np.testing.assert_array_equal(port.mt_fill(seed, 50000), ref.mt_fill(seed, 50000))
        np.testing.assert_array_equal(port.mt_fill(seed, 3000), ref.mt_next_stream(seed, 3000))
        np.testing.assert_array_equal(port.initial_spins(1000, seed), ref.initial_spins(1000, seed))
    rng = np.random.default_rng(5)
    for x in rng.integers(0, 2**32, 20000, dtype=np.uint64):
        assert port.u32_to_unit(int(x)) == ref.u32_to_unit(int(x))
    for x in np.concatenate([rng.uniform(-110, 110, 20000), [0.0, -0.0, -21.834136, 88.72]]).astype(np.float32):
        for kind in (1, 2, 3):
            a, b = np.float32(port.exp(kind, float(x))), np.float32(ref.exp(kind, float(x)))
            assert a.tobytes() == b.tobytes(), (kind, x)


@pytest.mark.parametrize("kind", [1, 2, 3])
def test_chain_trajectories_agree_every_sweep(port, ref, kind):
    # the trajectory_equivalence pattern (ref: src/oracle.cpp:176-207) with engine B = the port
    for name, csr in models():
        pm, rm = port.model(csr), ref.model(csr)
        assert rm.validate() is None
        for seed, beta, gamma in ((3, 0.4, 1.0), (4, 1.3, 0.6)):
            a = port.chain(pm, seed, beta, gamma, kind)
            b = ref.chain(rm, seed, beta, gamma, kind)
            for sweep in range(120):
                a.sweep(1)
                b.sweep(1)
                assert (a.spins == b.spins).all(), (name, seed, sweep)
            np.testing.assert_array_equal(bits(a.hs), bits(b.hs))
            np.testing.assert_array_equal(bits(a.ht), bits(b.ht))
            assert a.flips == b.flips and a.attempts == b.attempts
            assert port.total_cost(pm, a.spins) == ref.total_cost(rm, b.spins)
            assert port.checksum(a.spins) == ref.checksum(b.spins)


def test_tempering_replay_against_reference_sweeps(port, ref):
    """The swap rule is new, but everything between swaps is reference code: replaying the
    oracle's beta history through the reference's run_sweeps must give the oracle's spins."""
    csr = ins.build_layered_csr(*ins.layered_spec(12, 21), 6, 1.5)
    pm, rm = port.model(csr), ref.model(csr)
    betas = ins.geometric_betas(0.2, 2.0, 4)
    seeds = np.arange(500, 504, dtype=np.uint32)
    interval, rounds = 3, 10
    chains = [ref.chain(rm, int(s), float(betas[k]), 1.0, 2) for k, s in enumerate(seeds)]
    swapped = 0
    prev = np.arange(4)
    for r in range(1, rounds + 1):
        res = port.pt_run([pm], 1, betas, seeds, [9], r * interval, interval, exp_kind=2)
        for c in chains:
            c.sweep(interval)
        got = np.stack([c.spins.astype(np.int8) for c in chains])
        np.testing.assert_array_equal(got, res["spins"])
        np.testing.assert_array_equal([c.flips for c in chains], res["flips"])
        swapped += int((res["slot"] != prev).sum())
        prev = res["slot"].copy()
        for k, c in enumerate(chains):
            c.set_beta(float(betas[res["slot"][k]]))
    assert swapped > 0, "the replay never exercised a swap"
    assert sorted(prev.tolist()) == [0, 1, 2, 3]


def test_layered_builder_agrees(ref):
    from paper_1004_0024_b200 import instances
    positions, h, edges = instances.layered_spec(20, 31)
    mine = instances.build_layered_csr(positions, h, edges, 7, 1.25)
    theirs = ref.build_layered(positions, h, edges, 7, 1.25).csr()
    for key in ("h", "offsets", "targets", "couplings", "tau_counts"):
        np.testing.assert_array_equal(mine[key], theirs[key])


def test_numpy_enumeration_equals_the_reference_enumerate_boltzmann(ref):
    """The exact distributions the GPU statistics tests compare against (tests/helpers.py:
    enumerate_energies, restated with numpy) against the reference's own validator
    (ref: enumerate_boltzmann, proj/src/oracle.cpp:64-109) on the same 12-spin model: every state
    probability, the mean cost and the mean magnetization.  The reference indexes states with bit i
    set for s_i = +1, the tests with bit i set for s_i = -1: complementary indices."""
    from helpers import SMALL_N, enumerate_energies, small_model
    csr, pairs, h = small_model(2024)
    energies = enumerate_energies(pairs, h)
    model = ref.model(csr)
    full = (1 << SMALL_N) - 1
    for beta in (0.15, 0.5, 1.7):
        exact = ref.enumerate_boltzmann(model, beta)
        w = np.exp(-beta * (energies - energies.min()))
        prob = w / w.sum()
        np.testing.assert_allclose(prob[full - np.arange(full + 1)], exact["probabilities"], rtol=1e-10, atol=1e-300)
        assert abs((prob * energies).sum() - exact["mean_cost"]) < 1e-10
        spins = 1.0 - 2.0 * ((np.arange(full + 1)[:, None] >> np.arange(SMALL_N)[None, :]) & 1)
        assert abs((prob * spins.mean(axis=1)).sum() - exact["mean_magnetization"]) < 1e-12


def test_reference_chain_statistics_accepts_the_oracle_model(ref):
    """The reference's replicate-means z-test (ref: chain_statistics_test, proj/src/oracle.cpp:111-174)
    runs on the small model through the shim and passes for its own basic engine: the same bounds
    are applied to the device ladder in tests/test_gpu_statistics.py."""
    from helpers import small_model
    csr, _, _ = small_model(2024)
    rep = ref.chain_statistics(ref.model(csr), 0.5, sweeps=20000, burn_in=2000, replicates=12, base_seed=7)
    assert rep["pass"] == 1.0 and rep["z_cost"] <= 4.0 and rep["z_magnetization"] <= 4.0
    assert abs(rep["est_cost"] - rep["exact_cost"]) < 0.05 * abs(rep["exact_cost"])
