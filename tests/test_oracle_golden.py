"""Pins the plain-C oracle (oracle/ising_oracle.c) to (a) the known-answer values the
reference's own tests hold (ref: proj/tests/test_rng.cpp, test_fastexp.cpp, test_sweep.cpp) and
(b) golden vectors produced by the reference code itself (tests/golden/make_golden.py)."""
import math

import numpy as np
import pytest

from helpers import bits, csr_from_npz


def test_mt19937_known_answers(port):
    # ref: tests/test_rng.cpp:13-17 — canonical first outputs for the default seed
    assert port.mt_fill(5489, 2).tolist() == [3499211612, 581869302]
    # the 10000th output of the canonical generator for seed 5489 (C++ standard, [rand.predef])
    assert int(port.mt_fill(5489, 10000)[-1]) == 4123659995


def test_mt19937_matches_golden_streams(port, golden):
    g = golden("primitives")
    for row, seed in enumerate(g["seeds"]):
        stream = port.mt_fill(int(seed), 1_000_000)  # ref: tests/test_rng.cpp:19-27, 10^6 draws
        got = np.concatenate([stream[a:b] for a, b in g["mt_windows"]])
        np.testing.assert_array_equal(got, g["mt"][row])
        assert np.bitwise_xor.reduce(stream) == g["mt_xor_fold"][row]


def test_mt19937_matches_numpy_legacy_generator(port):
    # independent implementation: numpy's RandomState seeds by init_genrand like the reference
    for seed in (1, 5489, 123456789):
        want = np.random.RandomState(seed).randint(0, 2**32, 5000, dtype=np.uint64).astype(np.uint32)
        np.testing.assert_array_equal(port.mt_fill(seed, 5000), want)


def test_u32_to_unit_endpoints_and_truncation(port, golden):
    # ref: tests/test_rng.cpp:129-179
    assert port.u32_to_unit(0) == 0.0
    assert port.u32_to_unit(2**31) == 0.5
    assert port.u32_to_unit(2**32 - 1) == float.fromhex("0x1.fffffep-1")
    assert port.u32_to_unit(1) == 2.0**-32
    assert port.u32_to_unit(2**24 + 1) == 2.0**-8  # below the representable step: truncated
    g = golden("primitives")
    got = np.array([port.u32_to_unit(int(x)) for x in g["unit_in"]], np.float32)
    np.testing.assert_array_equal(bits(got), bits(g["unit_out"]))
    assert (got < 1.0).all()
    order = np.argsort(g["unit_in"], kind="stable")
    assert (np.diff(got[order]) >= 0).all()  # monotone


def test_exp_anchors_and_masks(port, golden):
    two_ln_sq2 = np.float32(0.9609060278364028)
    # ref: tests/test_fastexp.cpp:15-20 — grid anchors
    assert np.float32(port.exp(2, 0.0)) == two_ln_sq2
    assert np.float32(port.exp(2, float(np.float32(math.log(2.0))))) == np.float32(2) * two_ln_sq2
    # ref: tests/test_fastexp.cpp:82-91 — acceptance masking of exp_accurate
    assert port.exp(3, 0.0) == 1.0 and port.exp(3, 5.0) == 1.0
    assert port.exp(3, -21.9) == 0.0 and port.exp(3, -1e9) == 0.0
    # ref: tests/test_fastexp.cpp:22-34 — error bands
    xs = np.linspace(-20.0, 3.0, 2001)
    for kind, lo, hi in ((2, -0.0392, 0.0201), (3, -0.01, 0.0051)):
        xs_k = xs[xs < 0] if kind == 3 else xs
        rel = np.array([port.exp(kind, float(np.float32(x))) / math.exp(float(np.float32(x))) - 1 for x in xs_k])
        assert rel.min() > lo and rel.max() < hi
    g = golden("primitives")
    for row, kind in enumerate((1, 2, 3)):
        got = np.array([port.exp(kind, float(x)) for x in g["exp_in"]], np.float32)
        np.testing.assert_array_equal(bits(got), bits(g["exp_out"][row]))


def test_initial_spins_match_golden(port, golden):
    g = golden("primitives")
    for row, seed in enumerate(g["seeds"]):
        np.testing.assert_array_equal(port.initial_spins(700, int(seed)), g["initial_spins"][row])


@pytest.mark.parametrize("name", ["cubic4_pm1", "cubic6_gauss_h", "mixed6", "layered_24x8", "layered_16x4_gamma"])
def test_trajectories_match_reference_golden(port, golden, name):
    g = golden(f"traj_{name}")
    csr = csr_from_npz(g)
    model = port.model(csr)
    beta, gamma, sweeps = float(g["beta"]), float(g["tau_scale"]), int(g["sweeps"])
    for kind, seed in g["runs"]:
        tag = f"k{kind}_s{seed}"
        chain = port.chain(model, int(seed), beta, gamma, int(kind))
        np.testing.assert_array_equal(chain.spins.astype(np.int8), g[f"{tag}_spins0"])
        np.testing.assert_array_equal(bits(chain.hs), bits(g[f"{tag}_hs0"]))
        np.testing.assert_array_equal(bits(chain.ht), bits(g[f"{tag}_ht0"]))
        chain.sweep(sweeps // 2)
        np.testing.assert_array_equal(chain.spins.astype(np.int8), g[f"{tag}_spins_mid"])
        chain.sweep(sweeps - sweeps // 2)
        np.testing.assert_array_equal(chain.spins.astype(np.int8), g[f"{tag}_spins"])
        np.testing.assert_array_equal(bits(chain.hs), bits(g[f"{tag}_hs"]))
        np.testing.assert_array_equal(bits(chain.ht), bits(g[f"{tag}_ht"]))
        assert chain.flips == int(g[f"{tag}_flips"]) and chain.attempts == int(g[f"{tag}_attempts"])
        assert port.total_cost(model, chain.spins) == float(g[f"{tag}_cost"])
        assert port.checksum(chain.spins) == int(g[f"{tag}_checksum"])
        # running energy (new): tracks the energy the sweeps sample (tau couplings scaled by gamma) to
        # f32-rounding accuracy; that energy is the reference's total_cost when gamma == 1
        sampled = port.tempering_cost(model, chain.spins, gamma)
        if gamma == 1.0:
            assert sampled == float(g[f"{tag}_cost"])
        assert abs(chain.e_run - sampled) <= 1e-5 * max(1.0, abs(sampled))


def test_two_spin_forced_flip_hand_trace(port, golden):
    # ref: tests/test_sweep.cpp:132-145 — beta = 0 accepts everything (exact exp: p = 1 > u)
    two = dict(n_spins=2, h=np.zeros(2, np.float32), offsets=[0, 1, 2], targets=[1, 0],
               couplings=np.ones(2, np.float32))
    model = port.model(two)
    chain = port.chain(model, 1, 0.0, 1.0, 1, initial=[1, -1])
    assert chain.hs.tolist() == [-1.0, 1.0]  # ref: tests/test_sweep.cpp:54-64 (field init)
    chain.sweep(1)
    assert chain.spins.tolist() == [-1.0, 1.0]
    chain.sweep(1)
    assert chain.spins.tolist() == [1.0, -1.0]
    assert chain.flips == 4 and chain.attempts == 4
    g = golden("traj_two_spin")
    np.testing.assert_array_equal(chain.spins.astype(np.int8), g["spins"])


def test_frozen_chain_never_flips(port):
    # ref: tests/test_sweep.cpp:122-130 — one spin, h = 1, s = +1, beta = 200
    one = dict(n_spins=1, h=np.ones(1, np.float32), offsets=[0, 0], targets=[], couplings=[])
    model = port.model(one)
    for kind in (1, 2, 3):
        chain = port.chain(model, 1, 200.0, 1.0, kind, initial=[1])
        chain.sweep(100)
        assert chain.flips == 0 and chain.spins.tolist() == [1.0]


def test_fast_exp_rejects_some_zero_field_flips(port):
    # No min(1, .) clamp: with exp_fast p(0) = 2 ln^2 2 < 1, so a free spin is not always flipped
    # (ref: src/sweep_basic.cpp:36-37, tests/test_fastexp.cpp:17).
    one = dict(n_spins=1, h=np.zeros(1, np.float32), offsets=[0, 0], targets=[], couplings=[])
    model = port.model(one)
    chain = port.chain(model, 3, 1.0, 1.0, 2, initial=[1])
    chain.sweep(20000)
    assert 0.95 < chain.flips / 20000 < 0.97
    exact = port.chain(model, 3, 1.0, 1.0, 1, initial=[1])
    exact.sweep(20000)
    assert exact.flips == 20000


def test_exactly_one_uniform_per_spin_per_sweep(port):
    # ref: tests/test_sweep.cpp:327-336 — draw index = sweep * n + i.  A one-spin free chain under
    # the exact exponential at beta = 0 consumes but ignores its draws; interleave two chains of
    # different sizes and check their streams stay aligned with a replayed generator.
    n = 5
    free = dict(n_spins=n, h=np.zeros(n, np.float32), offsets=[0] * (n + 1), targets=[], couplings=[])
    model = port.model(free)
    chain = port.chain(model, 99, 1.0, 1.0, 2, initial=[1] * n)
    sweeps = 400
    stream = port.mt_fill(99, sweeps * n)
    p0 = np.float32(port.exp(2, 0.0))
    spins = np.ones(n)
    flips = 0
    for k, raw in enumerate(stream):
        if np.float32(port.u32_to_unit(int(raw))) < p0:
            spins[k % n] *= -1
            flips += 1
    chain.sweep(sweeps)
    assert chain.flips == flips and chain.spins.tolist() == spins.tolist()
