"""Parity of the CUDA path (through the C ABI) against the CPU oracle on identical seeded inputs:
spins, accept counts, beta slots and running energies bit-exact, energies within 1e-5 relative
(BASELINE.json north_star).  Shapes follow BASELINE.json's five configurations at sizes the
oracle finishes in seconds."""
import numpy as np
import pytest

import paper_1004_0024_b200 as ib
from paper_1004_0024_b200 import _lib
from helpers import assert_batch_matches, bits, csr_from_npz, ins, oracle_batch, product_model, random_graph

pytestmark = pytest.mark.gpu

REL_ENERGY = 1e-5  # north_star tolerance for energies
KERNELS = [ib.KERNEL_GENERIC]                       # any graph
LAYERED_KERNELS = [ib.KERNEL_GENERIC, ib.KERNEL_LAYERED, ib.KERNEL_STRAND]  # identical-layer models: all families


def run_both(port, csrs, n_ladders, betas, sweeps, swap_interval, *, seed0=ins.CHAIN_SEED_BASE, tau_scale=1.0,
             exp_kind=2, model_of_ladder=None, initial=None, kernel=ib.KERNEL_AUTO, chunks=None):
    betas = np.atleast_1d(np.asarray(betas, np.float32))
    chains = n_ladders * betas.size
    seeds = (seed0 + np.arange(chains)).astype(np.uint32)
    swap_seeds = (ins.SWAP_SEED_BASE + np.arange(n_ladders)).astype(np.uint32)
    want = oracle_batch(port, csrs, n_ladders, betas, seeds, swap_seeds, sweeps, swap_interval, tau_scale,
                        exp_kind, model_of_ladder, initial)
    models = [product_model(c) for c in csrs]
    state = ib.init_state(models, betas, n_ladders, seeds=seeds, swap_seeds=swap_seeds,
                          params=ib.SweepParams(tau_scale, exp_kind), model_of_ladder=model_of_ladder,
                          initial_spins=initial, kernel=kernel)
    for part in (chunks or [sweeps]):
        state.run(part, swap_interval)
    return state, want


@pytest.mark.parametrize("name", ["cubic4_pm1", "cubic6_gauss_h", "mixed6", "layered_24x8", "layered_16x4_gamma"])
def test_reference_golden_trajectories(lib, golden, name):
    """Outputs of the reference itself (tests/golden/make_golden.py), no oracle in the loop."""
    g = golden(f"traj_{name}")
    csr = csr_from_npz(g)
    model = product_model(csr)
    beta, gamma, sweeps = float(g["beta"]), float(g["tau_scale"]), int(g["sweeps"])
    families = LAYERED_KERNELS if name.startswith("layered") else KERNELS
    for kind, family in [(k, f) for k in (1, 2, 3) for f in families]:
        seeds = [int(s) for k, s in g["runs"] if k == kind]
        with ib.init_state(model, [beta], len(seeds), seeds=seeds, params=ib.SweepParams(gamma, kind),
                           kernel=family) as st:
            assert st.info()["kernel"] == family
            for c, seed in enumerate(seeds):
                tag = f"k{kind}_s{seed}"
                np.testing.assert_array_equal(st.spins(c, 1)[0], g[f"{tag}_spins0"])
                hs, ht = st.fields(c)
                np.testing.assert_array_equal(bits(hs), bits(g[f"{tag}_hs0"]))
                np.testing.assert_array_equal(bits(ht), bits(g[f"{tag}_ht0"]))
            st.run(sweeps // 2)
            for c, seed in enumerate(seeds):
                np.testing.assert_array_equal(st.spins(c, 1)[0], g[f"k{kind}_s{seed}_spins_mid"])
            st.run(sweeps - sweeps // 2)
            flips, attempts = st.stats()
            energies, sums, coh = st.energies(), st.checksums(), st.field_coherence_ulp()
            for c, seed in enumerate(seeds):
                tag = f"k{kind}_s{seed}"
                np.testing.assert_array_equal(st.spins(c, 1)[0], g[f"{tag}_spins"])
                hs, ht = st.fields(c)
                np.testing.assert_array_equal(bits(hs), bits(g[f"{tag}_hs"]))
                np.testing.assert_array_equal(bits(ht), bits(g[f"{tag}_ht"]))  # rebuilt, not stored, when layered
                assert flips[c] == g[f"{tag}_flips"] and attempts[c] == g[f"{tag}_attempts"]
                assert energies[c] == pytest.approx(float(g[f"{tag}_cost"]), rel=REL_ENERGY)
                assert energies[c] == float(g[f"{tag}_cost"])  # same f64 summation order: exact
                assert sums[c] == g[f"{tag}_checksum"]
                assert coh[c] == g[f"{tag}_coherence"]


def test_two_spin_hand_trace_and_frozen_chain(lib, golden):
    # ref: tests/test_sweep.cpp:122-145
    two = ib.SpinModel.from_csr(2, [0, 0], [0, 1, 2], [1, 0], [1.0, 1.0])
    with ib.init_state(two, [0.0], 1, seeds=[1], params=ib.SweepParams(1.0, ib.ExpKind.exact),
                       initial_spins=[[1, -1]]) as st:
        hs, ht = st.fields(0)
        assert hs.tolist() == [-1.0, 1.0] and ht.tolist() == [0.0, 0.0]
        st.run(1)
        assert st.spins()[0].tolist() == [-1, 1]
        st.run(1)
        assert st.spins()[0].tolist() == [1, -1]
        flips, attempts = st.stats()
        assert flips[0] == 4 and attempts[0] == 4
        np.testing.assert_array_equal(st.spins()[0], golden("traj_two_spin")["spins"])
    one = ib.SpinModel.from_csr(1, [1.0], [0, 0], [], [])
    for kind in (1, 2, 3):
        with ib.init_state(one, [200.0], 1, seeds=[1], params=ib.SweepParams(1.0, kind), initial_spins=[[1]]) as st:
            st.run(100)
            assert st.stats()[0][0] == 0 and st.spins()[0].tolist() == [1]


@pytest.mark.parametrize("kernel", KERNELS)
def test_c1_single_chain_cubic(lib, port, kernel):
    """BASELINE config 1: 16^3 periodic lattice, J = +/-1, h = 0, one replica at beta = 1."""
    csr = ins.cubic_pm1(16, ins.INSTANCE_SEED, 0.0)
    state, want = run_both(port, [csr], 1, [1.0], 1000, 0, kernel=kernel)
    e = assert_batch_matches(state, want, REL_ENERGY)
    assert 0.05 < want["flips"][0] / (1000 * 4096) < 0.15
    assert state.checksums()[0] == ib.state_checksum(want["spins"][0])
    assert abs(state.running_energies()[0] - e[0]) == 0.0  # +/-1 couplings, h = 0: every dE is exact


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("exp_kind", [1, 2, 3])
def test_c2_many_replicas_gaussian_fields(lib, port, kernel, exp_kind):
    """BASELINE config 2 shape: same lattice, h ~ N(0, 0.5^2), replicas seeded base + id; a chain
    count that leaves a ragged last tile."""
    csr = ins.cubic_pm1(16, ins.INSTANCE_SEED, 0.5)
    state, want = run_both(port, [csr], 70, [1.0], 60, 0, exp_kind=exp_kind, kernel=kernel)
    assert_batch_matches(state, want, REL_ENERGY)
    assert state.info()["n_tiles"] == 3


@pytest.mark.parametrize("kernel", KERNELS)
def test_c3_tempering_mixed_degree_distinct_graphs(lib, port, kernel):
    """BASELINE config 3 shape: lattice + 0-2 extra edges per spin, Gaussian J and h, a geometric
    ladder with a swap attempt every sweep, every system its own graph."""
    csrs = [ins.cubic_mixed_degree(8, ins.INSTANCE_SEED + k) for k in range(5)]
    betas = ins.geometric_betas(0.1, 3.0, 32)
    state, want = run_both(port, csrs, 5, betas, 120, 1, kernel=kernel)
    assert_batch_matches(state, want, REL_ENERGY)
    assert want["swap_acc"].sum() > 100 and (want["swap_att"][:, :31].sum(1) == 120 * 31 // 2).all()
    assert (np.sort(want["slot"].reshape(5, 32), 1) == np.arange(32)).all()


@pytest.mark.parametrize("kernel", LAYERED_KERNELS)
@pytest.mark.parametrize("swap_interval", [1, 10])
def test_c4_layered_tempering(lib, port, kernel, swap_interval):
    """BASELINE config 4/5 shape: identical layers, J = +/-1, J_perp = 1.5 ring along tau, Gaussian h."""
    csrs = [ins.build_layered_csr(*ins.layered_spec(32, ins.INSTANCE_SEED + k), 8, 1.5) for k in range(3)]
    betas = ins.geometric_betas(0.2, 5.0, 16)
    state, want = run_both(port, csrs, 3, betas, 90, swap_interval, kernel=kernel)
    assert_batch_matches(state, want, REL_ENERGY)
    assert want["swap_acc"].sum() > 0
    # tau fields only ever take the values {-2J, 0, +2J} (the basis of the on-chip tau elision)
    _, ht = state.fields(7)
    assert set(np.unique(ht)).issubset({-3.0, 0.0, 3.0})


@pytest.mark.parametrize("kernel", LAYERED_KERNELS)
def test_shared_graph_many_ladders_tau_scale(lib, port, kernel):
    csr = ins.build_layered_csr(*ins.layered_spec(16, 77), 6, 0.75)
    betas = ins.geometric_betas(0.3, 2.0, 6)
    state, want = run_both(port, [csr], 11, betas, 50, 2, tau_scale=0.5, exp_kind=3, kernel=kernel)
    assert_batch_matches(state, want, REL_ENERGY)


def test_split_runs_equal_one_run(lib, port):
    """run(a); run(b) == run(a + b): the swap cadence counts sweeps since creation."""
    csr = ins.cubic_mixed_degree(6, 9)
    betas = ins.geometric_betas(0.2, 2.0, 4)
    state, want = run_both(port, [csr], 6, betas, 35, 3, chunks=[1, 4, 7, 0, 23])
    assert_batch_matches(state, want, REL_ENERGY)


def test_explicit_swap_round_matches_interval(lib, port):
    csr = ins.cubic_mixed_degree(6, 9)
    betas = ins.geometric_betas(0.2, 2.0, 5)
    seeds = np.arange(40, 50, dtype=np.uint32)
    want = oracle_batch(port, [csr], 2, betas, seeds, [5, 6], 12, 4)
    with ib.init_state(product_model(csr), betas, 2, seeds=seeds, swap_seeds=[5, 6]) as st:
        for _ in range(3):
            st.run(4, 0)
            st.swap()
        assert_batch_matches(st, want, REL_ENERGY)


@pytest.mark.parametrize("kernel", LAYERED_KERNELS)
def test_results_do_not_depend_on_batch_composition(lib, port, kernel):
    """The reference's worker-count invariance (ref: tests/test_bench.cpp:153-166) as the
    multi-GPU property: a ladder's bits are the same alone, in a big batch, or in a shard
    addressed through first_ladder."""
    csr = ins.build_layered_csr(*ins.layered_spec(16, 3), 4, 1.5)
    model = product_model(csr)
    betas = ins.geometric_betas(0.2, 3.0, 8)
    with ib.init_state(model, betas, 9, base_seed=100, swap_base_seed=900, kernel=kernel) as full:
        full.run(40, 5)
        all_spins, all_sums, all_slots = full.spins(), full.checksums(), full.slots()
    for first, count in ((0, 4), (4, 5), (8, 1)):
        with ib.init_state(model, betas, count, base_seed=100, swap_base_seed=900, first_ladder=first,
                           kernel=kernel) as part:
            part.run(40, 5)
            np.testing.assert_array_equal(part.spins(), all_spins[first * 8:(first + count) * 8])
            np.testing.assert_array_equal(part.checksums(), all_sums[first * 8:(first + count) * 8])
            np.testing.assert_array_equal(part.slots(), all_slots[first * 8:(first + count) * 8])


def test_edge_cases(lib, port):
    # one spin, no edges; 33 chains (ragged second tile); zero sweeps; isolated spins in a graph
    one = dict(n_spins=1, h=np.array([0.3], np.float32), offsets=[0, 0], targets=[], couplings=[])
    state, want = run_both(port, [one], 33, [0.7], 500, 0)
    assert_batch_matches(state, want)
    state, want = run_both(port, [one], 1, [0.7], 0, 0)
    assert_batch_matches(state, want)
    iso = dict(n_spins=5, h=np.array([0.1, -0.2, 0, 1, -1], np.float32), offsets=[0, 1, 1, 2, 2, 2],
               targets=[2, 0], couplings=[0.5, 0.5])
    state, want = run_both(port, [iso], 2, [0.2, 1.5], 300, 1)
    assert_batch_matches(state, want)
    # beta = 0 with the exact exponential: every attempt is accepted
    with ib.init_state(product_model(iso), [0.0], 1, params=ib.SweepParams(1.0, 1)) as st:
        st.run(11)
        assert st.stats()[0][0] == 55


def test_one_shot_run_report(lib, port):
    """ref: ising_run, include/isingmc.h:74-106 / tests/test_capi.cpp:129-148."""
    csr = ins.cubic_pm1(6, 11, 0.5)
    rep = ib.run_single(product_model(csr), 200, 0.9, 321, exp_kind=ib.ExpKind.default)
    model = port.model(csr)
    chain = port.chain(model, 321, 0.9, 1.0, 2)
    chain.sweep(200)
    assert rep["flips"] == chain.flips and rep["attempts"] == 200 * 216
    assert rep["checksum"] == port.checksum(chain.spins)
    assert rep["final_cost"] == port.total_cost(model, chain.spins)
    assert rep["flip_rate"] == chain.flips / (200 * 216)


def test_argument_errors(lib):
    # ref: check_engine_model, src/sweep_state.cpp:148-157; capi status mapping capi.cpp:37-59
    model = product_model(ins.cubic_pm1(3, 1, 0.0))
    other = product_model(ins.cubic_pm1(4, 1, 0.0))
    cases = [
        (dict(betas=[-1.0]), "beta must be finite"),
        (dict(betas=[float("nan")]), "beta must be finite"),
        (dict(betas=[1.0], params=ib.SweepParams(float("inf"), 2)), "tau_scale must be finite"),
        (dict(betas=[1.0], params=ib.SweepParams(1.0, 9)), "invalid exp_kind"),
        (dict(betas=[1.0], device=99), "invalid device"),
        (dict(betas=[1.0], n_ladders=0), "at least one chain"),
        (dict(betas=[1.0], initial_spins=[[0] * 27]), "spins must be +/-1"),
    ]
    for kwargs, text in cases:
        kwargs.setdefault("n_ladders", 1)
        with pytest.raises(ib.IsingError) as err:
            ib.init_state(model, **kwargs)
        assert err.value.status == _lib.ISING_ERR_ARGUMENT and text in str(err.value), str(err.value)
    with pytest.raises(ib.IsingError) as err:
        ib.init_state([model, other], [1.0], 2)
    assert "same spin count" in str(err.value)
    with ib.init_state(model, [1.0], 2) as st:
        with pytest.raises(ib.IsingError):
            st.spins(1, 5)
        with pytest.raises(ib.IsingError):
            st.fields(2)


def test_pack_results_matches_host_readouts(lib):
    import torch
    csr = ins.cubic_mixed_degree(6, 9)
    with ib.init_state(product_model(csr), ins.geometric_betas(0.2, 2.0, 4), 5) as st:
        st.run(30, 2)
        buf = torch.zeros(st.n_chains * 4, dtype=torch.int64, device="cuda")
        st.pack_results(buf.data_ptr())
        rec = buf.cpu().numpy().reshape(-1, 4)
        np.testing.assert_array_equal(rec[:, 0].view(np.float64), st.energies())
        np.testing.assert_array_equal(rec[:, 1].view(np.float64), st.running_energies())
        np.testing.assert_array_equal(rec[:, 2].view(np.uint64), st.stats()[0])
        np.testing.assert_array_equal(rec[:, 3].view(np.uint64), st.checksums())


def test_layered_family_selection_and_rejection(lib):
    """AUTO picks the strand family exactly when every model qualifies (identical layers, one tau
    coupling per position, a multiple of 8 and at least 16 positions per layer), else the Tensor Memory
    family when that one does, else the generic one; asking for a family that does not apply is an
    argument error (no silent fallback)."""
    layered = product_model(ins.build_layered_csr(*ins.layered_spec(16, 3), 4, 1.5))
    short_layers = product_model(ins.build_layered_csr(*ins.layered_spec(8, 3), 8, 1.5))  # 8 positions per layer
    generic = product_model(ins.cubic_pm1(4, 1, 0.0))  # 64 spins like the layered ones
    with ib.init_state(layered, [1.0], 2) as st:
        assert st.info()["kernel"] == ib.KERNEL_STRAND and st.info()["strands"] >= 1
    with ib.init_state(layered, [1.0], 2, kernel=ib.KERNEL_LAYERED) as st:
        assert st.info()["kernel"] == ib.KERNEL_LAYERED and st.info()["strands"] == 0
    with ib.init_state(short_layers, [1.0], 2) as st:
        assert st.info()["kernel"] == ib.KERNEL_LAYERED
    with ib.init_state(generic, [1.0], 2) as st:
        assert st.info()["kernel"] == ib.KERNEL_GENERIC
    with ib.init_state([layered, generic], [1.0], 2) as st:
        assert st.info()["kernel"] == ib.KERNEL_GENERIC
    with pytest.raises(ib.IsingError) as err:
        ib.init_state(generic, [1.0], 2, kernel=ib.KERNEL_LAYERED)
    assert err.value.status == _lib.ISING_ERR_ARGUMENT and "layered kernel needs" in str(err.value)
    for bad in (generic, short_layers):
        with pytest.raises(ib.IsingError) as err:
            ib.init_state(bad, [1.0], 2, kernel=ib.KERNEL_STRAND)
        assert err.value.status == _lib.ISING_ERR_ARGUMENT and "strand kernel needs" in str(err.value)
    # unequal tau couplings per spin: still a valid layered model, but the tau field must be stored
    csr = ins.build_layered_csr(*ins.layered_spec(8, 5), 4, 1.5)
    csr["couplings"] = csr["couplings"].copy()
    P, n = 8, 32
    for i in range(n):  # scale the (up, down) pair of layer boundary 0|1 consistently
        l, p = divmod(i, P)
        end = csr["offsets"][i + 1]
        if l == 0:
            csr["couplings"][end - 2] = 0.5  # up edge of layer 0
        if l == 1:
            csr["couplings"][end - 1] = 0.5  # down edge of layer 1
    with ib.init_state(product_model(csr), [1.0], 1) as st:
        assert st.info()["kernel"] == ib.KERNEL_GENERIC


def test_layered_many_tiles_and_sweeps(lib, port):
    """More tiles than one CTA round holds warps for, ragged last tile, several launches."""
    csr = ins.build_layered_csr(*ins.layered_spec(40, 8), 5, 1.5)
    betas = ins.geometric_betas(0.3, 3.0, 3)
    state, want = run_both(port, [csr], 45, betas, 24, 4, kernel=ib.KERNEL_LAYERED, chunks=[3, 9, 12])
    assert state.info()["kernel"] == ib.KERNEL_LAYERED and state.info()["n_tiles"] == 5
    assert_batch_matches(state, want, REL_ENERGY)


def chord_spec(positions, seed, offsets, density=0.6, h_sigma=0.4):
    """A layer that stresses every class of far edge of the layered kernel: the +/-1, +/-2 ring plus
    chords at the given offsets (short ones land inside the columns a chunk has already loaded, medium
    ones in the next chunk's, long and backward ones are the far warp's), several per position and
    often several into the same target within one chunk; couplings are not powers of two."""
    rng = ins.MT19937(seed)
    present, far_deg, edges = set(), [0] * positions, []

    def add(a, b, far):
        key = (min(a, b), max(a, b))
        if a == b or key in present or (far and (far_deg[a] >= 12 or far_deg[b] >= 12)):
            return
        present.add(key)
        if far:
            far_deg[a] += 1
            far_deg[b] += 1
        edges.append(key)

    for off in (1, 2):
        if positions > 2 * off:
            for p in range(positions):
                add(p, (p + off) % positions, False)
    for p in range(positions):
        for off in offsets:
            if off < positions and rng.below(1000) < int(1000 * density):
                add(p, (p + off) % positions, min(off, positions - off) > 2)
    values = np.array([0.75, -1.25, 1.0, -0.5, 0.3, -0.7], np.float32)
    coup = [float(values[rng.below(len(values))]) for _ in edges]
    h = rng.normals(positions, h_sigma)
    return positions, h, [(a, b, c) for (a, b), c in zip(edges, coup)]


@pytest.mark.parametrize("positions,layers,offsets", [
    (8, 4, (3, 4)), (16, 4, (3, 5, 7)), (24, 5, (3, 4, 9, 11)), (64, 4, (3, 5, 6, 9, 13, 17, 26, 31)),
    (128, 4, (3, 7, 10, 12, 19, 40, 63)), (512, 4, (3, 4, 5, 8, 11, 16, 23, 100, 255)),
])
@pytest.mark.parametrize("exp_kind", [1, 2, 3])
def test_layered_chord_graphs_every_edge_class(lib, port, positions, layers, offsets, exp_kind):
    csr = ins.build_layered_csr(*chord_spec(positions, 100 + positions, offsets), layers, 0.8)
    betas = ins.geometric_betas(0.25, 2.0, 5)
    ladders = 9  # 45 chains: two tiles, the second ragged
    sweeps = 12 if positions < 512 else 6
    out = {}
    for kernel in LAYERED_KERNELS:
        if kernel == ib.KERNEL_STRAND and positions < 16:
            continue  # the strand family wants two chunks of 8 positions at least
        state, want = run_both(port, [csr], ladders, betas, sweeps, 3, tau_scale=1.25, exp_kind=exp_kind,
                               kernel=kernel, chunks=[sweeps // 2, sweeps - sweeps // 2])
        assert state.info()["kernel"] == kernel
        assert_batch_matches(state, want, REL_ENERGY)
        for c in (0, 44):
            hs, ht = state.fields(c)
            out.setdefault(c, []).append((hs.copy(), ht.copy()))
        state.close()
    for c, per_family in out.items():  # all families leave identical fields behind, bit for bit
        for other in per_family[1:]:
            np.testing.assert_array_equal(per_family[0][0].view(np.uint32), other[0].view(np.uint32))
            np.testing.assert_array_equal(per_family[0][1].view(np.uint32), other[1].view(np.uint32))


@pytest.mark.parametrize("kernel", LAYERED_KERNELS)
def test_wait_statistics_from_real_ballots(lib, port, kernel):
    """probability that a group of w neighbouring lanes (chains attempting the same spin
    in lockstep) holds at least one flip, measured on the warp's ballots, against the same quantity
    computed from the oracle's per-sweep flip flags (ref: accumulate_group_flags, sweep_state.cpp:356-372,
    with the group taken across chains instead of along one chain)."""
    csr = ins.build_layered_csr(*ins.layered_spec(16, 5), 4, 1.5)  # 64 spins
    betas = ins.geometric_betas(0.3, 2.0, 4)
    ladders, sweeps = 24, 9  # 96 chains = 3 full tiles
    seeds = (ins.CHAIN_SEED_BASE + np.arange(ladders * betas.size)).astype(np.uint32)
    with ib.init_state(product_model(csr), betas, ladders, seeds=seeds, kernel=kernel) as st:
        with pytest.raises(ib.IsingError, match="not recorded"):
            st.wait_stats()
        st.run(2)                      # not recorded
        st.record_wait(True)
        st.run(4)
        st.run(sweeps - 4)
        got = st.wait_stats()
        flips_recorded = st.stats()[0].sum()
        with pytest.raises(ib.IsingError, match="width 3 was not recorded"):
            st.wait_stats([3])
    # oracle: every chain on its own, a flip flag per (sweep, spin) = the spin changed in that sweep
    model = port.model(csr)
    n = csr["n_spins"]
    flags = np.zeros((sweeps, n, ladders * betas.size), bool)
    flips_before = 0
    for c in range(ladders * betas.size):
        chain = port.chain(model, int(seeds[c]), float(betas[c % betas.size]), 1.0, 2, None)
        chain.sweep(2)
        flips_before += chain.flips
        prev = chain.spins
        for s in range(sweeps):
            chain.sweep(1)
            cur = chain.spins
            flags[s, :, c] = cur != prev
            prev = cur
    for w in (1, 2, 4, 8, 16, 32):
        grouped = flags.reshape(sweeps, n, -1, w).any(axis=3)
        prob, groups, with_flip = got[w]
        assert groups == grouped.size and with_flip == int(grouped.sum())
        assert prob == pytest.approx(grouped.mean())
    assert got[1][2] == int(flags.sum()) == int(flips_recorded) - flips_before
    assert got[32][0] >= got[16][0] >= got[1][0]  # wider groups wait more often


def test_one_shot_run_json_has_the_reference_report_keys(lib, port, tmp_path):
    """model file -> device run -> JSON report with the keys of ising_run_json
    (ref: proj/src/capi.cpp:230-262)."""
    import json
    csr = ins.build_layered_csr(*ins.layered_spec(16, 9), 4, 1.5)
    path = tmp_path / "model.ising"
    product_model(csr).save(path)
    model = ib.SpinModel.load(path)
    report, text = ib.run_single_json(model, 25, 0.7, 4321, tau_scale=1.25, exp_kind=ib.ExpKind.fast)
    doc = json.loads(text)
    assert set(doc) == {"engine", "exp", "spins", "sweeps", "beta", "tau_scale", "seed", "workers", "final_cost",
                        "flip_rate", "flips", "attempts", "wait", "checksum", "environment"}
    chain = port.chain(port.model(csr), 4321, 0.7, 1.25, 2, None)
    chain.sweep(25)
    assert doc["flips"] == report["flips"] == chain.flips and doc["attempts"] == 25 * 64
    assert doc["checksum"] == f"{report['checksum']:016x}" == f"{port.checksum(chain.spins):016x}"
    assert doc["final_cost"] == report["final_cost"]  # shortest round-trip decimal: same double
    assert doc["final_cost"] == pytest.approx(port.total_cost(port.model(csr), chain.spins), rel=REL_ENERGY)
    assert doc["flip_rate"] == report["flips"] / report["attempts"]
    head = (doc["engine"], doc["exp"], doc["spins"], doc["sweeps"], doc["seed"], doc["workers"])
    assert head == ("b200-strand", "fast", 64, 25, 4321, 1)
    assert doc["beta"] == float(np.float32(0.7)) and doc["tau_scale"] == 1.25 and doc["wait"] == {}
    assert "device=" in doc["environment"]


def _with_coupling(csr, spin, slot, value):
    """The same graph with the coupling of `spin`'s `slot`-th edge (both directions) replaced."""
    out = dict(csr)
    out["couplings"] = csr["couplings"].copy()
    e = int(csr["offsets"][spin]) + slot
    t = int(csr["targets"][e])
    out["couplings"][e] = value
    back = [k for k in range(int(csr["offsets"][t]), int(csr["offsets"][t + 1])) if int(csr["targets"][k]) == spin]
    out["couplings"][back[0]] = value
    return out


def test_generic_family_update_variants(lib, port):
    """The generic family's three ways of applying a flip's updates land on the same bits as the oracle:
    f32 reductions with the own-field window (the default), reductions without it (a model whose window
    is unusable: an in-chunk tau edge), and read-modify-write (a coupling so small that a field could be
    subnormal, which a reduction would flush)."""
    betas = ins.geometric_betas(0.2, 3.0, 8)
    base = ins.cubic_mixed_degree(8, ins.INSTANCE_SEED + 40)
    state, want = run_both(port, [base], 6, betas, 80, 1, kernel=ib.KERNEL_GENERIC)
    assert state.info()["generic_variant"] == 2
    assert_batch_matches(state, want, REL_ENERGY)

    # four positions per layer: the tau partner of spin i is i + 4, inside i's chunk of eight attempts
    narrow = ins.build_layered_csr(*ins.layered_spec(4, 77), 6, 1.25)
    state, want = run_both(port, [narrow], 40, [0.7], 100, 0, tau_scale=0.75, kernel=ib.KERNEL_GENERIC)
    assert state.info()["generic_variant"] == 1
    assert_batch_matches(state, want, REL_ENERGY)

    # a subnormal coupling: fields of the two spins it joins carry subnormal parts
    tiny = _with_coupling(base, 5, 0, np.float32(3e-39))
    state, want = run_both(port, [tiny, base], 2, betas, 80, 1, kernel=ib.KERNEL_GENERIC)
    assert state.info()["generic_variant"] == 0
    assert_batch_matches(state, want, REL_ENERGY)


@pytest.mark.parametrize("exp_kind", [1, 2, 3])
def test_generic_family_high_degree_ragged_and_repeated_edges(lib, port, exp_kind):
    """Degrees up to ~20 (the split kernel's tail past eight edges), n = 77 (a last chunk of five
    attempts), ragged tiles, and a second model with repeated edges (own-field window unusable)."""
    plain = random_graph(77, 11, 901)
    assert int(np.diff(plain["offsets"]).max()) > 12
    repeated = random_graph(77, 9, 902, repeats=12)
    betas = ins.geometric_betas(0.15, 2.5, 11)
    state, want = run_both(port, [plain, repeated], 7, betas, 150, 1, exp_kind=exp_kind, kernel=ib.KERNEL_GENERIC,
                           model_of_ladder=[0, 1, 0, 1, 1, 0, 0])
    assert state.info()["generic_variant"] == 1  # reductions; the second model has no window
    assert_batch_matches(state, want, REL_ENERGY)
    state, want = run_both(port, [plain], 3, betas, 150, 2, exp_kind=exp_kind, kernel=ib.KERNEL_GENERIC)
    assert state.info()["generic_variant"] == 2
    assert_batch_matches(state, want, REL_ENERGY)


def test_results_all_gather_through_the_c_entry(lib):
    """ising_batch_all_gather_results: the data path's only collective behind the C ABI, for callers
    without torch.  One rank here (the run has one GPU): a 1-rank NCCL communicator made with NCCL's own
    C API, the gathered records against ising_batch_pack_results and the host readouts."""
    import ctypes as C
    import torch
    torch.cuda.set_device(0)
    nccl = C.CDLL("libnccl.so.2")  # the copy torch has loaded: the library looks it up the same way

    class UniqueId(C.Structure):
        _fields_ = [("internal", C.c_char * 128)]

    nccl.ncclCommInitRank.argtypes = [C.POINTER(C.c_void_p), C.c_int, UniqueId, C.c_int]
    nccl.ncclCommDestroy.argtypes = [C.c_void_p]
    uid, comm = UniqueId(), C.c_void_p()
    assert nccl.ncclGetUniqueId(C.byref(uid)) == 0
    assert nccl.ncclCommInitRank(C.byref(comm), 1, uid, 0) == 0
    try:
        csr = ins.build_layered_csr(*ins.layered_spec(32, 3), 8, 1.5)
        betas = ins.geometric_betas(0.3, 2.0, 4)
        with ib.init_state(product_model(csr), betas, 10, base_seed=5, swap_base_seed=6) as st:
            st.run(12, 3)
            chains = st.n_chains
            gathered = torch.zeros((chains, 4), dtype=torch.int64, device="cuda")
            packed = torch.zeros((chains, 4), dtype=torch.int64, device="cuda")
            st.all_gather_results(comm.value, gathered.data_ptr())
            st.pack_results(packed.data_ptr())
            torch.cuda.synchronize()
            rec = gathered.cpu().numpy()
            np.testing.assert_array_equal(rec, packed.cpu().numpy())
            np.testing.assert_array_equal(rec[:, 0].view(np.float64), st.energies())
            np.testing.assert_array_equal(rec[:, 2].view(np.uint64), st.stats()[0])
            np.testing.assert_array_equal(rec[:, 3].view(np.uint64), st.checksums())
    finally:
        nccl.ncclCommDestroy(comm)


@pytest.mark.parametrize("gamma", [1.0, 0.7])
def test_resync_energies_sets_the_tempering_cost(lib, port, gamma):
    """ising_batch_resync_energies: running energy := orc_tempering_cost of the current spins, in every
    family."""
    positions, h, edges = ins.layered_spec(16, 31)
    csr = ins.build_layered_csr(positions, h, edges, 8, 0.75)
    omodel = port.model(csr)
    betas = ins.geometric_betas(0.3, 1.2, 3)
    for family in LAYERED_KERNELS:
        with ib.init_state(product_model(csr), betas, 11, base_seed=77, params=ib.SweepParams(gamma, 2),
                           kernel=family) as st:
            st.run(40, 4)
            drifted = st.running_energies()
            st.resync_energies()
            fresh = st.running_energies()
            spins = st.spins(0, st.n_chains)
            want = np.array([port.tempering_cost(omodel, s, gamma) for s in spins])
            np.testing.assert_array_equal(fresh, want)
            np.testing.assert_allclose(drifted, want, rtol=REL_ENERGY, atol=1e-4)
            if gamma == 1.0:
                np.testing.assert_array_equal(fresh, st.energies())
            # the next sweeps add their flip energies to the resynchronised value
            st.run(3, 0)
            after = np.array([port.tempering_cost(omodel, s, gamma) for s in st.spins(0, st.n_chains)])
            np.testing.assert_allclose(st.running_energies(), after, rtol=REL_ENERGY, atol=1e-4)


@pytest.mark.parametrize("kernel", LAYERED_KERNELS)
def test_layered_families_keep_subnormal_field_parts(lib, port, kernel):
    """A far and a band coupling in the subnormal range (3e-39, 7e-40): such a model is not
    `reduction_safe` (a global f32 reduction flushes subnormals), so every family must apply its updates
    as plain f32 additions.  The strand family pulls far updates into registers and needs no special case."""
    positions, h, edges = ins.layered_spec(32, 4242)
    edges = [e for e in edges if {e[0], e[1]} != {3, 20} and {e[0], e[1]} != {9, 10}]
    edges += [(3, 20, float(np.float32(3e-39))), (9, 10, float(np.float32(7e-40)))]
    csr = ins.build_layered_csr(positions, h, edges, 4, 0.9)
    betas = ins.geometric_betas(0.3, 2.5, 6)
    state, want = run_both(port, [csr], 6, betas, 60, 2, kernel=kernel, chunks=[25, 35])
    assert state.info()["kernel"] == kernel
    assert_batch_matches(state, want, REL_ENERGY)
    state.close()


def test_strand_family_many_tiles_of_alternating_models(lib, port):
    """More tiles than SMs and two models alternating ladder by ladder (a tile never mixes models, so
    every ladder is a tile of its own): the strand family then reads graph and cells from global memory
    instead of staging them per CTA — the one launch variant the smaller multi-model tests do not reach."""
    a = ins.build_layered_csr(*ins.layered_spec(16, 501), 4, 1.25)
    b = ins.build_layered_csr(*chord_spec(16, 502, (3, 5, 7)), 4, 0.8)
    ladders = 170
    betas = ins.geometric_betas(0.3, 2.0, 3)
    state, want = run_both(port, [a, b], ladders, betas, 24, 3, kernel=ib.KERNEL_STRAND,
                           model_of_ladder=[k % 2 for k in range(ladders)], chunks=[10, 14])
    info = state.info()
    assert info["kernel"] == ib.KERNEL_STRAND and info["n_tiles"] == ladders
    assert_batch_matches(state, want, REL_ENERGY)
    state.close()


def test_strand_family_more_tiles_than_one_round_holds(lib, port):
    """1,600 tiles of one small model: with one strand and one producer per tile only 1,480 tiles are
    resident at once on 148 SMs, so the launch sweeps them in two rounds of 800 (every warp of a round
    must be resident: the rounds are sized by the launcher)."""
    csr = ins.build_layered_csr(*ins.layered_spec(16, 733), 4, 1.0)
    betas = ins.geometric_betas(0.4, 1.6, 4)
    ladders = 1600 * 8  # 32 chains per tile
    state, want = run_both(port, [csr], ladders, betas, 12, 4, kernel=ib.KERNEL_STRAND, chunks=[5, 7])
    info = state.info()
    assert info["n_tiles"] == 1600 and info["strands"] == 1
    assert_batch_matches(state, want, REL_ENERGY)
    state.close()
