"""BASELINE.json's full-size configurations on the GPU, checked through size-independent
properties (the oracle cannot finish them): agreement of the kernel families, the running
energy against the recomputed energy, determinism (a checksum of checksums), shard invariance,
bit parity with the oracle on a subsample of ladders inside the full batch for the FULL run
length of every configuration, and all 16,384 chains of config 5 against a record the reference
itself produced (tests/golden/make_golden_c5.py)."""
import os

import numpy as np
import pytest

import paper_1004_0024_b200 as ib
from paper_1004_0024_b200 import sharding, workloads
from helpers import assert_batch_matches, ins, oracle_batch, product_model, random_graph

pytestmark = pytest.mark.gpu


FAMILIES = (ib.KERNEL_STRAND, ib.KERNEL_LAYERED, ib.KERNEL_GENERIC)  # identical-layer models: all three


def fold(values) -> int:
    """Order-sensitive checksum of checksums (FNV-1a over the 64-bit words)."""
    h = 1469598103934665603
    for v in np.asarray(values, np.uint64).tolist():
        h = ((h ^ v) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


@pytest.fixture(scope="module")
def c5():
    wl = workloads.get("c5")
    return wl, wl.make_csrs()[0]


def test_c5_full_batch_properties_and_subsample_parity(lib, port, c5):
    """16,384 chains x 32,768 spins (config 5), 20 sweeps with a swap round every 10."""
    wl, csr = c5
    model = product_model(csr)
    sweeps = 20
    with ib.init_state(model, wl.betas, wl.n_ladders, base_seed=ins.CHAIN_SEED_BASE,
                       swap_base_seed=ins.SWAP_SEED_BASE) as st:
        info = st.info()
        assert info["kernel"] == ib.KERNEL_STRAND and info["n_chains"] == 16384 and info["n_tiles"] == 512
        e0 = st.energies()
        np.testing.assert_array_equal(st.running_energies(), e0)  # initial running energy == total_cost
        st.run(sweeps, wl.swap_interval)
        energies, e_run = st.energies(), st.running_energies()
        flips, attempts = st.stats()
        sums, slots = st.checksums(), st.slots()
        coherence = st.field_coherence_ulp()
        sample = st.spins(16 * 1000, 32)  # ladders 1000 and 1001, deep inside the batch
    assert (attempts == sweeps * 32768).all()
    # energies within 1e-5 relative of the f32-accumulated running energy (north_star tolerance)
    np.testing.assert_allclose(e_run, energies, rtol=1e-5)
    assert (energies < e0).mean() > 0.9  # cold and warm chains relax from the random start
    rate = flips.reshape(-1, 16).mean(0) / attempts[0]
    assert rate[0] > 0.3 and rate[-1] < 0.1  # hot end flips often, cold end rarely (slots barely move in 2 rounds)
    assert (np.sort(slots.reshape(-1, 16), 1) == np.arange(16)).all()
    assert coherence.max() <= 4096  # incremental fields stay a few ULP of a recompute away (near-zero fields inflate ULPs)
    # bit parity of a subsample against the oracle: seeds are functions of the global chain id
    seeds = sharding.chain_seeds(ins.CHAIN_SEED_BASE, 1000, 2, 16)
    swap_seeds = sharding.ladder_seeds(ins.SWAP_SEED_BASE, 1000, 2)
    want = oracle_batch(port, [csr], 2, wl.betas, seeds, swap_seeds, sweeps, wl.swap_interval)
    np.testing.assert_array_equal(sample, want["spins"])
    np.testing.assert_array_equal(flips[16000:16032], want["flips"])
    np.testing.assert_array_equal(e_run[16000:16032].view(np.uint64), want["e_run"].view(np.uint64))
    np.testing.assert_array_equal(slots[16000:16032], want["slot"])
    # determinism: a second run gives the same checksum of checksums
    with ib.init_state(model, wl.betas, wl.n_ladders, base_seed=ins.CHAIN_SEED_BASE,
                       swap_base_seed=ins.SWAP_SEED_BASE) as again:
        again.run(sweeps, wl.swap_interval)
        assert fold(again.checksums()) == fold(sums)


def test_c5_shards_reproduce_the_full_batch(lib, c5):
    """Weak-scaling property: a shard addressed by first_ladder carries the same bits as the
    corresponding slice of a larger batch (what makes 1/2/4/8-GPU results identical)."""
    wl, csr = c5
    model = product_model(csr)
    with ib.init_state(model, wl.betas, 192, base_seed=5, swap_base_seed=6) as whole:
        whole.run(10, 5)
        sums, slots = whole.checksums(), whole.slots()
    for rank in range(3):
        first, count = sharding.shard_ladders(192, rank, 3)
        with ib.init_state(model, wl.betas, count, base_seed=5, swap_base_seed=6, first_ladder=first) as part:
            part.run(10, 5)
            np.testing.assert_array_equal(part.checksums(), sums[first * 16:(first + count) * 16])
            np.testing.assert_array_equal(part.slots(), slots[first * 16:(first + count) * 16])


def test_c4_kernel_families_agree_on_distinct_instances(lib):
    """Config 4 shape (32 betas, one instance per ladder, swap every sweep): the on-chip layered
    kernel and the generic HBM kernel must produce identical chains."""
    wl = workloads.get("c4")
    csrs = [ins.build_layered_csr(*ins.layered_spec(512, ins.INSTANCE_SEED + k, 0.5, 6), 64, 1.5) for k in range(3)]
    models = [product_model(c) for c in csrs]
    out = {}
    for family in FAMILIES:
        with ib.init_state(models, wl.betas, 3, base_seed=11, swap_base_seed=12, kernel=family) as st:
            assert st.info()["kernel"] == family
            st.run(6, 1)
            out[family] = (st.checksums(), st.stats()[0], st.slots(), st.running_energies(), st.energies())
    for family in FAMILIES[1:]:
        for a, b in zip(out[FAMILIES[0]], out[family]):
            np.testing.assert_array_equal(a, b)
    assert out[ib.KERNEL_LAYERED][1].sum() > 0


def test_c3_full_width_ladder_subsample(lib, port):
    """Config 3 shape at full ladder width (32 betas, swap every sweep) on a few distinct graphs."""
    wl = workloads.get("c3")
    csrs = [ins.cubic_mixed_degree(16, ins.INSTANCE_SEED + k) for k in range(2)]
    seeds = sharding.chain_seeds(ins.CHAIN_SEED_BASE, 0, 2, 32)
    swap_seeds = sharding.ladder_seeds(ins.SWAP_SEED_BASE, 0, 2)
    want = oracle_batch(port, csrs, 2, wl.betas, seeds, swap_seeds, 60, 1)
    with ib.init_state([product_model(c) for c in csrs], wl.betas, 2, base_seed=ins.CHAIN_SEED_BASE,
                       swap_base_seed=ins.SWAP_SEED_BASE) as st:
        st.run(60, 1)
        np.testing.assert_array_equal(st.spins(), want["spins"])
        np.testing.assert_array_equal(st.stats()[0], want["flips"])
        np.testing.assert_array_equal(st.slots(), want["slot"])
        np.testing.assert_allclose(st.energies(), want["energy"], rtol=1e-5)


def test_layer_width_not_multiple_of_8_uses_generic_family(lib, port):
    csr = ins.build_layered_csr(*ins.layered_spec(12, 9), 5, 1.5)
    seeds = np.arange(10, 14, dtype=np.uint32)
    want = oracle_batch(port, [csr], 1, [0.3, 0.6, 1.2, 2.4], seeds, [3], 40, 2)
    with ib.init_state(product_model(csr), [0.3, 0.6, 1.2, 2.4], 1, seeds=seeds, swap_seeds=[3]) as st:
        assert st.info()["kernel"] == ib.KERNEL_GENERIC
        st.run(40, 2)
        np.testing.assert_array_equal(st.spins(), want["spins"])
    with pytest.raises(ib.IsingError):
        ib.init_state(product_model(csr), [1.0], 1, kernel=ib.KERNEL_LAYERED)


def test_more_tiles_than_warp_slots_each_pair_sweeps_several_tiles(lib, port):
    """700 tiles on 148 x 4 tile slots: every (sweep, producer, post, far) warp group walks more
    than one tile in a launch, across several launches.  Both families must agree everywhere and a
    subsample must match the oracle."""
    csr = ins.build_layered_csr(*ins.layered_spec(24, 17), 4, 1.5)
    model = product_model(csr)
    betas = ins.geometric_betas(0.3, 2.5, 4)
    ladders = 700 * 8  # 22,400 chains = 700 tiles
    out = {}
    for family in FAMILIES:
        with ib.init_state(model, betas, ladders, base_seed=31, swap_base_seed=32, kernel=family) as st:
            assert st.info()["n_tiles"] == 700 and st.info()["kernel"] == family
            st.run(7, 3)
            st.run(5, 3)
            out[family] = (st.checksums(), st.stats()[0], st.slots(), st.running_energies())
            if family == ib.KERNEL_LAYERED:
                sample = st.spins(4 * 5000, 8)  # ladders 5000, 5001: tile 625, in the second round of its pair
    for family in FAMILIES[1:]:
        for a, b in zip(out[FAMILIES[0]], out[family]):
            np.testing.assert_array_equal(a, b)
    want = oracle_batch(port, [csr], 2, betas, sharding.chain_seeds(31, 5000, 2, 4),
                        sharding.ladder_seeds(32, 5000, 2), 12, 3)
    np.testing.assert_array_equal(sample, want["spins"])


@pytest.mark.parametrize("seed", range(int(os.environ.get("ISING_FUZZ_SEEDS", "12"))))
def test_random_layer_graphs_all_families_bit_identical(lib, seed):
    """Seeded fuzz of the layered and strand kernels' edge classification (band / near in the loaded
    columns / near in the next chunk's / far, group splitting on repeated targets, padding): random
    layer graphs with chords at random distances, all kernel families must leave identical spins, flip
    counts, slots, running energies and FIELDS (bit for bit) behind."""
    rng = np.random.default_rng(1000 + seed)
    positions = int(rng.choice([8, 16, 24, 40, 64, 104, 160, 256, 512]))
    layers = int(rng.integers(4, 8))
    present, far_deg, edges = set(), [0] * positions, []
    for off in (1, 2):
        if positions > 2 * off:
            for p in range(positions):
                key = (min(p, (p + off) % positions), max(p, (p + off) % positions))
                if key not in present and key[0] != key[1]:
                    present.add(key)
                    edges.append(key)
    scale = int(rng.choice([4, 12, 40, positions]))
    for _ in range(int(positions * rng.uniform(0.3, 2.5))):
        a = int(rng.integers(0, positions))
        b = (a + int(rng.integers(3, max(4, min(scale, positions - 2))))) % positions
        key = (min(a, b), max(a, b))
        index_distance = key[1] - key[0]
        if key[0] == key[1] or key in present or index_distance <= 2:
            continue
        if far_deg[key[0]] >= 13 or far_deg[key[1]] >= 13:
            continue
        present.add(key)
        far_deg[key[0]] += 1
        far_deg[key[1]] += 1
        edges.append(key)
    couplings = rng.choice(np.array([1.0, -1.0, 0.5, -0.75, 0.3, -1.3], np.float32), size=len(edges))
    h = rng.normal(0.0, 0.4, positions).astype(np.float32)
    csr = ins.build_layered_csr(positions, h, [(a, b, float(j)) for (a, b), j in zip(edges, couplings)], layers,
                                float(rng.choice([0.5, 1.0, 1.5])))
    model = product_model(csr)
    betas = ins.geometric_betas(0.2, 3.0, int(rng.integers(2, 7)))
    ladders = int(rng.integers(3, 20))
    sweeps, interval = int(rng.integers(4, 12)), int(rng.integers(1, 4))
    gamma = float(rng.choice([1.0, 1.25]))
    chain = int(rng.integers(0, ladders * betas.size))
    first = None
    for family in (ib.KERNEL_LAYERED, ib.KERNEL_GENERIC, ib.KERNEL_STRAND):
        if family == ib.KERNEL_STRAND and positions < 16:
            continue  # the strand family wants two chunks of 8 positions at least
        with ib.init_state(model, betas, ladders, base_seed=7 + seed, swap_base_seed=99 + seed, kernel=family,
                           params=ib.SweepParams(gamma, 2)) as st:
            assert st.info()["kernel"] == family
            st.run(sweeps, interval)
            st.run(3, interval)
            hs, ht = st.fields(chain)
            got = (st.spins(), st.stats()[0], st.slots(), st.running_energies().view(np.uint64),
                   hs.view(np.uint32), ht.view(np.uint32))
        if first is None:
            first = got
        else:
            for a, b in zip(first, got):
                np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("seed", range(int(os.environ.get("ISING_FUZZ_SEEDS", "12"))))
def test_random_multigraphs_generic_family_matches_the_oracle(lib, port, seed):
    """Seeded fuzz of the generic family against the oracle: random multigraphs (sizes off the chunk
    grid, degrees from sparse to ~25, repeated edges, zero fields, now and then a subnormal coupling
    that sends the batch through the read-modify-write kernel), random ladders, all exp kinds."""
    rng = np.random.default_rng(5000 + seed)
    n = int(rng.choice([5, 8, 9, 31, 64, 77, 130, 257]))
    n_models = int(rng.integers(1, 4))
    csrs = []
    for k in range(n_models):
        degree = int(rng.integers(2, min(15, n - 1)))
        g = random_graph(n, degree, 7000 + 10 * seed + k, repeats=int(rng.choice([0, 0, 6])))
        if rng.random() < 0.3:
            g["h"] = np.zeros(n, np.float32)
        csrs.append(g)
    tiny = rng.random() < 0.25
    if tiny:
        g = csrs[0]
        e = int(rng.integers(0, g["targets"].size))
        a = int(np.searchsorted(g["offsets"], e, side="right") - 1)
        t = int(g["targets"][e])
        value = np.float32(2e-39)
        g["couplings"] = g["couplings"].copy()
        for x, y in ((a, t), (t, a)):  # every copy of the edge, both directions
            lo, hi = int(g["offsets"][x]), int(g["offsets"][x + 1])
            hit = lo + np.flatnonzero(g["targets"][lo:hi] == y)
            g["couplings"][hit] = value
    betas = ins.geometric_betas(0.1, 3.0, int(rng.integers(1, 9)))
    ladders = int(rng.integers(1, 12))
    model_of_ladder = [int(v) for v in rng.integers(0, n_models, ladders)]
    used = sorted(set(model_of_ladder))
    csrs = [csrs[k] for k in used]
    model_of_ladder = [used.index(k) for k in model_of_ladder]
    chains = ladders * betas.size
    seeds = (31 * seed + 1 + np.arange(chains)).astype(np.uint32)
    swap_seeds = (17 * seed + 5 + np.arange(ladders)).astype(np.uint32)
    sweeps, interval = int(rng.integers(20, 60)), int(rng.integers(0, 4))
    exp_kind = int(rng.integers(1, 4))
    want = oracle_batch(port, csrs, ladders, betas, seeds, swap_seeds, sweeps, interval, 1.0, exp_kind, model_of_ladder)
    with ib.init_state([product_model(c) for c in csrs], betas, ladders, seeds=seeds, swap_seeds=swap_seeds,
                       params=ib.SweepParams(1.0, exp_kind), model_of_ladder=model_of_ladder,
                       kernel=ib.KERNEL_GENERIC) as st:
        if tiny and 0 in used:
            assert st.info()["generic_variant"] == 0
        split = int(rng.integers(1, sweeps))
        st.run(split, interval)
        st.run(sweeps - split, interval)
        assert_batch_matches(st, want, 1e-5)


# ---- full-length runs ("bit parity on a subset for the full run") -----------------

def test_c5_full_length_two_ladders_inside_the_batch_and_family_soak(lib, port, c5):
    """Config 5 for its full 1,000 sweeps (swap every 10) on all 16,384 chains: ladders 1000 and 1001,
    deep inside the batch, bit for bit against the oracle; and every chain of the batch identical
    under the strand and the Tensor Memory families (checksum, accept count, slot, running energy,
    swap counts) — the long run crosses every MT19937 wrap, careful chunk and tape-ring wrap."""
    wl, csr = c5
    model = product_model(csr)
    out = {}
    for family in (ib.KERNEL_STRAND, ib.KERNEL_LAYERED):
        with ib.init_state(model, wl.betas, wl.n_ladders, base_seed=ins.CHAIN_SEED_BASE,
                           swap_base_seed=ins.SWAP_SEED_BASE, kernel=family) as st:
            st.run(wl.sweeps, wl.swap_interval)
            out[family] = (st.checksums(), st.stats()[0], st.slots(), st.running_energies().view(np.uint64),
                           st.swap_stats()[0])
            if family == ib.KERNEL_STRAND:
                sample, energies = st.spins(16 * 1000, 32), st.energies()
                e_run = st.running_energies()
    for a, b in zip(out[ib.KERNEL_STRAND], out[ib.KERNEL_LAYERED]):
        np.testing.assert_array_equal(a, b)
    # the running energy stays within f32-rounding distance of the exact energy over ~2e9 flips a chain
    np.testing.assert_allclose(e_run, energies, rtol=1e-5)
    seeds = sharding.chain_seeds(ins.CHAIN_SEED_BASE, 1000, 2, 16)
    swap_seeds = sharding.ladder_seeds(ins.SWAP_SEED_BASE, 1000, 2)
    want = oracle_batch(port, [csr], 2, wl.betas, seeds, swap_seeds, wl.sweeps, wl.swap_interval, threads=2)
    checks, flips, slots, e_bits, _ = out[ib.KERNEL_STRAND]
    np.testing.assert_array_equal(sample, want["spins"])
    np.testing.assert_array_equal(flips[16000:16032], want["flips"])
    np.testing.assert_array_equal(slots[16000:16032], want["slot"])
    np.testing.assert_array_equal(e_bits[16000:16032], want["e_run"].view(np.uint64))


def test_c5_all_chains_first_100_sweeps_against_the_reference_record(lib, golden):
    """Every one of the 16,384 chains of config 5, 100 sweeps without swaps, against accept counts and
    final total_cost the REFERENCE produced (tests/golden/make_golden_c5.py -> oracle/_ref): a checksum
    of checksums over the batch, one per tile to localise a failure, and 64 chains verbatim."""
    g = golden("c5_first100")
    wl = workloads.get("c5")
    csr = wl.make_csrs()[0]
    with ib.init_state(product_model(csr), wl.betas, wl.n_ladders, base_seed=ins.CHAIN_SEED_BASE,
                       swap_base_seed=ins.SWAP_SEED_BASE) as st:
        assert st.info()["n_chains"] == int(g["chains"])
        st.run(int(g["sweeps"]), 0)
        flips, energy = st.stats()[0], st.energies()
    np.testing.assert_array_equal(flips[:64], g["flips_head"])
    np.testing.assert_array_equal(energy[:64].view(np.uint64), g["energy_head"].view(np.uint64))
    tiles = flips.size // 32
    got_f = np.array([fold(flips[32 * t:32 * t + 32]) for t in range(tiles)], np.uint64)
    got_e = np.array([fold(energy[32 * t:32 * t + 32].view(np.uint64)) for t in range(tiles)], np.uint64)
    bad = np.nonzero((got_f != g["tile_flips_fold"]) | (got_e != g["tile_energy_fold"]))[0]
    assert bad.size == 0, f"tiles differing from the reference record: {bad[:10].tolist()}"
    assert fold(flips) == int(g["flips_fold"]) and fold(energy.view(np.uint64)) == int(g["energy_fold"])


def test_c2_full_length_replicas_inside_the_batch(lib, port):
    """Config 2: 1,024 replicas of the 16^3 lattice with Gaussian fields for the full 10,000 sweeps;
    replicas 480..511 (one tile in the middle) bit for bit against the oracle."""
    wl = workloads.get("c2")
    csr = wl.make_csrs()[0]
    with ib.init_state(product_model(csr), wl.betas, wl.n_ladders, base_seed=ins.CHAIN_SEED_BASE,
                       swap_base_seed=ins.SWAP_SEED_BASE) as st:
        st.run(wl.sweeps, 0)
        sample, flips, energies = st.spins(480, 32), st.stats()[0], st.energies()
    seeds = sharding.chain_seeds(ins.CHAIN_SEED_BASE, 480, 32, 1)
    want = oracle_batch(port, [csr], 32, wl.betas, seeds, sharding.ladder_seeds(ins.SWAP_SEED_BASE, 480, 32),
                        wl.sweeps, 0, threads=16)
    np.testing.assert_array_equal(sample, want["spins"])
    np.testing.assert_array_equal(flips[480:512], want["flips"])
    np.testing.assert_allclose(energies[480:512], want["energy"], rtol=1e-5)


def test_c3_full_length_one_ladder_inside_distinct_graphs(lib, port):
    """Config 3: 32 betas, swap every sweep, distinct mixed-degree graphs, the full 10,000 sweeps; ladder
    5 of a 12-system batch bit for bit against the oracle (spins, accept counts, slots, running energies)."""
    wl = workloads.get("c3")
    systems = 12
    csrs = [ins.cubic_mixed_degree(16, ins.INSTANCE_SEED + k) for k in range(systems)]
    with ib.init_state([product_model(c) for c in csrs], wl.betas, systems, base_seed=ins.CHAIN_SEED_BASE,
                       swap_base_seed=ins.SWAP_SEED_BASE) as st:
        st.run(wl.sweeps, wl.swap_interval)
        sample = st.spins(5 * 32, 32)
        flips, slots, e_run = st.stats()[0], st.slots(), st.running_energies()
    want = oracle_batch(port, [csrs[5]], 1, wl.betas, sharding.chain_seeds(ins.CHAIN_SEED_BASE, 5, 1, 32),
                        sharding.ladder_seeds(ins.SWAP_SEED_BASE, 5, 1), wl.sweeps, wl.swap_interval)
    np.testing.assert_array_equal(sample, want["spins"])
    np.testing.assert_array_equal(flips[160:192], want["flips"])
    np.testing.assert_array_equal(slots[160:192], want["slot"])
    np.testing.assert_array_equal(e_run[160:192].view(np.uint64), want["e_run"].view(np.uint64))


def test_c4_full_length_one_system_inside_distinct_instances(lib, port):
    """Config 4: 512x64 layered instances, 32 betas, swap every sweep, the full 5,000 sweeps; system 2
    of a 4-system batch bit for bit against the oracle."""
    wl = workloads.get("c4")
    systems = 4
    csrs = [ins.build_layered_csr(*ins.layered_spec(512, ins.INSTANCE_SEED + k, 0.5, 6), 64, 1.5) for k in range(systems)]
    with ib.init_state([product_model(c) for c in csrs], wl.betas, systems, base_seed=ins.CHAIN_SEED_BASE,
                       swap_base_seed=ins.SWAP_SEED_BASE) as st:
        assert st.info()["kernel"] == ib.KERNEL_STRAND
        st.run(wl.sweeps, wl.swap_interval)
        sample = st.spins(2 * 32, 32)
        flips, slots, e_run = st.stats()[0], st.slots(), st.running_energies()
    want = oracle_batch(port, [csrs[2]], 1, wl.betas, sharding.chain_seeds(ins.CHAIN_SEED_BASE, 2, 1, 32),
                        sharding.ladder_seeds(ins.SWAP_SEED_BASE, 2, 1), wl.sweeps, wl.swap_interval)
    np.testing.assert_array_equal(sample, want["spins"])
    np.testing.assert_array_equal(flips[64:96], want["flips"])
    np.testing.assert_array_equal(slots[64:96], want["slot"])
    np.testing.assert_array_equal(e_run[64:96].view(np.uint64), want["e_run"].view(np.uint64))


def test_bench_two_gpus_when_the_box_has_them():
    """`bench.py --gpus 2` started plainly spawns its two ranks (torch.distributed.run, NCCL) and prints one
    line for the whole job.  The GPU boxes of this project have one device: skipped there."""
    import json
    import os
    import subprocess
    import sys
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("one GPU")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
                          "--ladders", "64", "--no-cpu-baseline"], capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["first_ladder_of_rank"] == [0, 64]
    assert line["gpu_launches"] > 0 and line["value"] > 0
