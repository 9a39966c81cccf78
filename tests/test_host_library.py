"""CPU-only checks of the product library: it loads, exports every symbol the header declares,
and its host-side model functions (no GPU needed) behave like the reference's
(ref: proj/tests/test_model.cpp, proj/tests/test_capi.cpp:63-76)."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1004_0024_b200 as ib
from paper_1004_0024_b200 import _lib, instances as ins
from helpers import csr_from_npz, product_model

ROOT = Path(__file__).resolve().parents[1]


def test_library_exports_every_declared_symbol(lib):
    header = (ROOT / "include" / "isingmc_b200.h").read_text()
    declared = set(re.findall(r"ISING_B200_API[^;(]*?\b(ising_\w+)\s*\(", header))
    assert len(declared) >= 28
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)
    for name in declared:
        assert hasattr(lib, name), name


def test_device_count_never_fails(lib):
    assert lib.ising_b200_device_count() >= 0


def test_layered_builder_matches_reference_golden(lib, golden):
    g = golden("layered_builder")
    edges = [(int(p), int(q), float(j)) for (p, q), j in zip(g["edges"], g["edge_j"])]
    model = ib.build_layered_model(ib.LayerSpec(int(g["positions"]), g["h"], edges), int(g["n_layers"]),
                                   float(g["j_tau"]))
    csr = model.csr()
    for key in ("h", "offsets", "targets", "couplings", "tau_counts"):
        np.testing.assert_array_equal(csr[key], g[f"csr_{key}"])
    assert model.layered == (5, 12) and model.n_spins == 60
    mine = ins.build_layered_csr(int(g["positions"]), g["h"], edges, 5, 1.5)
    np.testing.assert_array_equal(mine["targets"], csr["targets"])


def test_builder_rejections(lib):
    # ref: build_layered_model, src/model.cpp:52-75
    spec = ib.LayerSpec(4, [0, 0, 0, 0], [(0, 1, 1.0)])
    for layers, layer, text in (
        (3, spec, "need at least 4 layers"),
        (4, ib.LayerSpec(4, [0] * 4, [(0, 0, 1.0)]), "self edge"),
        (4, ib.LayerSpec(4, [0] * 4, [(0, 1, 1.0), (1, 0, 1.0)]), "duplicate"),
        (4, ib.LayerSpec(4, [0] * 4, [(0, 9, 1.0)]), "out of range"),
        (4, ib.LayerSpec(4, [0] * 3, []), "field count"),
    ):
        with pytest.raises(ib.IsingError) as err:
            ib.build_layered_model(layer, layers, 1.0)
        assert err.value.status == _lib.ISING_ERR_ARGUMENT and text in str(err.value)


def test_validate_model_rejections(lib):
    # ref: validate_model, src/model.cpp:246-281
    def make(targets, couplings, tau=None, offsets=(0, 1, 2), n=2, layers=0, per_layer=0):
        return ib.SpinModel.from_csr(n, np.zeros(n), offsets, targets, couplings, tau, layers, per_layer)

    make([1, 0], [1.0, 1.0])
    for kwargs, text in (
        (dict(targets=[1, 0], couplings=[1.0, 2.0]), "no matching reverse record"),
        (dict(targets=[0, 0], couplings=[1.0, 1.0]), "self edge"),
        (dict(targets=[5, 0], couplings=[1.0, 1.0]), "out of range"),
        (dict(targets=[1, 0], couplings=[1.0, 1.0], tau=[1, 0]), "no matching reverse record"),
        (dict(targets=[1, 0], couplings=[1.0, 1.0], tau=[2, 0]), "tau_count exceeds degree"),
        (dict(targets=[1, 0], couplings=[1.0, 1.0], layers=3, per_layer=1), "layers * per_layer"),
    ):
        with pytest.raises(ib.IsingError) as err:
            make(**kwargs)
        assert err.value.status == _lib.ISING_ERR_ARGUMENT and text in str(err.value), str(err.value)


def test_total_cost_matches_brute_force_and_golden(lib, golden):
    # ref: tests/test_model.cpp:16-29,130-138 — brute-force cost oracle
    g = golden("traj_mixed6")
    csr = csr_from_npz(g)
    model = product_model(csr)
    spins = g["k2_s7_spins"]
    assert ib.total_cost(model, spins) == float(g["k2_s7_cost"])
    n = csr["n_spins"]
    dense = np.zeros((n, n))
    for i in range(n):
        for e in range(csr["offsets"][i], csr["offsets"][i + 1]):
            dense[i, csr["targets"][e]] = csr["couplings"][e]
    s = spins.astype(np.float64)
    brute = -(csr["h"].astype(np.float64) * s).sum() - 0.5 * s @ dense @ s
    assert abs(ib.total_cost(model, spins) - brute) < 1e-9 * max(1, abs(brute))
    with pytest.raises(ib.IsingError):
        ib.total_cost(model, spins[:-1])
    bad = spins.copy()
    bad[3] = 0
    with pytest.raises(ib.IsingError) as err:
        ib.total_cost(model, bad)
    assert "not +/-1" in str(err.value)


def test_null_arguments_are_reported_not_crashed(lib):
    # ref: tests/test_capi.cpp:63-76 — status codes + thread-local message
    out = C.c_void_p()
    assert lib.ising_b200_model_from_csr(2, None, None, None, None, None, 0, 0, C.byref(out)) == _lib.ISING_ERR_ARGUMENT
    assert lib.ising_b200_last_error() == b"null argument"
    assert lib.ising_batch_run(None, 1, 0) == _lib.ISING_ERR_ARGUMENT
    assert lib.ising_batch_create(None, 0, None, None, None) == _lib.ISING_ERR_ARGUMENT
    lib.ising_batch_free(None)
    lib.ising_b200_model_free(None)


def test_batch_without_gpu_fails_loudly(lib):
    """No CPU fallback: where no CUDA device is visible, creating a batch is an error."""
    if lib.ising_b200_device_count() > 0:
        pytest.skip("a CUDA device is visible here")
    model = product_model(ins.cubic_pm1(3, 1, 0.0))
    with pytest.raises(ib.IsingError) as err:
        ib.init_state(model, [1.0], 1)
    assert err.value.status == _lib.ISING_ERR_INTERNAL and "no CPU fallback" in str(err.value)


def test_instance_generators_have_the_advertised_shapes():
    c1 = ins.cubic_pm1(16, ins.INSTANCE_SEED)
    deg = np.diff(c1["offsets"])
    assert c1["n_spins"] == 4096 and (deg == 6).all() and (c1["h"] == 0).all()
    assert set(np.unique(c1["couplings"])) == {-1.0, 1.0}
    c3 = ins.cubic_mixed_degree(8, 5)
    deg = np.diff(c3["offsets"])
    assert deg.min() >= 6 and deg.max() <= 8 and deg.mean() > 6.5
    positions, h, edges = ins.layered_spec(512, ins.INSTANCE_SEED)
    space = np.zeros(positions, int)
    for p, q, _ in edges:
        space[p] += 1
        space[q] += 1
    assert space.min() >= 4 and space.max() <= 6 and len(edges) == 2 * 512 + 256
    betas = ins.geometric_betas(0.2, 5.0, 16)
    assert betas[0] == np.float32(0.2) and betas[-1] == np.float32(5.0) and (np.diff(betas) > 0).all()


def test_committed_dram_traffic_belongs_to_the_committed_kernels():
    """bench.py reports `roofline.traffic` from profiles/sweep_traffic.json only when the capture was taken
    with the kernel sources in the tree: the c5 entry of the benchmark's kernel family must be current."""
    import json
    import os
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench
    entry = json.load(open(os.path.join(root, "profiles", "sweep_traffic.json")))["c5:3"]
    assert entry["kernel_source_hash"] == bench.kernel_source_hash()
    traffic, source = bench.profiled_traffic("c5", 3, entry["attempts_in_profiled_launch"])
    assert traffic == pytest.approx(entry["dram_bytes_read"] + entry["dram_bytes_write"], rel=1e-3) and "r02" in source
    stale, why = bench.profiled_traffic("c5", 1, 1.0)
    assert stale is None and "no ncu capture" in why
