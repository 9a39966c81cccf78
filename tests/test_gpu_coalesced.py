"""The intra-system (`coalesced`) schedule on the device against the plain-C
restatement of the reference's coalesced engine (itself pinned to the reference every sweep in
tests/test_oracle_coalesced.py): spins, both field arrays and flip counts bit for bit."""
import numpy as np
import pytest

import paper_1004_0024_b200 as ib
from paper_1004_0024_b200 import _lib
from helpers import ins, product_model

pytestmark = pytest.mark.gpu


def permuted_to_original(values, forward):
    return values[forward]


@pytest.mark.parametrize("positions,layers,exp_kind", [
    (12, 4, 2), (16, 8, 1), (24, 6, 3), (40, 64, 2), (512, 64, 2), (96, 10, 2),
])
def test_coalesced_matches_the_oracle(lib, port, positions, layers, exp_kind):
    csr = ins.build_layered_csr(*ins.layered_spec(positions, 31 + positions), layers, 1.25)
    betas = [0.4, 0.9, 2.5]
    seeds = [777, 5000, 123456]
    sweeps = 9 if positions < 512 else 4
    chains = [port.coalesced(port.model(csr), s, b, 1.5, exp_kind) for s, b in zip(seeds, betas)]
    with ib.init_coalesced(product_model(csr), betas, seeds=seeds, params=ib.SweepParams(1.5, exp_kind)) as st:
        assert st.info()["lanes"] == layers // 2
        for part in (0, 1, sweeps - 1):   # the initial state, then two launches
            if part:
                st.run(part)
                for c in chains:
                    c.sweep(part)
            for k, c in enumerate(chains):
                np.testing.assert_array_equal(st.spins(k), c.spins)
                hs, ht = st.fields(k)
                np.testing.assert_array_equal(hs.view(np.uint32), c.hs_new_order[c.forward].view(np.uint32))
                np.testing.assert_array_equal(ht.view(np.uint32), c.ht_new_order[c.forward].view(np.uint32))
            flips, attempts = st.stats()
            assert flips.tolist() == [c.flips for c in chains]
            assert attempts.tolist() == [c.attempts for c in chains]
        model = port.model(csr)
        energies, checksums = st.energies(), st.checksums()
        for k, c in enumerate(chains):
            assert energies[k] == port.total_cost(model, c.spins)
            assert int(checksums[k]) == port.checksum(c.spins)


def test_coalesced_given_initial_spins_and_default_seeds(lib, port):
    csr = ins.build_layered_csr(*ins.layered_spec(16, 3), 6, 0.75)
    n = csr["n_spins"]
    rng = np.random.default_rng(5)
    initial = (1 - 2 * rng.integers(0, 2, size=(2, n))).astype(np.int8)  # original order
    with ib.init_coalesced(product_model(csr), [0.7, 1.1], base_seed=40, initial_spins=initial) as st:
        np.testing.assert_array_equal(st.spins(1), initial[1])
        st.run(6)
        for k, beta in enumerate([0.7, 1.1]):
            probe = port.coalesced(port.model(csr), 40 + 3 * k, beta, 1.0, 2)
            ordered = np.empty(n, np.int8)
            ordered[probe.forward] = initial[k]
            chain = port.coalesced(port.model(csr), 40 + 3 * k, beta, 1.0, 2, ordered)
            chain.sweep(6)
            np.testing.assert_array_equal(st.spins(k), chain.spins)


def test_coalesced_rejections(lib):
    odd = product_model(ins.build_layered_csr(*ins.layered_spec(8, 3), 5, 1.0))
    generic = product_model(ins.cubic_pm1(4, 5, 0.0))
    too_deep = product_model(ins.build_layered_csr(*ins.layered_spec(8, 3), 66, 1.0))
    for model, text in ((odd, "even layer count"), (generic, "needs a layered model"), (too_deep, "at most 64 layers")):
        with pytest.raises(ib.IsingError) as err:
            ib.init_coalesced(model, [1.0])
        assert err.value.status == _lib.ISING_ERR_ARGUMENT and text in str(err.value)
    ok = product_model(ins.build_layered_csr(*ins.layered_spec(8, 3), 4, 1.0))
    with pytest.raises(ib.IsingError, match="beta must be finite"):
        ib.init_coalesced(ok, [-1.0])
    with pytest.raises(ib.IsingError, match="seed count"):
        ib.init_coalesced(ok, [1.0, 2.0], seeds=[1])
    # tau updates go out as global f32 reductions, which flush subnormals: a model that could hold a
    # subnormal field is refused (the batch API runs it through the read-modify-write kernel instead)
    tiny = ins.build_layered_csr(*ins.layered_spec(8, 3), 4, 1.0)
    tiny["h"] = tiny["h"].copy()
    tiny["h"][3::8] = np.float32(1e-39)  # the same position of every layer: layers stay identical
    with pytest.raises(ib.IsingError, match="2\\^-100"):
        ib.init_coalesced(product_model(tiny), [1.0])


def test_coalesced_walks_the_csr_when_the_layer_graph_does_not_fit(lib, port):
    """86,400 spins: one region (219 KB) fits shared memory, the staged layer graph next to it does
    not, so the kernel falls back to walking the permuted CSR in global memory."""
    csr = ins.build_layered_csr(*ins.layered_spec(1350, 11), 64, 1.0)
    chain = port.coalesced(port.model(csr), 9, 0.8, 1.0, 2)
    with ib.init_coalesced(product_model(csr), [0.8], seeds=[9]) as st:
        st.run(3)
        chain.sweep(3)
        np.testing.assert_array_equal(st.spins(0), chain.spins)
        hs, ht = st.fields(0)
        np.testing.assert_array_equal(hs.view(np.uint32), chain.hs_new_order[chain.forward].view(np.uint32))
        np.testing.assert_array_equal(ht.view(np.uint32), chain.ht_new_order[chain.forward].view(np.uint32))
        assert int(st.stats()[0][0]) == chain.flips


def test_layers_must_be_identical_so_the_staged_graph_always_applies(lib):
    """validate_model (ref: src/model.cpp:283-330) rejects layers that differ, couplings included."""
    csr = ins.build_layered_csr(*ins.layered_spec(16, 3), 6, 0.75)
    csr = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in csr.items()}
    a = 2 * 16 + 5
    e = csr["offsets"][a]
    b = int(csr["targets"][e])
    csr["couplings"][e] = np.float32(0.625)
    back = [k for k in range(csr["offsets"][b], csr["offsets"][b + 1]) if csr["targets"][k] == a][0]
    csr["couplings"][back] = np.float32(0.625)
    with pytest.raises(ib.IsingError, match="layers are not identical"):
        product_model(csr)
