"""The plain-C restatement of the reference's intra-system `coalesced` schedule
pinned to the reference itself: same permutation, and every sweep the same spins, fields and flip
counts as `EngineKind::coalesced` running on the reference's own permuted model
(ref: proj/src/sweep_coalesced.cpp, proj/src/model.cpp:190-245, proj/tests/test_sweep.cpp:236-291)."""
import numpy as np
import pytest

from helpers import ins

COALESCED = 3  # EngineKind::coalesced in oracle/ref_shim.cpp


@pytest.mark.parametrize("positions,layers,exp_kind", [(12, 4, 2), (16, 8, 1), (24, 6, 3), (8, 64, 2)])
def test_port_follows_the_reference_coalesced_engine_every_sweep(port, ref, positions, layers, exp_kind):
    csr = ins.build_layered_csr(*ins.layered_spec(positions, 31 + positions), layers, 1.25)
    ref_identity = ref.model(csr)
    ref_model, forward = ref_identity.prepared_for(COALESCED)
    mine = port.coalesced(port.model(csr), 777, 0.8, 1.5, exp_kind)
    np.testing.assert_array_equal(mine.forward, forward)
    theirs = ref.chain(ref_model, 777, 0.8, 1.5, exp_kind, None, engine=COALESCED)
    for sweep in range(12):
        spins, hs, ht, flips, attempts = theirs._read()
        np.testing.assert_array_equal(mine.spins_new_order, spins)
        np.testing.assert_array_equal(mine.hs_new_order.view(np.uint32), hs.view(np.uint32))
        np.testing.assert_array_equal(mine.ht_new_order.view(np.uint32), ht.view(np.uint32))
        assert (mine.flips, mine.attempts) == (flips, attempts)
        mine.sweep(1)
        theirs.sweep(1)
    # original-order readout
    np.testing.assert_array_equal(mine.spins, np.sign(theirs.spins[forward]).astype(np.int8))


def test_port_rejects_what_the_reference_rejects(port):
    odd = ins.build_layered_csr(*ins.layered_spec(8, 3), 5, 1.0)  # odd layer count
    with pytest.raises(ValueError):
        port.coalesced(port.model(odd), 1, 1.0)
    generic = ins.cubic_pm1(4, 5, 0.0)
    with pytest.raises(ValueError):
        port.coalesced(port.model(generic), 1, 1.0)
