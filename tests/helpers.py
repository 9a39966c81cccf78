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


__all__ = ["csr_from_npz", "product_model", "bits", "oracle_batch", "assert_batch_matches", "ins", "ib"]
