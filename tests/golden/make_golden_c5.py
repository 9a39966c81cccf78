"""Golden record of config 5's first 100 sweeps on ALL 16,384 chains, produced by the reference itself.

    python tests/golden/make_golden_c5.py        (needs /root/reference; about two minutes of CPU)

The reference's `basic` engine (oracle/_ref/libisingref.so, unmodified sources) runs every chain of
the c5 batch — one 512x64 layered instance, 1,024 ladders x 16 betas, chain seeds base + global chain
id — for 100 sweeps without tempering swaps (the reference has none).  Stored: per-chain accept counts
and final total_cost folded into checksums of checksums (whole batch and per tile of 32 chains), and
the first 64 chains verbatim.  tests/test_gpu_fullsize.py::test_c5_all_chains_first_100_sweeps
compares the CUDA path with it.
"""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import pyoracle  # noqa: E402
from paper_1004_0024_b200 import instances as ins, workloads  # noqa: E402

SWEEPS = 100


def fold(values: np.ndarray) -> int:
    """FNV-1a over 64-bit words (the reference's checksum recipe, sweep_state.cpp:325-336, on words)."""
    h = 1469598103934665603
    for v in np.ascontiguousarray(values).view(np.uint64).tolist():
        h = ((h ^ v) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def main():
    pyoracle.build(ref=True)
    ref = pyoracle.Reference()
    wl = workloads.get("c5")
    csr = wl.make_csrs()[0]
    model = ref.model(csr)
    nb = len(wl.betas)
    chains = wl.n_ladders * nb
    seeds = (ins.CHAIN_SEED_BASE + np.arange(chains)).astype(np.uint32)
    lad = ref.ladders([model] * wl.n_ladders, wl.n_ladders, wl.betas, seeds, None, 1.0, 2, 1)
    secs = lad.run(SWEEPS, 0, os.cpu_count() or 1)
    flips, energy = lad.read()
    tiles = chains // 32
    out = dict(sweeps=SWEEPS, chains=chains, flips_fold=np.uint64(fold(flips)), energy_fold=np.uint64(fold(energy)),
               tile_flips_fold=np.array([fold(flips[32 * t:32 * t + 32]) for t in range(tiles)], np.uint64),
               tile_energy_fold=np.array([fold(energy[32 * t:32 * t + 32]) for t in range(tiles)], np.uint64),
               flips_head=flips[:64].copy(), energy_head=energy[:64].copy())
    np.savez_compressed(Path(__file__).resolve().parent / "c5_first100.npz", **out)
    print(f"reference: {chains} chains x {SWEEPS} sweeps in {secs:.1f} s; flips fold {out['flips_fold']:016x}")


if __name__ == "__main__":
    main()
