"""BASELINE.json's five configurations as data: which instances, how many ladders, which beta
ladder, how many sweeps and the swap cadence.  Used by bench.py and the parity tests; the
instances are the seeded synthetic ones of instances.py (the reference names no dataset)."""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List

import numpy as np

from . import instances as ins


@dataclass
class Workload:
    name: str
    description: str
    make_csrs: Callable[[], List[dict]]  # distinct graph instances
    n_ladders: int                       # per GPU
    betas: np.ndarray
    sweeps: int
    swap_interval: int
    shared_graph: bool                   # True: every ladder uses csrs[0]; False: ladder l uses csrs[l]
    state_bytes_per_spin: int            # S of SURVEY.md §8(d): 5 generic, 9 layered

    @property
    def n_chains(self) -> int:
        return self.n_ladders * len(self.betas)


def _layered(seed: int) -> dict:
    return ins.build_layered_csr(*ins.layered_spec(512, seed, 0.5, 6), 64, 1.5)


def get(name: str) -> Workload:
    s = ins.INSTANCE_SEED
    if name == "c1":
        return Workload("c1", "16^3 periodic cubic lattice, J=+/-1, h=0, 1 chain, beta=1, 1000 sweeps",
                        lambda: [ins.cubic_pm1(16, s, 0.0)], 1, np.array([1.0], np.float32), 1000, 0, True, 5)
    if name == "c2":
        return Workload("c2", "16^3 cubic lattice, h~N(0,0.5^2), 1024 replicas at beta=1, 10000 sweeps",
                        lambda: [ins.cubic_pm1(16, s, 0.5)], 1024, np.array([1.0], np.float32), 10000, 0, True, 5)
    if name == "c3":
        return Workload("c3", "256 distinct 4096-spin mixed-degree (6-8) graphs, J~N(0,1), h~N(0,0.25^2), "
                        "32 betas geometric 0.1-3.0, swap every sweep, 10000 sweeps",
                        lambda: [ins.cubic_mixed_degree(16, s + k) for k in range(256)], 256,
                        ins.geometric_betas(0.1, 3.0, 32), 10000, 1, False, 5)
    if name == "c4":
        return Workload("c4", "64 distinct 512x64 layered instances (32768 spins, degree 6-8, J=+/-1, "
                        "J_perp=1.5, h~N(0,0.5^2)), 32 betas geometric 0.2-5.0, swap every sweep, 5000 sweeps",
                        lambda: [_layered(s + k) for k in range(64)], 64, ins.geometric_betas(0.2, 5.0, 32),
                        5000, 1, False, 9)
    if name == "c5":
        return Workload("c5", "one 512x64 layered instance (32768 spins, degree 6-8), 16384 chains per GPU = "
                        "1024 ladders x 16 betas geometric 0.2-5.0, swap every 10 sweeps, 1000 sweeps",
                        lambda: [_layered(s)], 1024, ins.geometric_betas(0.2, 5.0, 16), 1000, 10, True, 9)
    raise ValueError(f"unknown workload {name!r}")


def mean_degree(csr: dict) -> float:
    return float(len(csr["targets"])) / max(1, int(csr["n_spins"]))
