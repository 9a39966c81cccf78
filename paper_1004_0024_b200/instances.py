"""Seeded synthetic instances with the shapes of BASELINE.json's five configurations.

The reference measures on no public dataset and its own generator (ref:
proj/src/generate.cpp) cannot express a cubic lattice, Gaussian fields or J_perp = 1.5, so the
workloads are defined here, once, with the reference's draw idioms (ref: generate.cpp:12-16,81):

    sign   : (next_u32() >> 31) ? -1 : +1
    index  : (u64(next_u32()) * m) >> 32
    unit   : u32_to_unit(next_u32())            (x / 2^32 truncated to f32)
    normal : Box-Muller on two unit draws in f64, scaled by sigma, rounded once to f32
             (the reference has no Gaussian draw; parity never depends on this recipe because
             both sides are fed the same arrays)

Every generator returns plain numpy CSR arrays (a dict accepted by SpinModel.from_csr) or a
LayerSpec; nothing here touches the GPU.
"""
from __future__ import annotations

import math
from typing import Dict, List, Tuple

import numpy as np

INSTANCE_SEED = 12345
CHAIN_SEED_BASE = 1000
SWAP_SEED_BASE = 77000


class MT19937:
    """Canonical MT19937 (init_genrand seeding), block-vectorised in numpy."""

    def __init__(self, seed: int):
        w = np.empty(624, np.uint64)
        w[0] = seed & 0xFFFFFFFF
        for i in range(1, 624):
            p = int(w[i - 1])
            w[i] = (1812433253 * (p ^ (p >> 30)) + i) & 0xFFFFFFFF
        self.w = w.astype(np.uint32)
        self.buf = np.empty(0, np.uint32)
        self.pos = 0

    def _twist(self) -> None:
        w = self.w

        def gen(lo, hi, far):
            y = (w[lo:hi] & np.uint32(0x80000000)) | (w[lo + 1:hi + 1] & np.uint32(0x7FFFFFFF))
            w[lo:hi] = far ^ (y >> np.uint32(1)) ^ np.where(y & np.uint32(1), np.uint32(0x9908B0DF), np.uint32(0))

        gen(0, 227, w[397:624].copy())
        gen(227, 454, w[0:227].copy())
        gen(454, 623, w[227:396].copy())
        y = (w[623] & np.uint32(0x80000000)) | (w[0] & np.uint32(0x7FFFFFFF))
        w[623] = w[396] ^ (y >> np.uint32(1)) ^ (np.uint32(0x9908B0DF) if y & np.uint32(1) else np.uint32(0))

    def _block(self) -> np.ndarray:
        self._twist()
        y = self.w.copy()
        y ^= y >> np.uint32(11)
        y ^= (y << np.uint32(7)) & np.uint32(0x9D2C5680)
        y ^= (y << np.uint32(15)) & np.uint32(0xEFC60000)
        y ^= y >> np.uint32(18)
        return y

    def take(self, count: int) -> np.ndarray:
        """The next `count` raw 32-bit outputs."""
        out = np.empty(count, np.uint32)
        done = 0
        while done < count:
            if self.pos == self.buf.size:
                self.buf, self.pos = self._block(), 0
            k = min(count - done, self.buf.size - self.pos)
            out[done:done + k] = self.buf[self.pos:self.pos + k]
            self.pos += k
            done += k
        return out

    def next_u32(self) -> int:
        return int(self.take(1)[0])

    def below(self, m: int) -> int:
        return (self.next_u32() * m) >> 32

    def signs(self, count: int) -> np.ndarray:
        return np.where(self.take(count) >> np.uint32(31), np.float32(-1), np.float32(1)).astype(np.float32)

    def normals(self, count: int, sigma: float) -> np.ndarray:
        raw = self.take(2 * count)
        u1 = u32_to_unit(raw[0::2]).astype(np.float64)
        u2 = u32_to_unit(raw[1::2]).astype(np.float64)
        z = np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * math.pi * u2)
        return (z * sigma).astype(np.float32)


def u32_to_unit(x) -> np.ndarray:
    """ref: u32_to_unit, include/isingmc/rng.hpp:87-92 — keep the top 24 significant bits."""
    x = np.asarray(x, np.uint32)
    width = np.frexp(x.astype(np.float64))[1].astype(np.int64)  # exact bit length (0 for x == 0)
    drop = np.maximum(width - 24, 0).astype(np.uint32)
    kept = (x >> drop) << drop
    return (kept.astype(np.float32) * np.float32(2.0 ** -32)).astype(np.float32)


def csr_from_adjacency(h: np.ndarray, nbrs: List[List[Tuple[int, float]]], tau_counts=None, layers=0,
                       per_layer=0) -> Dict:
    n = len(nbrs)
    offsets = np.zeros(n + 1, np.uint32)
    offsets[1:] = np.cumsum([len(x) for x in nbrs])
    targets = np.array([t for lst in nbrs for t, _ in lst], np.uint32)
    couplings = np.array([c for lst in nbrs for _, c in lst], np.float32)
    return dict(n_spins=n, h=np.asarray(h, np.float32), offsets=offsets, targets=targets,
                couplings=couplings, tau_counts=None if tau_counts is None else np.asarray(tau_counts, np.uint8),
                layers=layers, per_layer=per_layer)


def cubic_lattice_edges(side: int) -> np.ndarray:
    """Undirected edges (i, j) of a periodic side^3 lattice, site (x,y,z) -> (z*side+y)*side+x,
    listed per site in +x, +y, +z order."""
    idx = np.arange(side ** 3)
    x, y, z = idx % side, (idx // side) % side, idx // (side * side)
    px = (z * side + y) * side + (x + 1) % side
    py = (z * side + (y + 1) % side) * side + x
    pz = (((z + 1) % side) * side + y) * side + x
    return np.stack([np.repeat(idx, 3), np.stack([px, py, pz], 1).reshape(-1)], 1)


def _adjacency(n: int, edges: np.ndarray, coup: np.ndarray) -> List[List[Tuple[int, float]]]:
    nbrs: List[List[Tuple[int, float]]] = [[] for _ in range(n)]
    for (a, b), c in zip(edges.tolist(), coup.tolist()):
        nbrs[a].append((b, c))
        nbrs[b].append((a, c))
    for lst in nbrs:
        lst.sort(key=lambda e: e[0])  # canonical order: ascending target (ref: model.hpp:23-29)
    return nbrs


def cubic_pm1(side: int = 16, seed: int = INSTANCE_SEED, h_sigma: float = 0.0) -> Dict:
    """C1 (h_sigma = 0) / C2 (h_sigma = 0.5): periodic cubic lattice, J = +/-1 by seeded MT19937."""
    rng = MT19937(seed)
    edges = cubic_lattice_edges(side)
    coup = rng.signs(len(edges))
    n = side ** 3
    h = rng.normals(n, h_sigma) if h_sigma > 0 else np.zeros(n, np.float32)
    return csr_from_adjacency(h, _adjacency(n, edges, coup))


def cubic_mixed_degree(side: int = 16, seed: int = INSTANCE_SEED, j_sigma: float = 1.0,
                       h_sigma: float = 0.25, max_degree: int = 8) -> Dict:
    """C3: the cubic lattice plus, per spin, 0-2 extra edges to uniformly drawn non-neighbours
    (symmetric insertion, every degree capped at max_degree), J ~ N(0, j_sigma^2), h ~ N(0, h_sigma^2)."""
    rng = MT19937(seed)
    base = cubic_lattice_edges(side)
    n = side ** 3
    present = set((min(a, b), max(a, b)) for a, b in base.tolist())
    degree = np.zeros(n, np.int64)
    np.add.at(degree, base.reshape(-1), 1)
    extra = []
    wanted = (rng.take(n).astype(np.uint64) * np.uint64(3)) >> np.uint64(32)  # below(3) per spin
    for i in range(n):
        tries = 0
        added = 0
        while added < int(wanted[i]) and tries < 16:
            tries += 1
            t = rng.below(n)
            key = (min(i, t), max(i, t))
            if t == i or key in present or degree[i] >= max_degree or degree[t] >= max_degree:
                continue
            present.add(key)
            degree[i] += 1
            degree[t] += 1
            extra.append((i, t))
            added += 1
    edges = np.concatenate([base, np.array(extra, np.int64).reshape(-1, 2)], 0)
    coup = rng.normals(len(edges), j_sigma)
    h = rng.normals(n, h_sigma)
    return csr_from_adjacency(h, _adjacency(n, edges, coup))


def layered_spec(positions: int = 512, seed: int = INSTANCE_SEED, h_sigma: float = 0.5,
                 degree_max: int = 6):
    """C4/C5 layer: circulant +/-1, +/-2 (degree 4) plus up to positions/2 seeded extra edges with
    every space degree capped at degree_max (the scheme of ref: generate.cpp:55-76), J = +/-1,
    h_p ~ N(0, h_sigma^2).  Returns (positions, h, edges[(p, q, J)])."""
    rng = MT19937(seed)
    present = set()
    degree = [0] * positions
    edges = []

    def add(a, b):
        key = (min(a, b), max(a, b))
        if a == b or key in present:
            return False
        present.add(key)
        degree[a] += 1
        degree[b] += 1
        edges.append(key)
        return True

    for off in (1, 2):
        if positions > 2 * off or (positions == 2 * off):
            for p in range(positions):
                add(p, (p + off) % positions)
    budget, attempts = positions // 2, 8 * positions + 64
    while budget > 0 and attempts > 0:
        attempts -= 1
        a, b = rng.below(positions), rng.below(positions)
        if degree[a] >= degree_max or degree[b] >= degree_max:
            continue
        if add(a, b):
            budget -= 1
    coup = rng.signs(len(edges))
    h = rng.normals(positions, h_sigma)
    return positions, h, [(p, q, float(c)) for (p, q), c in zip(edges, coup)]


def build_layered_csr(positions: int, h, edges, n_layers: int, j_tau: float) -> Dict:
    """numpy restatement of build_layered_model (ref: src/model.cpp:52-104) producing CSR arrays;
    the product path uses the C++ builder, this one feeds the CPU oracles."""
    nbr: List[List[Tuple[int, float]]] = [[] for _ in range(positions)]
    for p, q, c in edges:
        nbr[p].append((q, c))
        nbr[q].append((p, c))
    for lst in nbr:
        lst.sort(key=lambda e: e[0])
    out: List[List[Tuple[int, float]]] = []
    for l in range(n_layers):
        base, up, down = l * positions, ((l + 1) % n_layers) * positions, ((l - 1) % n_layers) * positions
        for p in range(positions):
            out.append([(base + t, c) for t, c in nbr[p]] + [(up + p, j_tau), (down + p, j_tau)])
    return csr_from_adjacency(np.tile(np.asarray(h, np.float32), n_layers), out,
                              tau_counts=np.full(n_layers * positions, 2, np.uint8), layers=n_layers,
                              per_layer=positions)


def geometric_betas(lo: float, hi: float, count: int) -> np.ndarray:
    """beta_k = lo * (hi/lo)^(k/(count-1)), computed in f64 and rounded to f32."""
    if count == 1:
        return np.array([lo], np.float32)
    k = np.arange(count, dtype=np.float64)
    return (lo * (hi / lo) ** (k / (count - 1))).astype(np.float32)
