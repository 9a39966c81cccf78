"""Host-side mirror of the reference's sweep interface, backed by the CUDA library.

Names and argument meaning follow the reference's C++ API so that tests read like the
reference's own (ref = /root/reference/proj):

    SpinModel / LayerSpec / build_layered_model / total_cost   ref: include/isingmc/model.hpp:52-90
    SweepParams / ExpKind                                       ref: include/isingmc/sweep.hpp:15-29
    init_state -> BatchState, run_sweeps                        ref: include/isingmc/sweep.hpp:126-157
    state_checksum, field_coherence_ulp                         ref: include/isingmc/sweep.hpp:159-163

A BatchState is the device-backed counterpart of MANY SweepStates (one per chain).  Failures
raise IsingError carrying the ising_status code and the library's thread-local message, the
same way the reference's C API reports them (ref: include/isingmc.h:15-38).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib as L


class IsingError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


class ExpKind:
    """ref: ising_exp_kind, include/isingmc.h:30-35"""
    default, exact, fast, accurate = L.EXP_DEFAULT, L.EXP_EXACT, L.EXP_FAST, L.EXP_ACCURATE


def _check(status: int) -> None:
    if status != L.ISING_OK:
        raise IsingError(status, L.load().ising_b200_last_error().decode())


def _arr(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)


def _p(a: Optional[np.ndarray], ctype):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))


@dataclass
class LayerSpec:
    """ref: LayerSpec / LayerEdge, include/isingmc/model.hpp:62-74"""
    positions: int
    h: Sequence[float]
    edges: Sequence[tuple] = field(default_factory=list)  # (p, q, coupling), undirected, once


class SpinModel:
    """Immutable graph + fields living in the host library (ref: SpinModel, model.hpp:52-60)."""

    def __init__(self, handle: int):
        self._h = handle

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            L.load().ising_b200_model_free(h)

    @classmethod
    def from_csr(cls, n_spins, h, offsets, targets, couplings, tau_counts=None, layers=0,
                 per_layer=0) -> "SpinModel":
        h = _arr(h, np.float32)
        offsets = _arr(offsets, np.uint32)
        targets = _arr(targets, np.uint32)
        couplings = _arr(couplings, np.float32)
        tau = None if tau_counts is None else _arr(tau_counts, np.uint8)
        if h.size != n_spins or offsets.size != n_spins + 1:
            raise IsingError(L.ISING_ERR_ARGUMENT, "validate_model: field/adjacency size mismatch")
        if targets.size != couplings.size or (offsets.size and int(offsets[-1]) != targets.size):
            raise IsingError(L.ISING_ERR_ARGUMENT, "validate_model: field/adjacency size mismatch")
        out = C.c_void_p()
        _check(L.load().ising_b200_model_from_csr(
            n_spins, _p(h, C.c_float), _p(offsets, C.c_uint32), _p(targets, C.c_uint32),
            _p(couplings, C.c_float), _p(tau, C.c_uint8), layers, per_layer, C.byref(out)))
        return cls(out.value)

    # --- `ising-model v1` documents (ref: model_io.hpp:10-28; ising_model_from_string / _load / _to_string)
    @classmethod
    def from_string(cls, text: str) -> "SpinModel":
        out = C.c_void_p()
        _check(L.load().ising_b200_model_from_string(text.encode(), C.byref(out)))
        return cls(out.value)

    @classmethod
    def load(cls, path) -> "SpinModel":
        out = C.c_void_p()
        _check(L.load().ising_b200_model_load(str(path).encode(), C.byref(out)))
        return cls(out.value)

    def to_string(self) -> str:
        out = C.c_void_p()
        _check(L.load().ising_b200_model_to_string(self._h, C.byref(out)))
        try:
            return C.string_at(out.value).decode()
        finally:
            L.load().ising_b200_string_free(out)

    def save(self, path) -> None:
        _check(L.load().ising_b200_model_save(self._h, str(path).encode()))

    @property
    def n_spins(self) -> int:
        return L.load().ising_b200_model_spins(self._h)

    @property
    def half_edges(self) -> int:
        return L.load().ising_b200_model_half_edges(self._h)

    @property
    def layered(self):
        """(layers, per_layer) or None (ref: ising_model_layers, isingmc.h:53)."""
        a, b = C.c_uint32(), C.c_uint32()
        if L.load().ising_b200_model_layers(self._h, C.byref(a), C.byref(b)):
            return a.value, b.value
        return None

    def csr(self) -> dict:
        n, e = self.n_spins, self.half_edges
        out = dict(h=np.empty(n, np.float32), offsets=np.empty(n + 1, np.uint32),
                   targets=np.empty(e, np.uint32), couplings=np.empty(e, np.float32),
                   tau_counts=np.empty(n, np.uint8))
        _check(L.load().ising_b200_model_export_csr(
            self._h, _p(out["h"], C.c_float), _p(out["offsets"], C.c_uint32),
            _p(out["targets"], C.c_uint32), _p(out["couplings"], C.c_float),
            _p(out["tau_counts"], C.c_uint8)))
        return out


def build_layered_model(layer: LayerSpec, n_layers: int, j_tau: float) -> SpinModel:
    """ref: build_layered_model, src/model.cpp:52-104"""
    h = _arr(layer.h, np.float32)
    if h.size != layer.positions:
        raise IsingError(L.ISING_ERR_ARGUMENT, "build_layered_model: layer field count != positions")
    edges = list(layer.edges)
    p = _arr([e[0] for e in edges], np.uint32)
    q = _arr([e[1] for e in edges], np.uint32)
    j = _arr([e[2] for e in edges], np.float32)
    out = C.c_void_p()
    _check(L.load().ising_b200_model_build_layered(
        layer.positions, _p(h, C.c_float), len(edges), _p(p, C.c_uint32), _p(q, C.c_uint32),
        _p(j, C.c_float), n_layers, j_tau, C.byref(out)))
    return SpinModel(out.value)


def total_cost(model: SpinModel, spins) -> float:
    """ref: total_cost, src/model.cpp:108-126 (host, f64)"""
    s = _arr(spins, np.int8)
    cost = C.c_double()
    _check(L.load().ising_b200_model_cost(model._h, _p(s, C.c_int8), s.size, C.byref(cost)))
    return cost.value


@dataclass
class SweepParams:
    """ref: SweepParams, include/isingmc/sweep.hpp:25-29 (beta becomes the ladder `betas`)."""
    tau_scale: float = 1.0
    exp_kind: int = ExpKind.fast


class BatchState:
    """Device-resident state of n_ladders * n_betas chains (ref: SweepState, sweep.hpp:85-121)."""

    def __init__(self, handle: int, models, n_ladders: int, n_betas: int):
        self._h = handle
        self._models = models  # keep the graphs alive
        self.n_ladders = n_ladders
        self.n_betas = n_betas
        self.n_chains = n_ladders * n_betas
        self.n_spins = models[0].n_spins

    def close(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            L.load().ising_batch_free(h)

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # --- stepping
    def run(self, sweeps: int, swap_interval: int = 0) -> None:
        _check(L.load().ising_batch_run(self._h, sweeps, swap_interval))

    def swap(self) -> None:
        _check(L.load().ising_batch_swap(self._h))

    def sync(self) -> None:
        _check(L.load().ising_batch_sync(self._h))

    # --- readout (host numpy arrays)
    def spins(self, first_chain: int = 0, n_chains: Optional[int] = None) -> np.ndarray:
        count = self.n_chains - first_chain if n_chains is None else n_chains
        out = np.empty((count, self.n_spins), np.int8)
        _check(L.load().ising_batch_read_spins(self._h, first_chain, count, _p(out, C.c_int8)))
        return out

    def fields(self, chain: int):
        hs, ht = np.empty(self.n_spins, np.float32), np.empty(self.n_spins, np.float32)
        _check(L.load().ising_batch_read_fields(self._h, chain, _p(hs, C.c_float), _p(ht, C.c_float)))
        return hs, ht

    def _f64(self, fn) -> np.ndarray:
        out = np.empty(self.n_chains, np.float64)
        _check(fn(self._h, _p(out, C.c_double)))
        return out

    def _u64(self, fn) -> np.ndarray:
        out = np.empty(self.n_chains, np.uint64)
        _check(fn(self._h, _p(out, C.c_uint64)))
        return out

    def energies(self) -> np.ndarray:
        return self._f64(L.load().ising_batch_read_energies)

    def running_energies(self) -> np.ndarray:
        return self._f64(L.load().ising_batch_read_running_energies)

    def resync_energies(self) -> None:
        """Running energies := tempering cost of the current spins (drops accumulated rounding)."""
        _check(L.load().ising_batch_resync_energies(self._h))

    def stats(self):
        flips, attempts = np.empty(self.n_chains, np.uint64), np.empty(self.n_chains, np.uint64)
        _check(L.load().ising_batch_read_stats(self._h, _p(flips, C.c_uint64), _p(attempts, C.c_uint64)))
        return flips, attempts

    def checksums(self) -> np.ndarray:
        return self._u64(L.load().ising_batch_checksums)

    def field_coherence_ulp(self) -> np.ndarray:
        return self._u64(L.load().ising_batch_field_coherence)

    def slots(self) -> np.ndarray:
        out = np.empty(self.n_chains, np.uint32)
        _check(L.load().ising_batch_read_slots(self._h, _p(out, C.c_uint32)))
        return out

    def swap_stats(self):
        acc = np.empty((self.n_ladders, self.n_betas), np.uint64)
        att = np.empty((self.n_ladders, self.n_betas), np.uint64)
        _check(L.load().ising_batch_read_swap_stats(self._h, _p(acc, C.c_uint64), _p(att, C.c_uint64)))
        return acc, att

    def pack_results(self, device_ptr: int) -> None:
        _check(L.load().ising_batch_pack_results(self._h, C.c_void_p(device_ptr)))

    def all_gather_results(self, nccl_comm: int, device_ptr: int) -> None:
        """Packs this shard's records and all-gathers every rank's over `nccl_comm` (an ncclComm_t as an
        integer) into device memory at `device_ptr` (n_ranks * n_chains * 32 bytes)."""
        _check(L.load().ising_batch_all_gather_results(self._h, C.c_void_p(nccl_comm), C.c_void_p(device_ptr)))

    def record_wait(self, on: bool = True) -> None:
        """Starts (counters zeroed) or stops recording wait statistics (ref: EngineConfig::stats_widths)."""
        _check(L.load().ising_batch_record_wait(self._h, int(on)))

    def wait_stats(self, widths=(1, 2, 4, 8, 16, 32)) -> dict:
        """ref: collect_wait_stats, src/sweep_state.cpp:33-44 — {width: (probability, groups, with_flip)}."""
        w = _arr(list(widths), np.uint32)
        prob = np.empty(w.size, np.float64)
        groups, flip = np.empty(w.size, np.uint64), np.empty(w.size, np.uint64)
        _check(L.load().ising_batch_read_wait_stats(self._h, w.size, _p(w, C.c_uint32), _p(prob, C.c_double),
                                                    _p(groups, C.c_uint64), _p(flip, C.c_uint64)))
        return {int(k): (float(p), int(g), int(f)) for k, p, g, f in zip(w, prob, groups, flip)}

    def set_timing(self, on: bool) -> None:
        _check(L.load().ising_batch_set_timing(self._h, int(on)))

    def info(self) -> dict:
        info = L.BatchInfo()
        _check(L.load().ising_batch_get_info(self._h, C.byref(info)))
        return {name: getattr(info, name) for name, _ in L.BatchInfo._fields_}


class CoalescedState:
    """Device-resident chains swept with the intra-system schedule (ref: EngineKind::coalesced;
    SweepState for that engine, sweep.hpp:85-121).  Readouts are in the original spin order."""

    def __init__(self, handle: int, model: SpinModel, n_chains: int):
        self._h, self._model, self.n_chains, self.n_spins = handle, model, n_chains, model.n_spins

    def close(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            L.load().ising_coalesced_free(h)

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def run(self, sweeps: int) -> None:
        _check(L.load().ising_coalesced_run(self._h, sweeps))

    def spins(self, chain: int = 0) -> np.ndarray:
        out = np.empty(self.n_spins, np.int8)
        _check(L.load().ising_coalesced_read_spins(self._h, chain, _p(out, C.c_int8)))
        return out

    def fields(self, chain: int = 0):
        hs, ht = np.empty(self.n_spins, np.float32), np.empty(self.n_spins, np.float32)
        _check(L.load().ising_coalesced_read_fields(self._h, chain, _p(hs, C.c_float), _p(ht, C.c_float)))
        return hs, ht

    def stats(self):
        flips, attempts = np.empty(self.n_chains, np.uint64), np.empty(self.n_chains, np.uint64)
        _check(L.load().ising_coalesced_read_stats(self._h, _p(flips, C.c_uint64), _p(attempts, C.c_uint64)))
        return flips, attempts

    def energies(self) -> np.ndarray:
        out = np.empty(self.n_chains, np.float64)
        _check(L.load().ising_coalesced_read_energies(self._h, _p(out, C.c_double)))
        return out

    def checksums(self) -> np.ndarray:
        out = np.empty(self.n_chains, np.uint64)
        _check(L.load().ising_coalesced_checksums(self._h, _p(out, C.c_uint64)))
        return out

    def info(self) -> dict:
        info = L.CoalescedInfo()
        _check(L.load().ising_coalesced_get_info(self._h, C.byref(info)))
        return {name: getattr(info, name) for name, _ in L.CoalescedInfo._fields_}


def init_coalesced(model: SpinModel, betas, *, seeds=None, base_seed: int = 1, params: SweepParams = SweepParams(),
                   initial_spins=None, device: int = 0) -> CoalescedState:
    """ref: prepare_model_for_engine(model, coalesced) + init_state per chain (sweep_state.cpp:218-323)."""
    betas_a = _arr(np.atleast_1d(betas), np.float32)
    seeds_a = None if seeds is None else _arr(seeds, np.uint32)
    if seeds_a is not None and seeds_a.size != betas_a.size:
        raise IsingError(L.ISING_ERR_ARGUMENT, "init_state: seed count mismatch")
    init = None if initial_spins is None else _arr(initial_spins, np.int8)
    if init is not None and init.size != betas_a.size * model.n_spins:
        raise IsingError(L.ISING_ERR_ARGUMENT, "init_state: initial spin count mismatch")
    p = L.CoalescedParams(n_chains=betas_a.size, betas=_p(betas_a, C.c_float), seeds=_p(seeds_a, C.c_uint32),
                          base_seed=base_seed, tau_scale=params.tau_scale, exp_kind=int(params.exp_kind),
                          device=device, initial_spins=_p(init, C.c_int8))
    out = C.c_void_p()
    _check(L.load().ising_coalesced_create(model._h, C.byref(p), C.byref(out)))
    return CoalescedState(out.value, model, int(betas_a.size))


def init_state(models, betas, n_ladders: int = 1, *, seeds=None, swap_seeds=None, base_seed: int = 1,
               swap_base_seed: int = 1, first_ladder: int = 0, params: SweepParams = SweepParams(),
               model_of_ladder=None, initial_spins=None, device: int = 0,
               kernel: int = L.KERNEL_AUTO) -> BatchState:
    """ref: init_state(model, cfg[, initial]), src/sweep_state.cpp:218-234 — for a whole batch."""
    if isinstance(models, SpinModel):
        models = [models]
    models = list(models)
    betas_a = _arr(np.atleast_1d(betas), np.float32)
    n_betas = betas_a.size
    n_chains = n_ladders * n_betas
    seeds_a = None if seeds is None else _arr(seeds, np.uint32)
    swap_a = None if swap_seeds is None else _arr(swap_seeds, np.uint32)
    if seeds_a is not None and seeds_a.size != n_chains:
        raise IsingError(L.ISING_ERR_ARGUMENT, "init_state: seed count mismatch")
    if swap_a is not None and swap_a.size != n_ladders:
        raise IsingError(L.ISING_ERR_ARGUMENT, "init_state: seed count mismatch")
    mol = None if model_of_ladder is None else _arr(model_of_ladder, np.uint32)
    if mol is not None and mol.size != n_ladders:
        raise IsingError(L.ISING_ERR_ARGUMENT, "init_state: model_of_ladder count mismatch")
    init_a = None
    if initial_spins is not None:
        init_a = _arr(initial_spins, np.int8).reshape(-1)
        if not models or init_a.size != n_chains * models[0].n_spins:
            raise IsingError(L.ISING_ERR_ARGUMENT, "init_state: initial spin count mismatch")
    p = L.BatchParams(
        n_ladders=n_ladders, n_betas=n_betas, betas=_p(betas_a, C.c_float), seeds=_p(seeds_a, C.c_uint32),
        swap_seeds=_p(swap_a, C.c_uint32), base_seed=base_seed, swap_base_seed=swap_base_seed,
        first_ladder=first_ladder, tau_scale=params.tau_scale, exp_kind=params.exp_kind, device=device,
        kernel=kernel, initial_spins=_p(init_a, C.c_int8))
    handles = (C.c_void_p * max(1, len(models)))(*[m._h for m in models])
    out = C.c_void_p()
    _check(L.load().ising_batch_create(handles, len(models), _p(mol, C.c_uint32), C.byref(p), C.byref(out)))
    return BatchState(out.value, models, n_ladders, n_betas)


def run_sweeps(state: BatchState, sweeps: int, swap_interval: int = 0) -> None:
    """ref: run_sweeps, src/sweep_state.cpp:272-291 (plus the tempering cadence)"""
    state.run(sweeps, swap_interval)


def state_checksum(spins) -> int:
    """ref: state_checksum, src/sweep_state.cpp:325-336 — host helper on a +/-1 array."""
    h = 1469598103934665603
    for s in np.asarray(spins).reshape(-1):
        h ^= 1 if s > 0 else 0
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def run_single(model: SpinModel, sweeps: int, beta: float, seed: int, tau_scale: float = 1.0,
               exp_kind: int = ExpKind.default, device: int = 0) -> dict:
    """ref: ising_run, include/isingmc.h:74-106 — one chain, report fields of ising_run_report."""
    p = L.RunParams(sweeps=sweeps, beta=beta, tau_scale=tau_scale, exp_kind=exp_kind, seed=seed, device=device)
    r = L.RunReport()
    _check(L.load().ising_b200_run(model._h, C.byref(p), C.byref(r)))
    return {name: getattr(r, name) for name, _ in L.RunReport._fields_}


def run_single_json(model: SpinModel, sweeps: int, beta: float, seed: int, tau_scale: float = 1.0,
                    exp_kind: int = ExpKind.default, device: int = 0):
    """ref: ising_run_json, include/isingmc.h:108-112 — (report dict, JSON text with the reference's keys)."""
    p = L.RunParams(sweeps=sweeps, beta=beta, tau_scale=tau_scale, exp_kind=exp_kind, seed=seed, device=device)
    r = L.RunReport()
    out = C.c_void_p()
    _check(L.load().ising_b200_run_json(model._h, C.byref(p), C.byref(r), C.byref(out)))
    try:
        text = C.string_at(out.value).decode()
    finally:
        L.load().ising_b200_string_free(out)
    return {name: getattr(r, name) for name, _ in L.RunReport._fields_}, text
