"""TEST INFRASTRUCTURE ONLY — ctypes access to the two CPU checkers:

    Port      oracle/liboracle.so          plain-C restatement (ising_oracle.c), always buildable
    Reference oracle/_ref/libisingref.so   the UNMODIFIED reference sources + ref_shim.cpp,
                                           built only where /root/reference exists

May be imported by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs only.  The product package never imports this module.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_LIB = HERE / "liboracle.so"
REF_LIB = HERE / "_ref" / "libisingref.so"
REFERENCE_ROOT = Path("/root/reference/proj")

u8p, i8p = C.POINTER(C.c_uint8), C.POINTER(C.c_int8)
u32p, u64p = C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)
f32p, f64p = C.POINTER(C.c_float), C.POINTER(C.c_double)

EXP_EXACT, EXP_FAST, EXP_ACCURATE = 1, 2, 3


def build(ref: bool = True) -> None:
    """Compiles the port, and the reference library when its sources are present."""
    subprocess.run(["make", "-s", "-C", str(HERE), "oracle"], check=True)
    if ref and REFERENCE_ROOT.exists():
        subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)
        # the reference-side binding of INTEGRATION.md, against the product library when that is built
        if (HERE.parent / "paper_1004_0024_b200" / "libisingb200.so").exists():
            subprocess.run(["make", "-s", "-C", str(HERE), "binding"], check=True)


def _p(a, ctype):
    return None if a is None else a.ctypes.data_as(C.POINTER(ctype))


class _Model(C.Structure):
    _fields_ = [("n_spins", C.c_uint32), ("h", f32p), ("offsets", u32p), ("targets", u32p),
                ("couplings", f32p), ("tau_counts", u8p), ("layers", C.c_uint32), ("per_layer", C.c_uint32)]


class _PtResult(C.Structure):
    _fields_ = [("spins", i8p), ("flips", u64p), ("e_run", f64p), ("energy", f64p), ("slot", u32p),
                ("swap_acc", u64p), ("swap_att", u64p)]


class _Mt(C.Structure):
    _fields_ = [("w", C.c_uint32 * 624), ("cursor", C.c_uint32)]


class _Chain(C.Structure):
    _fields_ = [("n", C.c_uint32), ("beta", C.c_float), ("tau_scale", C.c_float), ("exp_kind", C.c_int),
                ("spins", f32p), ("hs", f32p), ("ht", f32p), ("rng", _Mt), ("flips", C.c_uint64),
                ("attempts", C.c_uint64), ("e_run", C.c_double), ("energy_block", C.c_uint32)]


class _Coalesced(C.Structure):
    _fields_ = [("n", C.c_uint32), ("lanes", C.c_uint32), ("per_layer", C.c_uint32), ("beta", C.c_float),
                ("tau_scale", C.c_float), ("exp_kind", C.c_int), ("permuted", _Model), ("forward", u32p),
                ("spins", f32p), ("hs", f32p), ("ht", f32p), ("flags", u8p), ("lane_rng", C.c_void_p),
                ("flips", C.c_uint64), ("attempts", C.c_uint64)]


def _canon(csr: dict) -> dict:
    n = int(csr["n_spins"])
    tau = csr.get("tau_counts")
    return dict(
        n_spins=n,
        h=np.ascontiguousarray(csr["h"], np.float32),
        offsets=np.ascontiguousarray(csr["offsets"], np.uint32),
        targets=np.ascontiguousarray(csr["targets"], np.uint32),
        couplings=np.ascontiguousarray(csr["couplings"], np.float32),
        tau_counts=np.zeros(n, np.uint8) if tau is None else np.ascontiguousarray(tau, np.uint8),
        layers=int(csr.get("layers", 0) or 0), per_layer=int(csr.get("per_layer", 0) or 0))


class Port:
    """The plain-C restatement."""

    kind = "port"

    def __init__(self):
        if not PORT_LIB.exists():
            build(ref=False)
        lib = C.CDLL(str(PORT_LIB))
        lib.orc_mt_fill.argtypes = [C.c_uint32, u32p, C.c_size_t]
        lib.orc_u32_to_unit.restype = C.c_float
        lib.orc_u32_to_unit.argtypes = [C.c_uint32]
        for name in ("orc_exp_fast", "orc_exp_accurate", "orc_exp_exact"):
            getattr(lib, name).restype = C.c_float
            getattr(lib, name).argtypes = [C.c_float]
        lib.orc_initial_spins.argtypes = [C.c_uint32, C.c_uint32, i8p]
        lib.orc_recompute_fields.argtypes = [C.POINTER(_Model), f32p, f32p, f32p]
        lib.orc_total_cost.restype = C.c_double
        lib.orc_total_cost.argtypes = [C.POINTER(_Model), f32p]
        lib.orc_tempering_cost.restype = C.c_double
        lib.orc_tempering_cost.argtypes = [C.POINTER(_Model), f32p, C.c_float]
        lib.orc_checksum.restype = C.c_uint64
        lib.orc_checksum.argtypes = [f32p, C.c_uint32]
        lib.orc_field_coherence_ulp.restype = C.c_uint64
        lib.orc_field_coherence_ulp.argtypes = [C.POINTER(_Model), f32p, f32p, f32p]
        lib.orc_chain_create.restype = C.POINTER(_Chain)
        lib.orc_chain_create.argtypes = [C.POINTER(_Model), C.c_uint32, C.c_float, C.c_float, C.c_int, i8p]
        lib.orc_chain_free.argtypes = [C.POINTER(_Chain)]
        lib.orc_chain_sweep.argtypes = [C.POINTER(_Chain), C.POINTER(_Model), C.c_uint64]
        lib.orc_coalesced_create.restype = C.POINTER(_Coalesced)
        lib.orc_coalesced_create.argtypes = [C.POINTER(_Model), C.c_uint32, C.c_float, C.c_float, C.c_int, i8p]
        lib.orc_coalesced_free.argtypes = [C.POINTER(_Coalesced)]
        lib.orc_coalesced_sweep.argtypes = [C.POINTER(_Coalesced), C.c_uint64]
        lib.orc_coalesced_read_spins.argtypes = [C.POINTER(_Coalesced), i8p]
        lib.orc_pt_run.restype = C.c_int
        lib.orc_pt_run.argtypes = [C.POINTER(C.POINTER(_Model)), C.c_uint32, C.c_uint32, f32p, u32p, u32p,
                                   C.c_float, C.c_int, C.c_uint64, C.c_uint32, C.c_uint32, i8p,
                                   C.POINTER(_PtResult)]
        self.lib = lib

    # --- primitives
    def mt_fill(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, np.uint32)
        self.lib.orc_mt_fill(seed, _p(out, C.c_uint32), count)
        return out

    def u32_to_unit(self, x: int) -> float:
        return self.lib.orc_u32_to_unit(int(x))

    def exp(self, kind: int, x: float) -> float:
        return {1: self.lib.orc_exp_exact, 2: self.lib.orc_exp_fast, 3: self.lib.orc_exp_accurate}[kind](x)

    def initial_spins(self, n: int, seed: int) -> np.ndarray:
        out = np.empty(n, np.int8)
        self.lib.orc_initial_spins(n, seed, _p(out, C.c_int8))
        return out

    # --- models
    def model(self, csr: dict):
        keep = _canon(csr)
        m = _Model(keep["n_spins"], _p(keep["h"], C.c_float), _p(keep["offsets"], C.c_uint32),
                   _p(keep["targets"], C.c_uint32), _p(keep["couplings"], C.c_float),
                   _p(keep["tau_counts"], C.c_uint8), int(csr.get("layers") or 0), int(csr.get("per_layer") or 0))
        m._keep = keep
        return m

    def total_cost(self, model, spins) -> float:
        s = np.ascontiguousarray(spins, np.float32)
        return self.lib.orc_total_cost(C.byref(model), _p(s, C.c_float))

    def tempering_cost(self, model, spins, tau_scale) -> float:
        """total_cost with the tau couplings scaled by gamma in f32: what the running energy tracks."""
        s = np.ascontiguousarray(spins, np.float32)
        return self.lib.orc_tempering_cost(C.byref(model), _p(s, C.c_float), float(tau_scale))

    def checksum(self, spins) -> int:
        s = np.ascontiguousarray(spins, np.float32)
        return self.lib.orc_checksum(_p(s, C.c_float), s.size)

    def recompute_fields(self, model, spins):
        s = np.ascontiguousarray(spins, np.float32)
        hs, ht = np.empty(s.size, np.float32), np.empty(s.size, np.float32)
        self.lib.orc_recompute_fields(C.byref(model), _p(s, C.c_float), _p(hs, C.c_float), _p(ht, C.c_float))
        return hs, ht

    # --- one chain (SweepState)
    def chain(self, model, seed, beta, tau_scale=1.0, exp_kind=EXP_FAST, initial=None):
        return PortChain(self, model, seed, beta, tau_scale, exp_kind, initial)

    def coalesced(self, model, seed, beta, tau_scale=1.0, exp_kind=EXP_FAST, initial_new_order=None):
        return PortCoalesced(self, model, seed, beta, tau_scale, exp_kind, initial_new_order)

    # --- batch with tempering
    def pt_run(self, models, n_ladders, betas, seeds, swap_seeds, sweeps, swap_interval, tau_scale=1.0,
               exp_kind=EXP_FAST, threads=1, initial=None, want_spins=True) -> dict:
        betas = np.ascontiguousarray(betas, np.float32)
        nb = betas.size
        chains = n_ladders * nb
        n = models[0].n_spins
        seeds = np.ascontiguousarray(seeds, np.uint32)
        swap_seeds = np.ascontiguousarray(np.zeros(n_ladders) if swap_seeds is None else swap_seeds, np.uint32)
        assert seeds.size == chains and swap_seeds.size == n_ladders and len(models) == n_ladders
        res = dict(spins=np.empty((chains, n), np.int8) if want_spins else None,
                   flips=np.zeros(chains, np.uint64), e_run=np.zeros(chains, np.float64),
                   energy=np.zeros(chains, np.float64), slot=np.zeros(chains, np.uint32),
                   swap_acc=np.zeros((n_ladders, nb), np.uint64), swap_att=np.zeros((n_ladders, nb), np.uint64))
        out = _PtResult(_p(res["spins"], C.c_int8), _p(res["flips"], C.c_uint64), _p(res["e_run"], C.c_double),
                        _p(res["energy"], C.c_double), _p(res["slot"], C.c_uint32),
                        _p(res["swap_acc"], C.c_uint64), _p(res["swap_att"], C.c_uint64))
        ptrs = (C.POINTER(_Model) * n_ladders)(*[C.pointer(m) for m in models])
        init = None if initial is None else np.ascontiguousarray(initial, np.int8)
        rc = self.lib.orc_pt_run(ptrs, n_ladders, nb, _p(betas, C.c_float), _p(seeds, C.c_uint32),
                                 _p(swap_seeds, C.c_uint32), tau_scale, exp_kind, sweeps, swap_interval,
                                 threads, _p(init, C.c_int8), C.byref(out))
        if rc != 0:
            raise RuntimeError("orc_pt_run failed")
        return res


class PortCoalesced:
    """The plain-C restatement of the reference's coalesced engine on one chain."""

    def __init__(self, port, model, seed, beta, tau_scale, exp_kind, initial_new_order):
        self.port, self.model = port, model
        init = None if initial_new_order is None else np.ascontiguousarray(initial_new_order, np.int8)
        self.ptr = port.lib.orc_coalesced_create(C.byref(model), seed, beta, tau_scale, exp_kind, _p(init, C.c_int8))
        if not self.ptr:
            raise ValueError("coalesced: needs a layered model with an even layer count >= 4")
        self.n = model.n_spins

    def __del__(self):
        if getattr(self, "ptr", None):
            self.port.lib.orc_coalesced_free(self.ptr)
            self.ptr = None

    def sweep(self, sweeps: int = 1):
        self.port.lib.orc_coalesced_sweep(self.ptr, sweeps)

    def _new_order(self, p):
        return np.ctypeslib.as_array(p, shape=(self.n,)).copy()

    @property
    def forward(self):
        return self._new_order(self.ptr.contents.forward)

    @property
    def spins_new_order(self):
        return self._new_order(self.ptr.contents.spins)

    @property
    def hs_new_order(self):
        return self._new_order(self.ptr.contents.hs)

    @property
    def ht_new_order(self):
        return self._new_order(self.ptr.contents.ht)

    @property
    def spins(self):
        """+1/-1 in the ORIGINAL spin order."""
        out = np.empty(self.n, np.int8)
        self.port.lib.orc_coalesced_read_spins(self.ptr, _p(out, C.c_int8))
        return out

    @property
    def flips(self):
        return int(self.ptr.contents.flips)

    @property
    def attempts(self):
        return int(self.ptr.contents.attempts)


class PortChain:
    def __init__(self, port, model, seed, beta, tau_scale, exp_kind, initial):
        self.port, self.model = port, model
        init = None if initial is None else np.ascontiguousarray(initial, np.int8)
        self.ptr = port.lib.orc_chain_create(C.byref(model), seed, beta, tau_scale, exp_kind, _p(init, C.c_int8))
        if not self.ptr:
            raise MemoryError
        self.n = model.n_spins

    def __del__(self):
        if getattr(self, "ptr", None):
            self.port.lib.orc_chain_free(self.ptr)
            self.ptr = None

    def sweep(self, sweeps: int = 1):
        self.port.lib.orc_chain_sweep(self.ptr, C.byref(self.model), sweeps)

    def set_beta(self, beta: float):
        self.ptr.contents.beta = beta

    def _arr(self, p):
        return np.ctypeslib.as_array(p, shape=(self.n,)).copy() if self.n else np.empty(0, np.float32)

    @property
    def spins(self):
        return self._arr(self.ptr.contents.spins)

    @property
    def hs(self):
        return self._arr(self.ptr.contents.hs)

    @property
    def ht(self):
        return self._arr(self.ptr.contents.ht)

    @property
    def flips(self):
        return int(self.ptr.contents.flips)

    @property
    def attempts(self):
        return int(self.ptr.contents.attempts)

    @property
    def e_run(self):
        return float(self.ptr.contents.e_run)


class Reference:
    """The reference's own code (needs oracle/_ref/libisingref.so)."""

    kind = "reference"

    @staticmethod
    def available() -> bool:
        return REF_LIB.exists()

    def __init__(self):
        if not REF_LIB.exists():
            raise RuntimeError("oracle/_ref/libisingref.so is not built (needs /root/reference)")
        lib = C.CDLL(str(REF_LIB))
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_mt_fill.argtypes = [C.c_uint32, u32p, C.c_size_t]
        lib.ref_mt_next_stream.argtypes = [C.c_uint32, u32p, C.c_size_t]
        lib.ref_u32_to_unit.restype = C.c_float
        lib.ref_u32_to_unit.argtypes = [C.c_uint32]
        for name in ("ref_exp_fast", "ref_exp_accurate", "ref_exp_exact"):
            getattr(lib, name).restype = C.c_float
            getattr(lib, name).argtypes = [C.c_float]
        lib.ref_initial_spins.argtypes = [C.c_uint32, C.c_uint32, i8p]
        lib.ref_model_from_csr.restype = C.c_void_p
        lib.ref_model_from_csr.argtypes = [C.c_uint32, f32p, u32p, u32p, f32p, u8p, C.c_uint32, C.c_uint32]
        lib.ref_build_layered.restype = C.c_void_p
        lib.ref_build_layered.argtypes = [C.c_uint32, f32p, C.c_uint32, u32p, u32p, f32p, C.c_uint32, C.c_float]
        lib.ref_model_free.argtypes = [C.c_void_p]
        lib.ref_model_validate.argtypes = [C.c_void_p]
        lib.ref_model_spins.restype = C.c_uint32
        lib.ref_model_spins.argtypes = [C.c_void_p]
        lib.ref_model_half_edges.restype = C.c_uint64
        lib.ref_model_half_edges.argtypes = [C.c_void_p]
        lib.ref_model_export.argtypes = [C.c_void_p, f32p, u32p, u32p, f32p, u8p]
        lib.ref_prepare_model.restype = C.c_void_p
        lib.ref_prepare_model.argtypes = [C.c_void_p, C.c_int, u32p]
        lib.ref_model_to_string.restype = C.c_long
        lib.ref_model_to_string.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t]
        lib.ref_model_from_string.restype = C.c_void_p
        lib.ref_model_from_string.argtypes = [C.c_char_p]
        lib.ref_total_cost.restype = C.c_double
        lib.ref_total_cost.argtypes = [C.c_void_p, f32p]
        if hasattr(lib, "ref_enumerate_boltzmann"):  # (absent from a library built before round 2)
            lib.ref_enumerate_boltzmann.restype = C.c_int
            lib.ref_enumerate_boltzmann.argtypes = [C.c_void_p, C.c_double, f64p, f64p]
            lib.ref_chain_statistics.restype = C.c_int
            lib.ref_chain_statistics.argtypes = [C.c_void_p, C.c_int, C.c_float, C.c_float, C.c_int, C.c_uint64,
                                                 C.c_uint64, C.c_uint32, C.c_uint32, C.c_double, f64p]
        lib.ref_checksum.restype = C.c_uint64
        lib.ref_checksum.argtypes = [f32p, C.c_uint32]
        lib.ref_chain_create.restype = C.c_void_p
        lib.ref_chain_create.argtypes = [C.c_void_p, C.c_int, C.c_uint32, C.c_float, C.c_float, C.c_int, i8p]
        lib.ref_chain_free.argtypes = [C.c_void_p]
        lib.ref_chain_sweep.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64]
        lib.ref_chain_set_beta.argtypes = [C.c_void_p, C.c_float]
        lib.ref_chain_read.argtypes = [C.c_void_p, f32p, f32p, f32p, u64p, u64p]
        lib.ref_chain_coherence.restype = C.c_uint64
        lib.ref_chain_coherence.argtypes = [C.c_void_p, C.c_void_p]
        lib.ref_flip_probability.restype = C.c_float
        lib.ref_flip_probability.argtypes = [C.c_void_p, C.c_uint32]
        lib.ref_ladders_create.restype = C.c_void_p
        lib.ref_ladders_create.argtypes = [C.POINTER(C.c_void_p), C.c_uint32, C.c_uint32, f32p, u32p, u32p,
                                           C.c_float, C.c_int, C.c_int]
        lib.ref_ladders_free.argtypes = [C.c_void_p]
        lib.ref_ladders_run.restype = C.c_double
        lib.ref_ladders_run.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32]
        lib.ref_ladders_read.argtypes = [C.c_void_p, u64p, f64p]
        self.lib = lib

    def error(self) -> str:
        return self.lib.ref_last_error().decode()

    def mt_fill(self, seed, count):
        out = np.empty(count, np.uint32)
        self.lib.ref_mt_fill(seed, _p(out, C.c_uint32), count)
        return out

    def mt_next_stream(self, seed, count):
        out = np.empty(count, np.uint32)
        self.lib.ref_mt_next_stream(seed, _p(out, C.c_uint32), count)
        return out

    def u32_to_unit(self, x):
        return self.lib.ref_u32_to_unit(int(x))

    def exp(self, kind, x):
        return {1: self.lib.ref_exp_exact, 2: self.lib.ref_exp_fast, 3: self.lib.ref_exp_accurate}[kind](x)

    def initial_spins(self, n, seed):
        out = np.empty(n, np.int8)
        self.lib.ref_initial_spins(n, seed, _p(out, C.c_int8))
        return out

    def model(self, csr: dict):
        return RefModel(self, _canon(csr))

    def build_layered(self, positions, h, edges, n_layers, j_tau):
        h = np.ascontiguousarray(h, np.float32)
        p = np.ascontiguousarray([e[0] for e in edges], np.uint32)
        q = np.ascontiguousarray([e[1] for e in edges], np.uint32)
        j = np.ascontiguousarray([e[2] for e in edges], np.float32)
        handle = self.lib.ref_build_layered(positions, _p(h, C.c_float), len(edges), _p(p, C.c_uint32),
                                            _p(q, C.c_uint32), _p(j, C.c_float), n_layers, j_tau)
        if not handle:
            raise ValueError(self.error())
        return RefModel(self, None, handle)

    def total_cost(self, model, spins):
        s = np.ascontiguousarray(spins, np.float32)
        return self.lib.ref_total_cost(model.handle, _p(s, C.c_float))

    def checksum(self, spins):
        s = np.ascontiguousarray(spins, np.float32)
        return self.lib.ref_checksum(_p(s, C.c_float), s.size)

    def enumerate_boltzmann(self, model, beta: float) -> dict:
        """ref: enumerate_boltzmann, src/oracle.cpp:64-109.  probabilities[state], bit i set <=> s_i = +1."""
        prob = np.empty(1 << model.n_spins, np.float64)
        mom = np.empty(3, np.float64)
        if self.lib.ref_enumerate_boltzmann(model.handle, float(beta), _p(prob, C.c_double), _p(mom, C.c_double)):
            raise ValueError(self.error())
        return dict(probabilities=prob, mean_cost=float(mom[0]), mean_magnetization=float(mom[1]),
                    log_partition=float(mom[2]))

    def chain_statistics(self, model, beta, *, engine=1, tau_scale=1.0, exp_kind=EXP_EXACT, sweeps=20000,
                         burn_in=2000, replicates=12, base_seed=1, z_threshold=4.0) -> dict:
        """ref: chain_statistics_test, src/oracle.cpp:111-174."""
        out = np.empty(9, np.float64)
        if self.lib.ref_chain_statistics(model.handle, engine, beta, tau_scale, exp_kind, sweeps, burn_in, replicates,
                                         base_seed, z_threshold, _p(out, C.c_double)):
            raise ValueError(self.error())
        keys = ("exact_cost", "exact_magnetization", "est_cost", "est_magnetization", "se_cost", "se_magnetization",
                "z_cost", "z_magnetization", "pass")
        return dict(zip(keys, out.tolist()))

    def chain(self, model, seed, beta, tau_scale=1.0, exp_kind=EXP_FAST, initial=None, engine=1):
        return RefChain(self, model, seed, beta, tau_scale, exp_kind, initial, engine)

    def ladders(self, models, n_ladders, betas, seeds, swap_seeds, tau_scale=1.0, exp_kind=EXP_FAST, engine=1):
        """Persistent set of ladders for timed multi-threaded CPU runs (bench.py's reference arm)."""
        return RefLadders(self, models, n_ladders, betas, seeds, swap_seeds, tau_scale, exp_kind, engine)


class RefLadders:
    def __init__(self, ref, models, n_ladders, betas, seeds, swap_seeds, tau_scale, exp_kind, engine):
        self.ref, self.models = ref, models
        betas = np.ascontiguousarray(betas, np.float32)
        self.n_chains = n_ladders * betas.size
        seeds = np.ascontiguousarray(seeds, np.uint32)
        swap = None if swap_seeds is None else np.ascontiguousarray(swap_seeds, np.uint32)
        handles = (C.c_void_p * n_ladders)(*[m.handle for m in models])
        self.handle = ref.lib.ref_ladders_create(handles, n_ladders, betas.size, _p(betas, C.c_float),
                                                 _p(seeds, C.c_uint32), _p(swap, C.c_uint32), tau_scale,
                                                 exp_kind, engine)
        if not self.handle:
            raise ValueError(ref.error())

    def __del__(self):
        if getattr(self, "handle", None):
            self.ref.lib.ref_ladders_free(self.handle)
            self.handle = None

    def run(self, sweeps, swap_interval, threads) -> float:
        return self.ref.lib.ref_ladders_run(self.handle, sweeps, swap_interval, threads)

    def read(self):
        flips, energy = np.zeros(self.n_chains, np.uint64), np.zeros(self.n_chains, np.float64)
        self.ref.lib.ref_ladders_read(self.handle, _p(flips, C.c_uint64), _p(energy, C.c_double))
        return flips, energy


class RefModel:
    def __init__(self, ref, csr, handle=None):
        self.ref = ref
        if handle is None:
            handle = ref.lib.ref_model_from_csr(csr["n_spins"], _p(csr["h"], C.c_float),
                                                _p(csr["offsets"], C.c_uint32), _p(csr["targets"], C.c_uint32),
                                                _p(csr["couplings"], C.c_float), _p(csr["tau_counts"], C.c_uint8),
                                                csr["layers"], csr["per_layer"])
        self.handle = handle
        self.n_spins = ref.lib.ref_model_spins(handle)

    def __del__(self):
        if getattr(self, "handle", None):
            self.ref.lib.ref_model_free(self.handle)
            self.handle = None

    def validate(self):
        """None when valid, otherwise the reference's error message."""
        return None if self.ref.lib.ref_model_validate(self.handle) == 0 else self.ref.error()

    def prepared_for(self, engine: int):
        """The reference's prepare_model_for_engine (sweep_state.cpp:292-323): (permuted model, forward)."""
        forward = np.empty(self.n_spins, np.uint32)
        handle = self.ref.lib.ref_prepare_model(self.handle, engine, _p(forward, C.c_uint32))
        if not handle:
            raise ValueError(self.ref.error())
        return type(self)(self.ref, None, handle), forward

    def to_string(self) -> str:
        """The reference's model_to_string (model_io.cpp:45-72)."""
        size = self.ref.lib.ref_model_to_string(self.handle, None, 0)
        if size < 0:
            raise ValueError(self.ref.error())
        buf = C.create_string_buffer(size + 1)
        self.ref.lib.ref_model_to_string(self.handle, buf, size)
        return buf.raw[:size].decode()

    @classmethod
    def from_string(cls, ref, text: str):
        """The reference's model_from_string (model_io.cpp:74-205); raises ValueError with its message."""
        handle = ref.lib.ref_model_from_string(text.encode())
        if not handle:
            raise ValueError(ref.error())
        return cls(ref, None, handle)

    def csr(self) -> dict:
        n, e = self.n_spins, self.ref.lib.ref_model_half_edges(self.handle)
        out = dict(n_spins=n, h=np.empty(n, np.float32), offsets=np.empty(n + 1, np.uint32),
                   targets=np.empty(e, np.uint32), couplings=np.empty(e, np.float32),
                   tau_counts=np.empty(n, np.uint8))
        self.ref.lib.ref_model_export(self.handle, _p(out["h"], C.c_float), _p(out["offsets"], C.c_uint32),
                                      _p(out["targets"], C.c_uint32), _p(out["couplings"], C.c_float),
                                      _p(out["tau_counts"], C.c_uint8))
        return out


class RefChain:
    def __init__(self, ref, model, seed, beta, tau_scale, exp_kind, initial, engine):
        self.ref, self.model = ref, model
        init = None if initial is None else np.ascontiguousarray(initial, np.int8)
        self.handle = ref.lib.ref_chain_create(model.handle, engine, seed, beta, tau_scale, exp_kind,
                                               _p(init, C.c_int8))
        if not self.handle:
            raise ValueError(ref.error())
        self.n = model.n_spins

    def __del__(self):
        if getattr(self, "handle", None):
            self.ref.lib.ref_chain_free(self.handle)
            self.handle = None

    def sweep(self, sweeps: int = 1):
        self.ref.lib.ref_chain_sweep(self.handle, self.model.handle, sweeps)

    def set_beta(self, beta):
        self.ref.lib.ref_chain_set_beta(self.handle, beta)

    def _read(self):
        s, hs, ht = (np.empty(self.n, np.float32) for _ in range(3))
        flips, attempts = C.c_uint64(), C.c_uint64()
        self.ref.lib.ref_chain_read(self.handle, _p(s, C.c_float), _p(hs, C.c_float), _p(ht, C.c_float),
                                    C.byref(flips), C.byref(attempts))
        return s, hs, ht, flips.value, attempts.value

    spins = property(lambda self: self._read()[0])
    hs = property(lambda self: self._read()[1])
    ht = property(lambda self: self._read()[2])
    flips = property(lambda self: self._read()[3])
    attempts = property(lambda self: self._read()[4])

    def coherence(self):
        return self.ref.lib.ref_chain_coherence(self.handle, self.model.handle)

    def flip_probability(self, spin):
        return self.ref.lib.ref_flip_probability(self.handle, spin)
