"""ctypes binding of libisingb200.so — the stub a maintainer of the reference would write to
call the new C ABI (include/isingmc_b200.h).  No torch types cross this boundary: plain
pointers and sizes only.  The library must exist; there is no Python or CPU fallback."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libisingb200.so"

ISING_OK, ISING_ERR_ARGUMENT, ISING_ERR_PARSE, ISING_ERR_IO, ISING_ERR_INTERNAL = range(5)
EXP_DEFAULT, EXP_EXACT, EXP_FAST, EXP_ACCURATE = range(4)
KERNEL_AUTO, KERNEL_GENERIC, KERNEL_LAYERED, KERNEL_STRAND = range(4)

u8p, i8p = C.POINTER(C.c_uint8), C.POINTER(C.c_int8)
u32p, u64p = C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)
f32p, f64p = C.POINTER(C.c_float), C.POINTER(C.c_double)


class BatchParams(C.Structure):
    _fields_ = [
        ("n_ladders", C.c_uint32), ("n_betas", C.c_uint32), ("betas", f32p), ("seeds", u32p),
        ("swap_seeds", u32p), ("base_seed", C.c_uint32), ("swap_base_seed", C.c_uint32),
        ("first_ladder", C.c_uint64), ("tau_scale", C.c_float), ("exp_kind", C.c_int),
        ("device", C.c_int), ("kernel", C.c_int), ("initial_spins", i8p),
    ]


class BatchInfo(C.Structure):
    _fields_ = [
        ("n_chains", C.c_uint64), ("n_spins", C.c_uint32), ("n_tiles", C.c_uint32),
        ("kernel", C.c_int), ("sweeps_done", C.c_uint64), ("device_bytes", C.c_uint64),
        ("sweep_launches", C.c_uint64), ("swap_launches", C.c_uint64),
        ("other_launches", C.c_uint64), ("sweep_ms", C.c_double), ("swap_ms", C.c_double),
        ("last_run_ms", C.c_double), ("generic_variant", C.c_uint32), ("strands", C.c_uint32),
    ]


class CoalescedParams(C.Structure):
    _fields_ = [("n_chains", C.c_uint32), ("betas", f32p), ("seeds", u32p), ("base_seed", C.c_uint32),
                ("tau_scale", C.c_float), ("exp_kind", C.c_int), ("device", C.c_int), ("initial_spins", i8p)]


class CoalescedInfo(C.Structure):
    _fields_ = [("n_chains", C.c_uint64), ("n_spins", C.c_uint32), ("lanes", C.c_uint32),
                ("sweeps_done", C.c_uint64), ("launches", C.c_uint64), ("last_run_ms", C.c_double)]


class RunParams(C.Structure):
    _fields_ = [("sweeps", C.c_uint64), ("beta", C.c_float), ("tau_scale", C.c_float),
                ("exp_kind", C.c_int), ("seed", C.c_uint32), ("device", C.c_int)]


class RunReport(C.Structure):
    _fields_ = [("final_cost", C.c_double), ("flip_rate", C.c_double), ("flips", C.c_uint64),
                ("attempts", C.c_uint64), ("checksum", C.c_uint64)]


# name -> (restype, argtypes); the complete export list of include/isingmc_b200.h
SIGNATURES = {
    "ising_b200_last_error": (C.c_char_p, []),
    "ising_b200_device_count": (C.c_int, []),
    "ising_b200_model_from_csr": (C.c_int, [C.c_uint32, f32p, u32p, u32p, f32p, u8p, C.c_uint32,
                                            C.c_uint32, C.POINTER(C.c_void_p)]),
    "ising_b200_model_build_layered": (C.c_int, [C.c_uint32, f32p, C.c_uint32, u32p, u32p, f32p,
                                                 C.c_uint32, C.c_float, C.POINTER(C.c_void_p)]),
    "ising_b200_model_free": (None, [C.c_void_p]),
    "ising_b200_model_spins": (C.c_uint32, [C.c_void_p]),
    "ising_b200_model_half_edges": (C.c_uint64, [C.c_void_p]),
    "ising_b200_model_layers": (C.c_int, [C.c_void_p, u32p, u32p]),
    "ising_b200_model_export_csr": (C.c_int, [C.c_void_p, f32p, u32p, u32p, f32p, u8p]),
    "ising_b200_model_cost": (C.c_int, [C.c_void_p, i8p, C.c_uint32, f64p]),
    "ising_batch_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_uint32, u32p,
                                     C.POINTER(BatchParams), C.POINTER(C.c_void_p)]),
    "ising_batch_free": (None, [C.c_void_p]),
    "ising_batch_run": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32]),
    "ising_batch_swap": (C.c_int, [C.c_void_p]),
    "ising_batch_sync": (C.c_int, [C.c_void_p]),
    "ising_batch_read_spins": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, i8p]),
    "ising_batch_read_fields": (C.c_int, [C.c_void_p, C.c_uint64, f32p, f32p]),
    "ising_batch_read_energies": (C.c_int, [C.c_void_p, f64p]),
    "ising_batch_read_running_energies": (C.c_int, [C.c_void_p, f64p]),
    "ising_batch_resync_energies": (C.c_int, [C.c_void_p]),
    "ising_batch_read_stats": (C.c_int, [C.c_void_p, u64p, u64p]),
    "ising_batch_checksums": (C.c_int, [C.c_void_p, u64p]),
    "ising_batch_field_coherence": (C.c_int, [C.c_void_p, u64p]),
    "ising_batch_read_slots": (C.c_int, [C.c_void_p, u32p]),
    "ising_batch_read_swap_stats": (C.c_int, [C.c_void_p, u64p, u64p]),
    "ising_batch_pack_results": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ising_batch_all_gather_results": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "ising_batch_set_timing": (C.c_int, [C.c_void_p, C.c_int]),
    "ising_batch_record_wait": (C.c_int, [C.c_void_p, C.c_int]),
    "ising_batch_read_wait_stats": (C.c_int, [C.c_void_p, C.c_uint32, u32p, f64p, u64p, u64p]),
    "ising_batch_get_info": (C.c_int, [C.c_void_p, C.POINTER(BatchInfo)]),
    "ising_batch_stream": (C.c_void_p, [C.c_void_p]),
    "ising_coalesced_create": (C.c_int, [C.c_void_p, C.POINTER(CoalescedParams), C.POINTER(C.c_void_p)]),
    "ising_coalesced_free": (None, [C.c_void_p]),
    "ising_coalesced_run": (C.c_int, [C.c_void_p, C.c_uint64]),
    "ising_coalesced_read_spins": (C.c_int, [C.c_void_p, C.c_uint64, i8p]),
    "ising_coalesced_read_fields": (C.c_int, [C.c_void_p, C.c_uint64, f32p, f32p]),
    "ising_coalesced_read_stats": (C.c_int, [C.c_void_p, u64p, u64p]),
    "ising_coalesced_read_energies": (C.c_int, [C.c_void_p, f64p]),
    "ising_coalesced_checksums": (C.c_int, [C.c_void_p, u64p]),
    "ising_coalesced_get_info": (C.c_int, [C.c_void_p, C.POINTER(CoalescedInfo)]),
    "ising_b200_run": (C.c_int, [C.c_void_p, C.POINTER(RunParams), C.POINTER(RunReport)]),
    "ising_b200_run_json": (C.c_int, [C.c_void_p, C.POINTER(RunParams), C.POINTER(RunReport),
                                      C.POINTER(C.c_void_p)]),
    "ising_b200_model_from_string": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "ising_b200_model_to_string": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "ising_b200_model_load": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "ising_b200_model_save": (C.c_int, [C.c_void_p, C.c_char_p]),
    "ising_b200_string_free": (None, [C.c_void_p]),
}

_lib = None


def load() -> C.CDLL:
    """Loads the CUDA library or fails loudly — the product path has no fallback."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1004_0024_b200.build` "
                "(this engine has no CPU fallback)")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib
