"""B200-native batched Metropolis sweep engine for sparse Ising systems under parallel tempering
(the data-parallel hot path of arXiv 1004.0024 / the `isingmc` reference).

The compute path is libisingb200.so (hand-written sm_100a CUDA kernels behind the C ABI declared
in include/isingmc_b200.h); this package is the ctypes binding plus the host-side mirror of the
reference's sweep interface.  There is no CPU fallback: importing works anywhere, creating a
batch needs the built library and a CUDA device.
"""
from .api import (BatchState, CoalescedState, init_coalesced, ExpKind, IsingError, LayerSpec, SpinModel, SweepParams,
                  build_layered_model, init_state, run_single, run_single_json, run_sweeps, state_checksum,
                  total_cost)
from ._lib import KERNEL_AUTO, KERNEL_GENERIC, KERNEL_LAYERED, KERNEL_STRAND

__all__ = [
    "BatchState", "CoalescedState", "init_coalesced", "ExpKind", "IsingError", "LayerSpec", "SpinModel", "SweepParams",
    "build_layered_model", "init_state", "run_single", "run_single_json", "run_sweeps", "state_checksum",
    "total_cost",
    "KERNEL_AUTO", "KERNEL_GENERIC", "KERNEL_LAYERED", "KERNEL_STRAND",
]
