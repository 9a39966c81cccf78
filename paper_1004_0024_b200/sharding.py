"""Multi-GPU plan for the batched sweep path: whole ladders are dealt to ranks in contiguous
blocks, seeds are functions of the GLOBAL chain / ladder index, so every chain's bits are the
same at 1, 2, 4 or 8 GPUs (the reference's worker-count invariance, ref:
proj/tests/test_bench.cpp:153-166, proj/src/bench.cpp:49-50).  There is no collective on the
data path; the only exchange is one all-gather of the packed per-chain results at the end.

torch.distributed is plumbing here (NCCL over NVLink on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Tuple

import numpy as np

RECORD_WORDS = 4  # {energy f64, running energy f64, flips u64, checksum u64} = 32 bytes per chain


def shard_ladders(n_ladders: int, rank: int, world: int) -> Tuple[int, int]:
    """(first_ladder, count) of rank's contiguous block; blocks differ by at most one ladder."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    base, extra = divmod(n_ladders, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def chain_seeds(base_seed: int, first_ladder: int, n_ladders: int, n_betas: int) -> np.ndarray:
    """Sweep-stream seeds of a shard: base + global chain id (ref lane-seed rule, sweep.hpp:59)."""
    first_chain = first_ladder * n_betas
    return ((base_seed + first_chain + np.arange(n_ladders * n_betas, dtype=np.uint64)) & 0xFFFFFFFF).astype(np.uint32)


def ladder_seeds(base_seed: int, first_ladder: int, n_ladders: int) -> np.ndarray:
    return ((base_seed + first_ladder + np.arange(n_ladders, dtype=np.uint64)) & 0xFFFFFFFF).astype(np.uint32)


def pack_records(energy, e_run, flips, checksum) -> np.ndarray:
    """Host-side twin of ising_batch_pack_results: int64 [chains, 4] with the f64 fields bit-cast."""
    out = np.empty((len(energy), RECORD_WORDS), np.int64)
    out[:, 0] = np.asarray(energy, np.float64).view(np.int64)
    out[:, 1] = np.asarray(e_run, np.float64).view(np.int64)
    out[:, 2] = np.asarray(flips, np.uint64).view(np.int64)
    out[:, 3] = np.asarray(checksum, np.uint64).view(np.int64)
    return out


def unpack_records(rec: np.ndarray) -> dict:
    rec = np.ascontiguousarray(rec, np.int64).reshape(-1, RECORD_WORDS)
    return dict(energy=rec[:, 0].copy().view(np.float64), e_run=rec[:, 1].copy().view(np.float64),
                flips=rec[:, 2].copy().view(np.uint64), checksum=rec[:, 3].copy().view(np.uint64))


def all_gather_records(local, counts):
    """Gathers every rank's [chains_r, 4] int64 record tensor into one [sum chains, 4] tensor in
    global chain order.  `local` is a torch tensor on the communicator's device (CUDA for NCCL,
    CPU for gloo); `counts` lists every rank's chain count (equal counts use one all_gather_into_tensor)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size()
    assert len(counts) == world
    if len(set(counts)) == 1:
        out = torch.empty((world * counts[0], RECORD_WORDS), dtype=torch.int64, device=local.device)
        dist.all_gather_into_tensor(out, local.contiguous())
        return out
    # uneven blocks: pad to the largest, gather once, trim
    widest = max(counts)
    padded = torch.zeros((widest, RECORD_WORDS), dtype=torch.int64, device=local.device)
    padded[: local.shape[0]] = local
    out = torch.empty((world * widest, RECORD_WORDS), dtype=torch.int64, device=local.device)
    dist.all_gather_into_tensor(out, padded)
    return torch.cat([out[r * widest: r * widest + c] for r, c in enumerate(counts)], 0)
