"""The N>1 path on CPU: two gloo ranks each run their shard (the C oracle stands in for the GPU,
which this container lacks), gather the packed records, and must reproduce the single-process
run bit for bit — the property bench.py relies on when it shards ladders over GPUs."""
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]

WORKER = r'''
import os, sys
import numpy as np
import torch, torch.distributed as dist
sys.path.insert(0, os.environ["REPO_ROOT"])
from oracle import pyoracle
from paper_1004_0024_b200 import instances as ins, sharding

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
total_ladders, sweeps, interval = int(os.environ["T_LADDERS"]), 30, 5
betas = ins.geometric_betas(0.2, 3.0, 4)
csr = ins.build_layered_csr(*ins.layered_spec(16, 3), 4, 1.5)
port = pyoracle.Port()
model = port.model(csr)
first, count = sharding.shard_ladders(total_ladders, rank, world)
seeds = sharding.chain_seeds(1000, first, count, len(betas))
swap_seeds = sharding.ladder_seeds(77000, first, count)
res = port.pt_run([model] * count, count, betas, seeds, swap_seeds, sweeps, interval) if count else None
if count:
    sums = np.array([port.checksum(s.astype(np.float32)) for s in res["spins"]], np.uint64)
    rec = sharding.pack_records(res["energy"], res["e_run"], res["flips"], sums)
else:
    rec = np.empty((0, 4), np.int64)
counts = [sharding.shard_ladders(total_ladders, r, world)[1] * len(betas) for r in range(world)]
gathered = sharding.all_gather_records(torch.from_numpy(rec), counts)
if rank == 0:
    np.save(os.environ["OUT_FILE"], gathered.numpy())
dist.barrier()
dist.destroy_process_group()
'''


def run_world(tmp_path, world, ladders):
    import subprocess
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    out = tmp_path / f"gathered_{world}.npy"
    env = dict(os.environ, REPO_ROOT=str(ROOT), T_LADDERS=str(ladders), OUT_FILE=str(out), OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + world + os.getpid() % 200), str(script)]
    subprocess.run(cmd, check=True, env=env, timeout=300, capture_output=True)
    return np.load(out)


def test_shard_arithmetic():
    from paper_1004_0024_b200 import sharding
    for n, world in ((1024, 8), (7, 2), (5, 8), (0, 3)):
        blocks = [sharding.shard_ladders(n, r, world) for r in range(world)]
        assert blocks[0][0] == 0 and sum(c for _, c in blocks) == n
        for (f0, c0), (f1, _) in zip(blocks, blocks[1:]):
            assert f0 + c0 == f1
        assert max(c for _, c in blocks) - min(c for _, c in blocks) <= 1
    seeds = np.concatenate([sharding.chain_seeds(1000, f, c, 4) for f, c in (sharding.shard_ladders(7, r, 2) for r in range(2))])
    np.testing.assert_array_equal(seeds, sharding.chain_seeds(1000, 0, 7, 4))
    rec = sharding.pack_records([1.5, -2.0], [0.25, 3.0], [7, 2**40], [2**63 + 5, 9])
    back = sharding.unpack_records(rec)
    assert back["energy"].tolist() == [1.5, -2.0] and back["checksum"].tolist() == [2**63 + 5, 9]


@pytest.mark.parametrize("ladders", [6, 5])
def test_two_ranks_reproduce_one_rank(tmp_path, port, ladders):
    """Even and uneven splits: records gathered from 2 gloo ranks == the 1-rank records."""
    one = run_world(tmp_path, 1, ladders)
    two = run_world(tmp_path, 2, ladders)
    assert one.shape == (ladders * 4, 4)
    np.testing.assert_array_equal(one, two)
