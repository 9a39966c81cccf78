#!/usr/bin/env python
"""Headline benchmark: spin-flip attempts/s of batched Metropolis sweeps under parallel tempering.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5] [--impl ours|reference]

A "step" is one pass of the hot path over the whole batch: `swap_interval` sweeps of every chain
followed by one tempering swap round (10 sweeps + 1 swap round for the default workload c5, the
configuration BASELINE.json's metric is quoted on: 32,768-spin layered instance, 16,384 chains per
GPU).  Weak scaling: chains per GPU are fixed, ladders are sharded by global index, no collective
on the data path, one NCCL all-gather of the 32-byte per-chain results at the end of the e2e run.

Prints ONE JSON line (rank 0).  `value` is device-timed with the state resident in HBM; `e2e` is
the same metric through the C ABI with host buffers (model/seed upload, device init, per-step
host readout of the statistics, final energies/checksums readout) on the wall clock.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "spin_flip_attempts_per_sec"
UNIT = "attempts/s"
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)  # 100 steps x 10 sweeps = the 1000 sweeps of c5
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c5", choices=["c1", "c2", "c3", "c4", "c5", "all"],
                    help="all: c1..c5 one after the other, one JSON line each (see --save)")
    ap.add_argument("--save", default="", help="with --workload all: also write the lines to this JSON file")
    ap.add_argument("--ladders", type=int, default=0, help="override ladders per GPU (0: the workload's)")
    ap.add_argument("--exp", default="fast", choices=["exact", "fast", "accurate"])
    ap.add_argument("--kernel", default="auto", choices=["auto", "generic", "layered", "strand", "coalesced"],
                    help="coalesced: the intra-system schedule (one warp per chain; layered workloads, 1 GPU)")
    ap.add_argument("--chains", type=int, default=148, help="chains for --kernel coalesced")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-ladders", type=int, default=0, help="CPU sample size in ladders (0: auto)")
    return ap.parse_args()


def peak_hbm():
    path = ROOT / "MEASURED_PEAKS.json"
    if path.exists():
        try:
            return float(json.loads(path.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
        except Exception:
            pass
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.tmp = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.proc = None
        self.device_index = device_index

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.device_index)], stdout=self.tmp, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.tmp.flush()
        rows = [r.split(",") for r in Path(self.tmp.name).read_text().strip().splitlines() if r.strip()]
        os.unlink(self.tmp.name)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                smax.append(float(r[2]))
            except (ValueError, IndexError):
                continue
            for name, cell in zip(names, r[5:9]):
                if cell.strip().lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(smax)), "reasons": sorted(reasons),
                "samples": len(sm)}



def config_of(wl, exp_name, sweeps_per_step, world):
    """The `config` object of the JSON line — the same keys and values in both arms."""
    return {"workload": f"{wl.name}: {wl.description}", "chains_per_gpu": int(wl.n_ladders * len(wl.betas)),
            "sweeps_per_step": int(sweeps_per_step), "swap_interval": int(wl.swap_interval), "exp_kind": exp_name,
            "l2": "per-GPU state streamed every sweep (far larger than the 126 MB L2 at full size), no explicit flush",
            "parallelism": f"ladders sharded over {world} GPU(s), no data-path collective"}


def kernel_source_hash() -> str:
    """Identifies the kernel sources a DRAM-traffic profile was taken with (profiles/sweep_traffic.json)."""
    import hashlib
    h = hashlib.sha256()
    for name in ("kernels_strand.cu", "kernels_layered.cu", "kernels_generic.cu", "device_math.cuh", "device_mt.cuh"):
        h.update((ROOT / "paper_1004_0024_b200" / "csrc" / name).read_bytes())
    return h.hexdigest()[:16]


def profiled_traffic(workload: str, kernel: int, attempts_per_launch: float):
    """DRAM bytes per launch from the committed ncu capture of this workload and kernel family, or
    (None, why): a capture taken with other kernel sources is refused."""
    prof = ROOT / "profiles" / "sweep_traffic.json"
    if not prof.exists():
        return None, "no ncu capture committed"
    try:
        entry = json.loads(prof.read_text()).get(f"{workload}:{kernel}")
    except Exception as exc:  # malformed file: say so, do not guess
        return None, f"unreadable profile: {exc}"
    if entry is None:
        return None, "no ncu capture of this workload and kernel family"
    if entry.get("kernel_source_hash") != kernel_source_hash():
        return None, f"stale: capture {entry.get('source')} was taken with other kernel sources"
    return entry["dram_bytes_per_attempt"] * attempts_per_launch, entry.get("source")


def free_port() -> int:
    import socket
    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        return sock.getsockname()[1]

def build_models(wl, csrs):
    """One product model per instance (validation and layer analysis run in C++ with the GIL released, so
    workloads with many distinct instances build them on a few host threads)."""
    import paper_1004_0024_b200 as ib
    from concurrent.futures import ThreadPoolExecutor

    def one(c):
        return ib.SpinModel.from_csr(c["n_spins"], c["h"], c["offsets"], c["targets"], c["couplings"],
                                     c["tau_counts"], c["layers"], c["per_layer"])
    if len(csrs) < 4:
        return [one(c) for c in csrs]
    with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as pool:
        return list(pool.map(one, csrs))


def model_bytes(csrs) -> int:
    return int(sum(c["h"].nbytes + c["offsets"].nbytes + c["targets"].nbytes + c["couplings"].nbytes +
                   (0 if c["tau_counts"] is None else c["tau_counts"].nbytes) for c in csrs))


def cpu_baseline(wl, csrs, exp_kind, sample_ladders, sweeps_per_step, steps, warmup, engine=1):
    """Times the reference's CPU path (oracle/_ref when built, else the C port) on a bounded sample
    of the same workload, all host cores.  engine 1: `basic`, the tier the GPU path is bit-exact
    with; engine 2: `vector4` on the reference's own permuted model (its fastest tier: another
    trajectory, timing only, reference library only).  Returns (dict, seconds_per_step)."""
    from oracle import pyoracle
    from paper_1004_0024_b200 import instances as ins
    cores = os.cpu_count() or 1
    nb = len(wl.betas)
    ladders = sample_ladders
    seeds = (ins.CHAIN_SEED_BASE + np.arange(ladders * nb)).astype(np.uint32)
    swap_seeds = (ins.SWAP_SEED_BASE + np.arange(ladders)).astype(np.uint32)
    pick = (lambda l: 0) if wl.shared_graph else (lambda l: l % len(csrs))
    pyoracle.build(ref=True)
    if pyoracle.Reference.available():
        ref = pyoracle.Reference()
        models = [ref.model(c) for c in csrs]
        if engine == 2:
            models = [m.prepared_for(2)[0] for m in models]
        lad = ref.ladders([models[pick(l)] for l in range(ladders)], ladders, wl.betas, seeds, swap_seeds, 1.0,
                          exp_kind, engine)
        for _ in range(warmup):
            lad.run(sweeps_per_step, wl.swap_interval, cores)
        secs = sum(lad.run(sweeps_per_step, wl.swap_interval, cores) for _ in range(steps))
        kind = "reference"
    elif engine != 1:
        return None, None
    else:
        port = pyoracle.Port()
        models = [port.model(c) for c in csrs]
        per = [models[pick(l)] for l in range(ladders)]
        total = sweeps_per_step * (steps + warmup)
        t0 = time.perf_counter()
        port.pt_run(per, ladders, wl.betas, seeds, swap_seeds, total, wl.swap_interval, 1.0, exp_kind, cores,
                    want_spins=False)
        secs = (time.perf_counter() - t0) * steps / (steps + warmup)  # includes state setup
        kind = "port"
    attempts = ladders * nb * csrs[0]["n_spins"] * sweeps_per_step * steps
    tier = "basic" if engine == 1 else "vector4 (another trajectory: timing only)"
    sample = (f"{ladders} ladders x {nb} betas = {ladders * nb} chains of {csrs[0]['n_spins']} spins, "
              f"{sweeps_per_step * steps} sweeps (swap every {wl.swap_interval}), {tier} engine / "
              f"{exp_kind_name(exp_kind)} exp")
    return {"value": attempts / secs, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample}, secs / steps


def exp_kind_name(k):
    return {1: "exact", 2: "fast", 3: "accurate"}[k]


def bench_coalesced(args, wl, exp_kind):
    """The intra-system (coalesced) family on a layered workload: `--chains` independent chains of the
    workload's first instance, one warp each.  One JSON line in the same shape as the main arm; the
    CPU baseline is the reference's own coalesced engine on one host thread per chain sample."""
    import paper_1004_0024_b200 as ib
    from paper_1004_0024_b200 import instances as ins
    c = wl.make_csrs()[0]
    if not c["layers"]:
        raise SystemExit("--kernel coalesced needs a layered workload (c4 or c5)")
    n = c["n_spins"]
    model = ib.SpinModel.from_csr(n, c["h"], c["offsets"], c["targets"], c["couplings"], c["tau_counts"],
                                  c["layers"], c["per_layer"])
    betas = np.resize(np.asarray(wl.betas, np.float32), args.chains)
    sweeps_per_step = 10
    state = ib.init_coalesced(model, betas, base_seed=ins.CHAIN_SEED_BASE, params=ib.SweepParams(1.0, exp_kind))
    for _ in range(args.warmup):
        state.run(sweeps_per_step)
    state.info()
    sampler = ClockSampler(0)
    sampler.start()
    state.run(sweeps_per_step * args.steps)
    ms = state.info()["last_run_ms"]
    clocks = sampler.stop()
    flips, attempts = state.stats()
    value = args.chains * n * sweeps_per_step * args.steps / (ms * 1e-3)
    t0 = time.perf_counter()
    again = ib.init_coalesced(model, betas, base_seed=ins.CHAIN_SEED_BASE, params=ib.SweepParams(1.0, exp_kind))
    for _ in range(args.steps):
        again.run(sweeps_per_step)
        again.stats()
    energies = again.energies()
    wall = time.perf_counter() - t0
    again.close()
    flip_rate = float(flips.sum()) / float(attempts.sum())
    dbar = float(len(c["targets"])) / n
    bytes_per_attempt = 9.0 + flip_rate * (1.0 + 8.0 * dbar)
    peak, peak_src = peak_hbm()
    achieved = bytes_per_attempt * value / 1e9
    base = None
    if not args.no_cpu_baseline:
        from oracle import pyoracle
        pyoracle.build(ref=True)
        sample = min(args.chains, 4)
        if pyoracle.Reference.available():
            ref = pyoracle.Reference()
            permuted, _ = ref.model(c).prepared_for(3)
            chains = [ref.chain(permuted, ins.CHAIN_SEED_BASE + 32 * k, float(betas[k]), 1.0, exp_kind, None, engine=3)
                      for k in range(sample)]
            kind = "reference"
        else:
            port = pyoracle.Port()
            chains = [port.coalesced(port.model(c), ins.CHAIN_SEED_BASE + 32 * k, float(betas[k]), 1.0, exp_kind)
                      for k in range(sample)]
            kind = "port"
        t1 = time.perf_counter()
        for ch in chains:
            ch.sweep(40)
        secs = time.perf_counter() - t1
        base = {"value": sample * n * 40 / secs, "unit": UNIT, "cores": 1, "kind": kind,
                "sample": f"{sample} chains x 40 sweeps of the coalesced engine, one host thread"}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{wl.name} instance, {args.chains} independent chains, intra-system (coalesced) "
                                   f"schedule, {sweeps_per_step * args.steps} sweeps", "chains_per_gpu": args.chains,
                       "n_spins": n, "sweeps_per_step": sweeps_per_step, "exp_kind": args.exp,
                       "kernel_family": "sweep_coalesced",
                       "l2": "state of the chains is L2 resident; the kernel is latency bound (see DESIGN.md 4.5)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": None, "peak_source": peak_src, "bytes_per_attempt": bytes_per_attempt,
                         "flip_rate": flip_rate, "mean_degree": dbar, "kernel": "sweep_coalesced",
                         "kernel_ms_per_launch": ms},
            "cpu_baseline": base,
            "e2e": {"value": args.chains * n * sweeps_per_step * args.steps / wall, "unit": UNIT,
                    "h2d_bytes_per_step": (state.n_chains * n * 9 + model_bytes([c])) / args.steps,
                    "d2h_bytes_per_step": 16 * args.chains + energies.nbytes / args.steps,
                    "includes": "host init_state (permutation, fields), upload, K steps with per-step flip counts, "
                                "final energies (host f64 from downloaded spins)"},
            "gpu_launches": int(state.info()["launches"]) - args.warmup, "clocks": clocks}
    state.close()
    print(json.dumps(line), flush=True)


def respawn_ranks(args) -> int:
    """`python bench.py --gpus N` with N > 1 and no launcher around it: start N ranks of this very
    command under torch.distributed.run (one per GPU, NCCL over 127.0.0.1) and wait for them."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} asked, {have} CUDA device(s) visible",
                          "n_gpus": args.gpus}), flush=True)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def main():
    args = parse_args()
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.kernel != "coalesced":
        raise SystemExit(respawn_ranks(args))
    names = ["c1", "c2", "c3", "c4", "c5"] if args.workload == "all" else [args.workload]
    lines = []
    for name in names:
        line = run_workload(args, name)
        if line is not None:
            print(json.dumps(line), flush=True)
            lines.append(line)
    if args.save and lines:
        Path(args.save).write_text(json.dumps(lines, indent=1) + "\n")
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()


def run_workload(args, name):
    """One workload, this rank; returns the JSON line on rank 0 (None elsewhere)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    exp_kind = {"exact": 1, "fast": 2, "accurate": 3}[args.exp]

    from paper_1004_0024_b200 import workloads
    wl = workloads.get(name)
    if args.kernel == "coalesced":
        if rank == 0 and args.impl == "ours":
            bench_coalesced(args, wl, exp_kind)
        return None
    if args.ladders:
        wl.n_ladders = args.ladders
    sweeps_per_step = wl.swap_interval if wl.swap_interval else 10
    nb = len(wl.betas)

    # ------------------------------------------------------------------ reference arm (CPU)
    if args.impl == "reference":
        if rank != 0:
            return None
        csrs = wl.make_csrs() if wl.shared_graph else wl.make_csrs()[: max(1, min(wl.n_ladders, 8))]
        n = csrs[0]["n_spins"]
        sample = args.cpu_ladders or max(1, min(wl.n_ladders, int(4.0e8 // (nb * n * sweeps_per_step)) or 1))
        base, per_step = cpu_baseline(wl, csrs, exp_kind, sample, sweeps_per_step, args.steps, args.warmup)
        config = config_of(wl, args.exp, sweeps_per_step, max(world, args.gpus))
        config["n_spins"] = int(n)
        return {
            "impl": "reference", "metric": METRIC, "value": base["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": config,
            "cpu_baseline": base,
            "e2e": {"value": base["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0,
        }

    # ------------------------------------------------------------------ our arm (GPU)
    import torch
    import torch.distributed as dist
    import paper_1004_0024_b200 as ib
    from paper_1004_0024_b200 import build as libbuild, instances as ins
    libbuild.build()

    torch.cuda.set_device(local_rank)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    csrs = wl.make_csrs()
    if not wl.shared_graph:
        csrs = [csrs[(rank * wl.n_ladders + l) % len(csrs)] for l in range(wl.n_ladders)]
    n = csrs[0]["n_spins"]
    dbar = float(np.mean([workloads.mean_degree(c) for c in csrs[:8]]))
    kernel = {"auto": ib.KERNEL_AUTO, "generic": ib.KERNEL_GENERIC, "layered": ib.KERNEL_LAYERED,
              "strand": ib.KERNEL_STRAND}[args.kernel]
    first_ladder = rank * wl.n_ladders

    def make_state():
        models = build_models(wl, csrs)
        return ib.init_state(models, wl.betas, wl.n_ladders, base_seed=ins.CHAIN_SEED_BASE,
                             swap_base_seed=ins.SWAP_SEED_BASE, first_ladder=first_ladder,
                             params=ib.SweepParams(1.0, exp_kind), device=local_rank, kernel=kernel)

    state = make_state()
    chains = state.n_chains
    attempts_per_step = chains * n * sweeps_per_step

    # ---- device-timed run: W warm-up steps, then exactly K steps
    for _ in range(args.warmup):
        state.run(sweeps_per_step, wl.swap_interval)
    state.sync()
    before = state.info()
    flips0 = state.stats()[0].sum()
    state.set_timing(True)
    sampler = ClockSampler(local_rank)
    sampler.start()
    barrier()
    state.run(sweeps_per_step * args.steps, wl.swap_interval)  # exactly K steps, enqueued back to back
    state.sync()
    barrier()
    clocks = sampler.stop()
    after = state.info()
    state.set_timing(False)
    # CUDA events on the batch's own stream around the K steps (gaps between launches included)
    ms = after["last_run_ms"]
    flips = int(state.stats()[0].sum() - flips0)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total_attempts = attempts_per_step * args.steps * world
    value = total_attempts / (ms_max * 1e-3)
    sweep_launches = after["sweep_launches"] - before["sweep_launches"]
    swap_launches = after["swap_launches"] - before["swap_launches"]
    other_launches = after["other_launches"] - before["other_launches"]
    sweep_ms = after["sweep_ms"] - before["sweep_ms"]

    # ---- roofline of the sweep kernel (this rank): algorithmic bytes B = S + f*(1 + 8*dbar)
    flip_rate = flips / float(attempts_per_step * args.steps)
    bytes_per_attempt = wl.state_bytes_per_spin + flip_rate * (1.0 + 8.0 * dbar)
    peak, peak_src = peak_hbm()
    achieved = bytes_per_attempt * attempts_per_step * args.steps / (sweep_ms * 1e-3) / 1e9
    traffic, traffic_src = profiled_traffic(wl.name, after["kernel"],
                                            attempts_per_step * args.steps / max(1, sweep_launches))
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
                "bytes_per_attempt": bytes_per_attempt, "flip_rate": flip_rate, "mean_degree": dbar,
                "kernel": {1: "sweep_generic", 2: "sweep_layered", 3: "sweep_strand"}[after["kernel"]],
                "strands_per_tile": after.get("strands", 0),
                "kernel_ms_per_launch": sweep_ms / max(1, sweep_launches),
                "roofline_attempts_per_sec": peak * 1e9 / bytes_per_attempt}
    info = after
    state.close()

    # ---- end to end through the C ABI with host buffers
    e2e = None
    if not args.no_e2e:
        barrier()
        t0 = time.perf_counter()
        st = make_state()  # H2D: graphs, seeds, betas; device-side init_state
        d2h = 0
        for _ in range(args.steps):
            st.run(sweeps_per_step, wl.swap_interval)
            fl, _att = st.stats()          # D2H per step: accept counts
            er = st.running_energies()     # D2H per step: energies used by the swap rule
            d2h += fl.nbytes + er.nbytes
        if world > 1:  # one NCCL all-gather of the packed per-chain results, no host round trip
            from paper_1004_0024_b200 import sharding
            rec = torch.empty((chains, sharding.RECORD_WORDS), dtype=torch.int64, device="cuda")
            st.pack_results(rec.data_ptr())
            allrec = sharding.all_gather_records(rec, [chains] * world)
            host = allrec.cpu() if rank == 0 else None  # noqa: F841 (the read-back is the point)
            d2h_final = world * chains * 32 if rank == 0 else 0
        else:
            en, cs = st.energies(), st.checksums()
            d2h_final = en.nbytes + cs.nbytes
        sample_spins = st.spins(0, min(chains, 16))  # parity sample read back as int8
        d2h_final += sample_spins.nbytes
        st.sync()
        barrier()
        wall = time.perf_counter() - t0
        st.close()
        tw = torch.tensor([wall], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tw, op=dist.ReduceOp.MAX)
        h2d = model_bytes(csrs if not wl.shared_graph else csrs[:1]) + chains * 4 + wl.n_ladders * 4 + nb * 4
        e2e = {"value": total_attempts / float(tw.item()), "unit": UNIT,
               "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": (d2h + d2h_final) / args.steps,
               "includes": "graph/seed upload, device init_state, K steps with per-step host readout of accept "
                           "counts and running energies, final energies+checksums" +
                           (" via NCCL all-gather" if world > 1 else "") + ", 16-chain spin readout"}

    # ---- CPU baselines beside it (rank 0, N = 1 only): the tier the GPU path is bit-exact with, and
    # for layered workloads the reference's fastest tier (vector4 on its own permuted model)
    base = best = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sample = args.cpu_ladders or max(1, min(wl.n_ladders, int(2.0e9 // (nb * n * sweeps_per_step * 4)) or 1))
        some = csrs[:8] if not wl.shared_graph else csrs
        base, _ = cpu_baseline(wl, some, exp_kind, sample, sweeps_per_step, 4, 1)
        if csrs[0]["layers"]:
            best, _ = cpu_baseline(wl, some, exp_kind, sample, sweeps_per_step, 4, 1, engine=2)

    if rank != 0:
        return None
    config = config_of(wl, args.exp, sweeps_per_step, world)
    config["n_spins"] = int(n)
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config, "first_ladder_of_rank": [r * wl.n_ladders for r in range(world)],
        "device_bytes_per_gpu": int(info["device_bytes"]),
        "roofline": roofline, "cpu_baseline": base, "cpu_baseline_best": best, "e2e": e2e,
        # the strand family brackets its sweep kernel with two small conversion kernels (spin words <-> bytes)
        "gpu_launches": int(sweep_launches + swap_launches + other_launches),
        "launch_breakdown": {"sweep": int(sweep_launches), "swap": int(swap_launches),
                             "spin_format_conversions": int(other_launches)},
        "clocks": clocks,
    }


if __name__ == "__main__":
    main()
