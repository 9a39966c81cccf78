"""Refreshes the committed round-2 artefacts from a capture brought back in gpurun_out/:
python profiles/refresh_r02.py TAG   (after `ncu -i gpurun_out/r02_TAG_full.ncu-rep --page raw --csv > /tmp/TAG_raw.csv`)"""
import csv
import json
import shutil
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402

tag = sys.argv[1]
shutil.copy(f"gpurun_out/r02_{tag}_launches.csv", "profiles/r02_launches_gpu_time_duration.csv")
shutil.copy("gpurun_out/r02_workloads.json", "profiles/r02_workloads.json")
shutil.copy("gpurun_out/r02_bench_c5.json", "profiles/r02_bench_c5.json")
rows = list(csv.reader(open(f"/tmp/{tag}_raw.csv")))
h, u, v = rows[0], rows[1], rows[2]
keep = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct", "lts__t_bytes.sum",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__icc_request_hit_rate.pct",
        "smsp__average_warps_issue_stalled"]
with open("profiles/r02_strand_ncu_metrics.csv", "w") as f:
    w = csv.writer(f)
    w.writerow(["metric", "unit", "value"])
    for a, b, c in zip(h, u, v):
        if any(a.startswith(k) for k in keep) and "per_second" not in a:
            w.writerow([a, b, c])
d = {r[0]: r[2] for r in csv.reader(open("profiles/r02_strand_ncu_metrics.csv"))}
for k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
          "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "launch__shared_mem_per_block_dynamic"):
    print(k, d[k])
rd, wr = float(d["dram__bytes_read.sum"]) * 1e9, float(d["dram__bytes_write.sum"]) * 1e9
attempts = 16384 * 32768 * 10
t = json.load(open("profiles/sweep_traffic.json"))
t["c5:3"] = {"dram_bytes_per_attempt": round((rd + wr) / attempts, 3), "dram_bytes_read": rd, "dram_bytes_write": wr,
             "attempts_in_profiled_launch": attempts, "kernel_source_hash": bench.kernel_source_hash(),
             "source": "profiles/r02_strand_ncu_summary.md, r02_strand_ncu_metrics.csv (ncu --set full --clock-control none, "
                       "one launch of sweep_strand_kernel<fast, staged>, profiles/capture_r02.sh)"}
json.dump(t, open("profiles/sweep_traffic.json", "w"), indent=2)
print(t["c5:3"])
b = json.loads(open("profiles/r02_bench_c5.json").read().strip().splitlines()[-1])
print("c5", b["value"], b["ms_per_step"], b["roofline"]["frac"], b["e2e"]["value"], b["cpu_baseline"]["value"],
      b["cpu_baseline_best"]["value"], b["clocks"])
for e in json.load(open("profiles/r02_workloads.json")):
    print(e["config"]["workload"][:40], "%.3e" % e["value"], "e2e %.3e" % e["e2e"]["value"], "frac %.3f" % e["roofline"]["frac"],
          e["roofline"]["kernel"], e["roofline"].get("strands_per_tile"))
