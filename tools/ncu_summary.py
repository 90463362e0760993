#!/usr/bin/env python
"""Summarise ncu captures for profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py launches gpurun_out/launches.csv        -> per-kernel share of device time
  python tools/ncu_summary.py full gpurun_out/prof_stream.ncu-rep     -> key counters of the captured kernel
  python tools/ncu_summary.py full gpurun_out/prof_stream_raw.csv     -> the same from its --page raw --csv export
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum", "lts__t_requests_op_red.sum", "lts__t_sectors_op_red.sum",
    "smsp__average_warp_latency_issue_stalled_barrier", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].split("<")[0]
        tot[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
    all_ns = sum(tot.values())
    print(f"{'kernel':40s} {'launches':>8s} {'avg_us':>10s} {'share':>7s}")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{k:40s} {cnt[k]:8d} {v / cnt[k] / 1e3:10.1f} {100 * v / all_ns:6.1f}%")


def full(path):
    # an .ncu-rep, or the `--page raw --csv` export of one (tools/gpu_run.sh keeps only that)
    if path.endswith(".csv"):
        out = open(path).read()
    else:
        out = subprocess.check_output(["ncu", "-i", path, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(out)))
    rows = rows[next(i for i, r in enumerate(rows) if "Kernel Name" in r or "ID" in r[:2]):]
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print("kernel:", name[:120])
        for k in KEYS:
            for i, h in enumerate(hdr):
                if h == k:
                    print(f"  {k:70s} {r[i]:>20s} {units[i]}")
        stalls = [(h, r[i]) for i, h in enumerate(hdr) if h.startswith("smsp__average_warp_latency_issue_stalled_") or
                  h.startswith("smsp__pcsamp_warps_issue_stalled_")]
        vals = []
        for h, v in stalls:
            try:
                vals.append((float(v.replace(",", "")), h))
            except ValueError:
                pass
        print("  top stall reasons:")
        for v, h in sorted(vals, reverse=True)[:10]:
            print(f"    {h:80s} {v:12.2f}")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
