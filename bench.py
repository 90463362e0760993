#!/usr/bin/env python
"""Benchmark of the SINET discrimination + ms-histogram hot path (BASELINE.json metric).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config c2]
  torchrun --nproc-per-node N bench.py --gpus N ...          (one rank per GPU, NCCL)

A "step" = one pass of the whole hot path over one batch: reset the
histogram, discriminate + bin every record resident in HBM (one fused
kernel), materialise untouched bins, and (N > 1) merge the per-GPU
partials with the NCCL reduce-scatter + totals all-reduce.
N == 1 runs BASELINE configs[1] (c2: 100M sessions, one day of 1 ms bins, 64
prefixes).  N > 1 is weak scaling: each rank holds a contiguous 100M-record
shard of one day of N x 100M sessions.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sessions/sec classified+histogrammed at 1/2/4/8 B200; % of HBM roofline"
UNIT = "sessions/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default=None, help="c1..c5 (default c2 at N=1, weak-scaled c2 at N>1)")
    ap.add_argument("--order", choices=["stream", "shuffled"], default="stream")
    ap.add_argument("--strategy", choices=["auto", "stream", "shuffled"], default="auto")
    ap.add_argument("--records-per-gpu", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-comparator", action="store_true")
    ap.add_argument("--no-parse", action="store_true", help="skip the NEXT-3 text-parse leg")
    ap.add_argument("--cpu-target-s", type=float, default=12.0)
    ap.add_argument("--profile", action="store_true",
                    help="for ncu: no soak, no parity gate, no e2e, no CPU leg (numbers not valid)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_for(args, world):
    from synth import WORKLOADS
    name = args.config or "c2"
    wl = WORKLOADS[name].with_(order=args.order)
    if args.records_per_gpu:
        wl = wl.with_(n=args.records_per_gpu * world)
    elif args.config is None and world > 1:
        wl = wl.with_(n=WORKLOADS["c2"].n * world)     # weak scaling: 100M per GPU
    return wl


def describe(wl, world, strategy):
    return {
        "workload": (f"{wl.name}: {wl.n:,} synthetic sessions, window {wl.window_ms:,} ms in "
                     f"{wl.nbins:,} bins of {wl.bin_width_ms} ms, {wl.n_prefixes} prefixes ({wl.table}), "
                     f"{wl.ts_mode} ts, {wl.order} order"
                     + (f", {world} contiguous shards (weak scaling, {wl.n // world:,}/GPU)" if world > 1 else "")),
        "records": wl.n, "records_per_gpu": wl.n // world, "bins": wl.nbins, "prefixes": wl.n_prefixes,
        "order": wl.order, "strategy": strategy, "parallelism": f"dp{world}",
        "exchange": ("none (1 GPU)" if world == 1 else
                     "NCCL: all-gather touched ranges + send/recv of overlaps (sparse) or reduce-scatter (dense)"),
        "l2": "no flush: inputs (24 B/record) and bins (32 B/bin) are each larger than the 126 MB L2",
    }


# ------------------------------------------------------------------ clocks sampler
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 8 and r[0].isdigit()]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        load = [r for r in rows if r[7].isdigit() and int(r[7]) > 0] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in load for i in range(4) if r[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(int(r[0]) for r in load), "sm_max_mhz": max(int(r[1]) for r in rows),
                "reasons": reasons, "samples": len(load)}


# ------------------------------------------------------------------ CPU oracle timing
def cpu_oracle_rate(cols_fn, nets, lens, wl, target_s, threads):
    """Oracle as it stands (multi-threaded time-slab variant), on a bounded prefix sample."""
    from oracle import core as oracle
    start, window, width = wl.window_start_ms, wl.window_ms, wl.bin_width_ms
    n_cal = min(wl.n, 2_000_000)
    cols = cols_fn(0, n_cal)
    res = oracle.OracleResult(wl.nbins)
    t0 = time.perf_counter()
    oracle.classify_histogram(*cols, nets, lens, start, window, width, threads=threads, into=res)
    cal = time.perf_counter() - t0
    n, el = n_cal, cal
    # the calibration run carries fixed costs (the day of bins), so it over-estimates the
    # per-record time: re-size from the last run until the sample takes >= 3/4 of the target
    for _ in range(3):
        if el >= 0.75 * target_s or n >= wl.n:
            break
        n_next = int(min(wl.n, max(n + 1, n * target_s / max(el, 1e-3))))
        cols = cols_fn(0, n_next)
        res = oracle.OracleResult(wl.nbins)
        t0 = time.perf_counter()
        oracle.classify_histogram(*cols, nets, lens, start, window, width, threads=threads, into=res)
        n, el = n_next, time.perf_counter() - t0
    return n / el, n, el


# ------------------------------------------------------------------ reference arm (the oracle)
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import torch
    from synth import prefix_table, records
    from synth.sinet_synth import to_numpy
    wl = workload_for(args, world)
    nets, lens = prefix_table(wl)
    threads = len(os.sched_getaffinity(0))
    order = None
    dev = "cuda" if torch.cuda.is_available() else "cpu"

    def cols_fn(lo, hi):
        nonlocal order
        from synth.sinet_synth import stream_order
        if order is None:
            order = stream_order(wl, dev)
        r = records(wl, lo, hi, device=dev, order=order)
        return to_numpy({k: v.cpu() for k, v in r.items()})

    from oracle import core as oracle
    # each step: the oracle on a bounded sample of the workload (the first S records)
    rate, n_s, el = cpu_oracle_rate(cols_fn, nets, lens, wl, min(args.cpu_target_s, 20.0 / max(1, args.steps)), threads)
    cols = cols_fn(0, n_s)
    times = []
    for i in range(args.warmup + args.steps):
        res = oracle.OracleResult(wl.nbins)
        t0 = time.perf_counter()
        oracle.classify_histogram(*cols, nets, lens, wl.window_start_ms, wl.window_ms, wl.bin_width_ms,
                                  threads=threads, into=res)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    ms = 1e3 * sum(times) / len(times)
    value = n_s / (ms / 1e3)
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
           "config": describe(wl, world, "oracle"),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                            "sample": f"first {n_s:,} of {wl.n:,} records of the same workload per step "
                                      f"(oracle/sinet_oracle.c multi-threaded time-slab variant)"},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "gpu_launches": 0}
    print(json.dumps(out))
    return 0


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    rank, world, local = dist_env()
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    import paper_2106_12863_b200 as S
    from synth import prefix_table, records
    from synth.sinet_synth import stream_order, to_numpy

    wl = workload_for(args, world)
    nets, lens = prefix_table(wl)
    strategy = {"auto": S.ORDER_AUTO, "stream": S.ORDER_STREAM, "shuffled": S.ORDER_SHUFFLED}[args.strategy]
    lo, hi = S.shard_range(wl.n, rank, world)
    R = hi - lo

    # ---- inputs: generated on the device, resident in HBM before timing
    order = stream_order(wl, dev)
    rec = records(wl, lo, hi, device=dev, order=order)
    del order
    torch.cuda.empty_cache()
    ts, src, dst, nb = rec["ts"], rec["src"], rec["dst"], rec["bytes"]
    del rec["cls"]

    stream = torch.cuda.current_stream(dev)
    h = S.SinetHistogram(nets, lens, wl.window_start_ms, wl.window_ms, wl.bin_width_ms, device=local,
                         rank=rank, world=world, stream=stream, order=strategy)
    if world > 1:
        h.comm_init_from_group()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier(device_ids=[local])

    def step():
        h.reset()
        h.classify(ts, src, dst, nb)
        h.reduce()

    clocks = Clocks(local)
    clocks.start()
    # warm-up: W steps, then at least ~1 s of steps so clocks reach steady state
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    t_soak = time.perf_counter()
    while not args.profile and time.perf_counter() - t_soak < 1.0:
        step()
        torch.cuda.synchronize()

    # ---- timed region: exactly K steps
    h.set_kernel_timing(True)
    l0 = h.launches
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = h.launches - l0
    ms = e0.elapsed_time(e1) / args.steps
    kern_ms_total, kern_n = h.kernel_time()
    h.set_kernel_timing(False)
    clk = clocks.stop()
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms, kern_ms_total / max(kern_n, 1)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kern_avg = float(t[0]), float(t[1])
    else:
        kern_avg = kern_ms_total / max(kern_n, 1)
    strat_used = {1: "stream", 2: "shuffled"}.get(h.last_strategy, str(h.last_strategy))
    exch_used = {0: None, 1: "dense", 2: "sparse"}.get(h.last_exchange)

    # ---- correctness gate (properties at full size + sampled bins vs the oracle)
    gate = None if args.profile else check_result(S, h, wl, ts, src, dst, nb, nets, lens, rank, world, dev)

    # ---- NEXT-4 comparator: the paper's sort + reduce_by_key design on the same input
    comp = None
    if not args.no_comparator and not args.profile and world == 1:
        comp = run_comparator(h, ts, src, dst, nb, args, wl)

    # ---- NEXT-3: session-log text -> columns (the step before the path), rank 0 at N == 1
    parse = None
    if not args.no_parse and not args.profile and world == 1:
        parse = run_parse_leg(S, wl, args, dev)

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e and not args.profile:
        e2e = run_e2e(h, ts, src, dst, nb, args, world, local, barrier)

    # ---- CPU oracle baseline (rank 0, N == 1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and not args.profile:
        threads = len(os.sched_getaffinity(0))
        del h
        torch.cuda.empty_cache()
        host = {"ts": ts.cpu(), "src": src.cpu(), "dst": dst.cpu(), "bytes": nb.cpu()}

        def cols_fn(a, b):
            return to_numpy({k: v[a:b] for k, v in host.items()})
        rate, n_s, el = cpu_oracle_rate(cols_fn, nets, lens, wl, args.cpu_target_s, threads)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": f"first {n_s:,} of the {wl.n:,} records (oracle/sinet_oracle.c, time-slab threads), "
                         f"{el:.1f} s"}

    if rank == 0:
        peaks = load_peaks()
        bw = peaks.get("hbm_gbs", 6554.2)
        B = wl.nbins
        alg_step = 24.0 * R + 32.0 * B                     # per GPU
        achieved = alg_step / (kern_avg * 1e-3) / 1e9
        step_gbs = alg_step / (ms * 1e-3) / 1e9
        value = wl.n / (ms * 1e-3)
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": dict(describe(wl, world, strat_used), exchange_used=exch_used),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": bw, "unit": "GB/s",
                         "frac": achieved / bw, "traffic": ncu_traffic(wl.name, strat_used),
                         "kernel": "k_hist_stream" if strat_used == "stream" else "k_hist_atomic",
                         "kernel_ms": kern_avg, "alg_bytes_per_launch": alg_step,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)" if peaks else "fallback 6554.2"},
            "step_roofline": {"achieved": step_gbs, "frac": step_gbs / bw,
                              "note": "(24 B/record + 32 B/bin) per GPU / whole-step time"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "comparator": comp,
            "next3_parse": parse,
            "gpu_launches": launches,
            "clocks": clk,
            "parity_gate": gate,
        }
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def ncu_traffic(workload, strategy):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        return d.get(f"{workload}/{strategy}", {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def check_result(S, h, wl, ts, src, dst, nb, nets, lens, rank, world, dev):
    """Full-size properties on the device + bit-exact sampled bins vs the oracle (N == 1)."""
    import torch
    h.reset()
    h.classify(ts, src, dst, nb)
    h.reduce()
    tot = h.read_totals().astype(object)
    lo, hi = h.owned_range()
    bv = h.bins_view()[lo:hi]
    # sums of the owned bins (int64 wraps mod 2^64 like the u64 bins)
    sums = [[int(bv[:, d, m].sum().item()) & ((1 << 64) - 1) for m in (0, 1)] for d in (0, 1)]
    n_local = torch.tensor([ts.numel()], dtype=torch.int64, device=dev)
    bsum = torch.tensor([int(nb.sum().item())], dtype=torch.int64, device=dev)
    s_t = torch.tensor([x if x < (1 << 63) else x - (1 << 64) for m in sums for x in m], dtype=torch.int64, device=dev)
    if world > 1:
        import torch.distributed as dist
        for t in (n_local, bsum, s_t):
            dist.all_reduce(t)
    M = (1 << 64) - 1
    s_all = [int(x) & M for x in s_t.tolist()]
    ok = int(sum(tot[0:4])) == wl.n and int(sum(tot[4:8])) & M == int(bsum.item()) & M
    lut = S.LUT_SRC_PRIORITY
    for d in (0, 1):
        cells = [k for k in range(4) if lut[k] == d]
        ok &= (s_all[2 * d] + int(tot[8 + d])) & M == sum(int(tot[k]) for k in cells) & M
        ok &= (s_all[2 * d + 1] + int(tot[10 + d])) & M == sum(int(tot[4 + k]) for k in cells) & M
    sampled = None
    if world == 1:
        from oracle import core as oracle
        g = torch.Generator(device="cpu").manual_seed(12863)
        pick = torch.randint(0, wl.nbins, (256,), generator=g).to(dev)
        sel = torch.isin((ts - wl.window_start_ms) // wl.bin_width_ms, pick)
        cols = tuple(x.cpu().numpy() for x in (ts[sel].view(torch.int64), src[sel], dst[sel], nb[sel]))
        cols = (cols[0].view(np.uint64), cols[1].view(np.uint32), cols[2].view(np.uint32), cols[3].view(np.uint64))
        o = oracle.classify_histogram(*cols, nets, lens, wl.window_start_ms, wl.window_ms, wl.bin_width_ms)
        p = pick.cpu().numpy()
        got = h.bins_view()[pick].cpu().numpy().view(np.uint64)   # [k, dir, metric]
        sampled = bool(np.array_equal(got[:, :, 0].T, o.count[:, p]) and np.array_equal(got[:, :, 1].T, o.bytes[:, p]))
        ok &= sampled
    if not ok:
        raise SystemExit("PARITY GATE FAILED: refusing to report a timing")
    return {"properties": True, "sampled_bins_vs_oracle": sampled}


def run_comparator(h, ts, src, dst, nb, args, wl):
    """The paper's histogram design (Thrust-style sort by key + reduce_by_key)
    re-done with CUB on this GPU, same records, same C ABI semantics; bins must be identical."""
    import torch
    h.reset()
    h.classify(ts, src, dst, nb)
    h.reduce()
    ref = h.bins_view()[: wl.nbins].clone()
    ref_tot = h.read_totals()
    scratch = None
    k = max(1, min(args.steps, 5))
    for i in range(2 + k):
        if i == 2:
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
        h.reset()
        scratch = h.classify_sortreduce(ts, src, dst, nb, scratch=scratch)
        h.reduce()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / k
    same = bool(torch.equal(h.bins_view()[: wl.nbins], ref)) and np.array_equal(h.read_totals(), ref_tot)
    del scratch, ref
    torch.cuda.empty_cache()
    return {"impl": "paper design on B200: classify -> cub radix sort by (bin,dir) -> reduce_by_key + "
                    "run-length encode -> scatter (P:L213-214)", "ms_per_step": ms,
            "value": wl.n / (ms * 1e-3), "unit": UNIT, "bins_identical": same}


def run_parse_leg(S, wl, args, dev, n_lines=5_000_000):
    """NEXT-3 on this GPU: PA-7080 text (Table 1 lines, ~280 B each, synth/sinet_text.py) parsed
    into the four columns by k_parse_text; checked against the generator's records, timed with
    CUDA events.  Roofline bytes = text read once + 24 B per valid record written."""
    import torch
    from synth import records
    from synth.sinet_text import session_text_batched
    w = wl.with_(n=n_lines)
    rec = records(w, 0, n_lines, device=dev)
    text, _ = session_text_batched(w, rec)
    del rec["cls"]
    out = {"ts": torch.empty(n_lines, dtype=torch.int64, device=dev),
           "src": torch.empty(n_lines, dtype=torch.int32, device=dev),
           "dst": torch.empty(n_lines, dtype=torch.int32, device=dev),
           "bytes": torch.empty(n_lines, dtype=torch.int64, device=dev)}
    wsb = torch.empty(S._native.lib.sinet_parse_workspace_bytes(text.numel()), dtype=torch.uint8, device=dev)
    k = max(3, min(args.steps, 10))
    for _ in range(3):
        cols, _, info = S.parse_text(text, 540, out=out, workspace=wsb)
    ok = (info["valid"] == n_lines and all(torch.equal(cols[c], rec[c]) for c in ("ts", "src", "dst", "bytes")))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        S.parse_text(text, 540, out=out, workspace=wsb)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / k
    nbytes = text.numel()
    alg = nbytes + 24 * n_lines
    bw = load_peaks().get("hbm_gbs", 6554.2)
    res = {"lines": n_lines, "text_bytes": nbytes, "ms": ms, "records_per_s": n_lines / (ms * 1e-3),
           "text_gbs": nbytes / (ms * 1e-3) / 1e9, "roofline_frac": alg / (ms * 1e-3) / 1e9 / bw,
           "columns_equal_generator": bool(ok),
           "note": "sinet_parse_text (k_parse_text), 5 M generated Table-1 lines, includes the result read-back sync"}
    del text, out, wsb, rec
    torch.cuda.empty_cache()
    return res


def run_e2e(h, ts, src, dst, nb, args, world, local, barrier):
    import torch
    pin = [x.cpu().pin_memory() for x in (ts, src, dst, nb)]
    R = ts.numel()
    k = max(1, min(args.steps, 3))

    def step():
        h.reset()
        h.classify_host(*pin, chunk_records=1 << 24)
        h.reduce()
        return h.read_totals()

    step()
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        step()
    torch.cuda.synchronize()
    el = (time.perf_counter() - t0) / k
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([el], dtype=torch.float64, device=torch.device("cuda", local))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t[0])
    total = R * world
    return {"value": total / el, "unit": UNIT, "h2d_bytes_per_step": 24 * R, "d2h_bytes_per_step": 96,
            "ms_per_step": el * 1e3, "steps": k,
            "path": "sinet_classify_histogram_host (pinned host columns -> 2x16M-record staging, copies overlapped "
                    "with the kernel) + sinet_reduce + sinet_read_totals"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
