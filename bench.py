#!/usr/bin/env python
"""Benchmark of the SINET discrimination + ms-histogram hot path (BASELINE.json metric).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config c2] [--legs ...]
  torchrun --nproc-per-node N bench.py --gpus N ...          (one rank per GPU, NCCL)

A "step" = one pass of the whole hot path over one batch: reset the histogram,
discriminate + bin every record resident in HBM (one fused kernel), materialise
untouched bins, and (N > 1) merge the per-GPU partials (sparse touched-range
exchange or dense reduce-scatter) + the totals all-reduce.

Workloads (BASELINE.json configs, synth/):
  * N == 1: the headline line is configs[1] = C2 (100 M sessions, one day of 1 ms bins,
    64 prefixes); the legs add C4 (1.6 B bursty, the north-star day, on one GPU = the
    scaling baseline), C3 (1.2 B), C5 (400 M, 4096-entry /8-/32 list), C1 (1 M, 1 h) and
    the shuffled order of C2 and C4, each at full size.
  * N > 1: C3 (1.2 B sessions, strong scaling: contiguous shards of one day); at N == 8
    the C4 leg (1.6 B bursty) as well.
Every measured config is gated on bit-exact parity before its timing is reported: the
SHA-256 of each full (dir, metric) plane and the 12 totals must equal the oracle's
(tests/golden/digests.json, written by tools/oracle_digests.py from oracle/ only).
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sessions/sec classified+histogrammed at 1/2/4/8 B200; % of HBM roofline"
UNIT = "sessions/s"
L2_BYTES = 126 * 1024 * 1024
DIGESTS = os.path.join(ROOT, "tests", "golden", "digests.json")
PLANES = ("out_count", "out_bytes", "in_count", "in_bytes")   # (dir, metric) = (0,0) (0,1) (1,0) (1,1)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default=None, help="c1..c5 (default: c2 at N=1, c3 at N>1)")
    ap.add_argument("--order", choices=["stream", "shuffled"], default="stream")
    ap.add_argument("--strategy", choices=["auto", "stream", "shuffled"], default="auto")
    ap.add_argument("--records-per-gpu", type=int, default=None)
    ap.add_argument("--legs", default=None,
                    help="comma list of extra configs, name[@shuffled] (default: N=1 c4,c3,c5,c1,c2@shuffled,"
                         "c4@shuffled; N=8 c4; else none); 'none' for none")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-comparator", action="store_true")
    ap.add_argument("--no-parse", action="store_true", help="skip the NEXT-3 text-parse leg")
    ap.add_argument("--no-gate", action="store_true", help="skip the digest parity gate (numbers not valid)")
    ap.add_argument("--cpu-target-s", type=float, default=12.0)
    ap.add_argument("--knob", action="append", default=[],
                    help="name=value library performance knob (sinet_set_knob) for A/B runs; repeatable")
    ap.add_argument("--profile", action="store_true",
                    help="for ncu: no soak, no legs, no parity gate, no e2e, no CPU leg (numbers not valid)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def main_workload(args, world):
    from synth import WORKLOADS
    name = args.config or ("c2" if world == 1 else "c3")
    wl = WORKLOADS[name].with_(order=args.order)
    if args.records_per_gpu:
        wl = wl.with_(n=args.records_per_gpu * world)
    return wl


def leg_workloads(args, world):
    from synth import WORKLOADS
    spec = args.legs
    if spec is None:
        spec = ("c4,c3,c5,c1,c2@shuffled,c4@shuffled" if world == 1 else "c4" if world == 8 else "none")
    if args.profile or spec in ("", "none"):
        return []
    out = []
    for item in spec.split(","):
        name, _, order = item.strip().partition("@")
        out.append(WORKLOADS[name].with_(order=order or "stream"))
    return out


def fits_l2(wl, world):
    return 24 * (wl.n // world) + 32 * wl.nbins < 2 * L2_BYTES


def describe(wl, world, strategy):
    R = wl.n // world
    return {
        "workload": (f"{wl.name}: {wl.n:,} synthetic sessions, window {wl.window_ms:,} ms in "
                     f"{wl.nbins:,} bins of {wl.bin_width_ms} ms, {wl.n_prefixes} prefixes ({wl.table}), "
                     f"{wl.ts_mode} ts, {wl.order} order"
                     + (f", {world} contiguous shards ({R:,}/GPU, strong scaling: the same day over "
                        f"{world} GPUs)" if world > 1 else "")),
        "records": wl.n, "records_per_gpu": R, "bins": wl.nbins, "prefixes": wl.n_prefixes,
        "order": wl.order, "strategy": strategy, "parallelism": f"dp{world}",
        "exchange": ("none (1 GPU)" if world == 1 else
                     "NCCL: all-gather touched ranges + send/recv of overlaps (sparse) or reduce-scatter (dense)"),
        "l2": (f"flushed between steps (a 256 MB write outside the per-step events): inputs "
               f"{24 * R / 1e6:.0f} MB + bins {32 * wl.nbins / 1e6:.0f} MB fit in the 126 MB L2 twice over"
               if fits_l2(wl, world) else
               f"no flush: inputs ({24 * R / 1e9:.2f} GB) + bins ({32 * wl.nbins / 1e9:.2f} GB) exceed the "
               f"126 MB L2 many times"),
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
        return self

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


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


# ------------------------------------------------------------------ CPU oracle timing
def oracle_rate(cols_fn, nets, lens, wl, target_s, threads, res=None):
    """Oracle as it stands (oracle/sinet_oracle.c; the time-slab multi-threaded variant for
    threads > 1) on a bounded prefix sample of the workload, into a result whose pages are
    touched before timing.  Returns (records/s, records, seconds)."""
    from oracle import core as oracle
    start, window, width = wl.window_start_ms, wl.window_ms, wl.bin_width_ms
    if res is None:
        res = oracle.OracleResult(wl.nbins)
    n, el = min(wl.n, 200_000 if threads == 1 else 2_000_000), 0.0
    for _ in range(4):
        cols = cols_fn(0, n)
        for a in (res.count, res.bytes, res.totals):
            a.fill(0)                                       # page-in + reset, outside the timing
        t0 = time.perf_counter()
        oracle.classify_histogram(*cols, nets, lens, start, window, width, threads=threads, into=res)
        el = time.perf_counter() - t0
        if el >= 0.75 * target_s or n >= wl.n:
            break
        n = int(min(wl.n, max(n + 1, n * target_s / max(el, 1e-3))))
    return n / el, n, el


def host_cols_fn(wl, dev):
    """Records [lo, hi) of the workload's stream/shuffled order as host numpy columns."""
    from synth import records
    from synth.sinet_synth import stream_order, to_numpy
    order = None

    def cols_fn(lo, hi):
        nonlocal order
        if order is None:
            order = stream_order(wl, dev)
        r = records(wl, lo, hi, device=dev, order=order)
        return to_numpy({k: v.cpu() for k, v in r.items() if k != "cls"})
    return cols_fn


# ------------------------------------------------------------------ reference arm (the oracle)
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import torch
    from synth import prefix_table
    from oracle import core as oracle
    wl = main_workload(args, world)
    nets, lens = prefix_table(wl)
    threads = len(os.sched_getaffinity(0))
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    cols_fn = host_cols_fn(wl, dev)
    res = oracle.OracleResult(wl.nbins)
    # each step: the oracle on the first S records of the workload, S sized so that the whole
    # --warmup W --steps K run takes about a minute (a bounded sample, the same per-record
    # arithmetic as the full config; the result buffer is pre-touched and reset outside timing)
    per_step = max(0.2, min(args.cpu_target_s, 60.0 / max(1, args.steps + args.warmup)))
    _, n_s, _ = oracle_rate(cols_fn, nets, lens, wl, per_step, threads, res)
    cols = cols_fn(0, n_s)
    times = []
    for i in range(args.warmup + args.steps):
        for a in (res.count, res.bytes, res.totals):
            a.fill(0)
        t0 = time.perf_counter()
        oracle.classify_histogram(*cols, nets, lens, wl.window_start_ms, wl.window_ms, wl.bin_width_ms,
                                  threads=threads, into=res)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    ms = 1e3 * sum(times) / len(times)
    value = n_s / (ms / 1e3)
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
           "ms_median": 1e3 * statistics.median(times), "higher_is_better": True,
           "scaling": "weak" if world == 1 else "strong", "vs_baseline": None, "dtype": "u64",
           "data": "synthetic", "config": describe(wl, world, "oracle"),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "cpu": cpu_model(),
                            "sample": f"first {n_s:,} of {wl.n:,} records of the same workload per step "
                                      f"(oracle/sinet_oracle.c, time-slab threads, pre-touched result)"},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "gpu_launches": 0}
    print(json.dumps(out))
    return 0


# ------------------------------------------------------------------ parity gate
def load_digests():
    try:
        with open(DIGESTS) as f:
            return json.load(f)
    except Exception:
        return {}


def expected_digest(wl):
    d = load_digests().get(wl.name)
    if not d:
        return None
    same = (d["n"] == wl.n and d["nbins"] == wl.nbins and d["window_start_ms"] == wl.window_start_ms
            and d["bin_width_ms"] == wl.bin_width_ms and d["seed"] == wl.seed and d["ts_mode"] == wl.ts_mode)
    return d if same else None


def gather_planes(h, wl, world, rank, dev):
    """Rank 0: int64[B, 2, 2] host copy of the merged bins (gathered from the owners at N > 1)."""
    import torch
    lo, hi = h.owned_range()
    if world == 1:
        return h.bins_view()[:wl.nbins].cpu()
    import torch.distributed as dist
    per = h.B_pad // world
    mine = torch.zeros((per, 2, 2), dtype=torch.int64, device=dev)
    mine[: hi - lo].copy_(h.bins_view()[lo:hi])
    full = torch.empty((world * per, 2, 2), dtype=torch.int64, device=dev) if rank == 0 else None
    dist.gather(mine, [full[r * per:(r + 1) * per] for r in range(world)] if rank == 0 else None, dst=0)
    return full[:wl.nbins].cpu() if rank == 0 else None


def digests_of(bins_cpu, totals):
    a = bins_cpu.numpy()

    def one(k):
        d, m = divmod(k, 2)
        return hashlib.sha256(np.ascontiguousarray(a[:, d, m]).view(np.uint64).astype("<u8").tobytes()).hexdigest()
    with ThreadPoolExecutor(4) as ex:
        shas = list(ex.map(one, range(4)))
    return {"sha256": dict(zip(PLANES, shas)), "totals": [int(x) for x in totals]}


def gate(S, h, wl, ts, src, dst, nb, nets, lens, rank, world, dev):
    """Full-size parity: every plane's SHA-256 + the totals vs the oracle's digest (when the
    workload is a committed BASELINE config), else the full-size conservation properties plus
    256 bins re-computed by the oracle from the records that fall in them."""
    import torch
    h.reset()
    h.classify(ts, src, dst, nb)
    h.reduce()
    tot = h.read_totals()
    exp = expected_digest(wl)
    if exp is not None:
        bins = gather_planes(h, wl, world, rank, dev)
        ok = True
        if rank == 0:
            got = digests_of(bins, tot)
            ok = got["sha256"] == exp["sha256"] and got["totals"] == exp["totals"]
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([1 if ok else 0], device=dev)
            dist.broadcast(t, 0)
            ok = bool(t.item())
        if not ok:
            raise SystemExit(f"PARITY GATE FAILED ({wl.name}, {wl.order}): plane digests differ from the oracle's")
        return {"full_digest_vs_oracle": True, "planes": 4, "bins": wl.nbins}
    # fallback (non-standard sizes): properties + sampled bins vs the oracle
    from oracle import core as oracle
    M = (1 << 64) - 1
    lo, hi = h.owned_range()
    bv = h.bins_view()[lo:hi]
    sums = [[int(bv[:, d, m].sum().item()) & M for m in (0, 1)] for d in (0, 1)]
    s_t = torch.tensor([x if x < (1 << 63) else x - (1 << 64) for m in sums for x in m], dtype=torch.int64, device=dev)
    n_local = torch.tensor([ts.numel()], dtype=torch.int64, device=dev)
    bsum = torch.tensor([int(nb.sum().item())], dtype=torch.int64, device=dev)
    if world > 1:
        import torch.distributed as dist
        for t in (n_local, bsum, s_t):
            dist.all_reduce(t)
    s_all = [int(x) & M for x in s_t.tolist()]
    tot = tot.astype(object)
    ok = int(sum(tot[0:4])) == wl.n and int(sum(tot[4:8])) & M == int(bsum.item()) & M
    lut = S.LUT_SRC_PRIORITY
    for d in (0, 1):
        cells = [k for k in range(4) if lut[k] == d]
        ok &= (s_all[2 * d] + int(tot[8 + d])) & M == sum(int(tot[k]) for k in cells) & M
        ok &= (s_all[2 * d + 1] + int(tot[10 + d])) & M == sum(int(tot[4 + k]) for k in cells) & M
    sampled = None
    if world == 1:
        g = torch.Generator(device="cpu").manual_seed(12863)
        pick = torch.randint(0, wl.nbins, (256,), generator=g).to(dev)
        sel = torch.isin((ts - wl.window_start_ms) // wl.bin_width_ms, pick)
        cols = tuple(x.cpu().numpy() for x in (ts[sel], src[sel], dst[sel], nb[sel]))
        cols = (cols[0].view(np.uint64), cols[1].view(np.uint32), cols[2].view(np.uint32), cols[3].view(np.uint64))
        o = oracle.classify_histogram(*cols, nets, lens, wl.window_start_ms, wl.window_ms, wl.bin_width_ms)
        p = pick.cpu().numpy()
        got = h.bins_view()[pick].cpu().numpy().view(np.uint64)
        sampled = bool(np.array_equal(got[:, :, 0].T, o.count[:, p]) and np.array_equal(got[:, :, 1].T, o.bytes[:, p]))
        ok &= sampled
    if not ok:
        raise SystemExit(f"PARITY GATE FAILED ({wl.name}): properties / sampled bins differ from the oracle")
    return {"full_digest_vs_oracle": False, "properties": True, "sampled_bins_vs_oracle": sampled}


# ------------------------------------------------------------------ one measured config
class Ctx:
    def __init__(self, args, rank, world, local, dev):
        self.args, self.rank, self.world, self.local, self.dev = args, rank, world, local, dev

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier(device_ids=[self.local])


def make_inputs(wl, cx):
    import torch
    import paper_2106_12863_b200 as S
    from synth.sinet_synth import records_into
    lo, hi = S.shard_range(wl.n, cx.rank, cx.world)
    rec = records_into(wl, lo, hi, cx.dev)
    torch.cuda.empty_cache()
    return rec


def open_hist(wl, cx, stream):
    import paper_2106_12863_b200 as S
    from synth import prefix_table
    nets, lens = prefix_table(wl)
    strategy = {"auto": S.ORDER_AUTO, "stream": S.ORDER_STREAM, "shuffled": S.ORDER_SHUFFLED}[cx.args.strategy]
    h = S.SinetHistogram(nets, lens, wl.window_start_ms, wl.window_ms, wl.bin_width_ms, device=cx.local,
                         rank=cx.rank, world=cx.world, stream=stream, order=strategy)
    if cx.world > 1:
        h.comm_init_from_group()
    for kv in cx.args.knob:
        name, _, val = kv.partition("=")
        h.set_knob(name, int(val))
    if wl.order == "shuffled":
        # partition-then-bin scratch for the whole shard (one sub-batch: every bin written once)
        h.set_scratch(S.shard_range(wl.n, cx.rank, cx.world)[1] - S.shard_range(wl.n, cx.rank, cx.world)[0])
    return h, nets, lens


def measure(wl, cx, rec, steps, warmup):
    """Time `steps` steps of config `wl` (after warm-up + a 1 s soak), gate on parity.
    Returns (summary dict, histogram) -- summary on every rank (timings max-reduced)."""
    import torch
    import paper_2106_12863_b200 as S
    args = cx.args
    stream = torch.cuda.current_stream(cx.dev)
    h, nets, lens = open_hist(wl, cx, stream)
    ts, src, dst, nb = rec["ts"], rec["src"], rec["dst"], rec["bytes"]
    R = ts.numel()
    flush = fits_l2(wl, cx.world)
    scrub = torch.empty(256 << 20, dtype=torch.uint8, device=cx.dev) if flush else None

    def step():
        h.reset()
        h.classify(ts, src, dst, nb)
        h.reduce()

    clocks = Clocks(cx.local).start()
    for _ in range(max(3, warmup)):
        step()
    torch.cuda.synchronize()
    t_soak = time.perf_counter()
    while not args.profile and time.perf_counter() - t_soak < 1.0:
        step()
        torch.cuda.synchronize()

    # ---- timed region: exactly `steps` steps, per-step events (median) inside the bracket
    h.set_kernel_timing(True)
    l0 = h.launches
    cx.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(steps):
        if flush:
            scrub.fill_(k & 0xFF)        # evict the previous step's inputs and bins from the L2
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    cx.barrier()
    launches = h.launches - l0
    per = [a.elapsed_time(b) for a, b in ev]
    ms_total = e0.elapsed_time(e1) / steps
    kern_ms_total, kern_n = h.kernel_time()
    h.set_kernel_timing(False)
    clk = clocks.stop()
    vals = [sum(per) / steps, statistics.median(per), kern_ms_total / max(kern_n, 1), ms_total]
    if cx.world > 1:
        import torch.distributed as dist
        t = torch.tensor(vals, dtype=torch.float64, device=cx.dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        vals = [float(x) for x in t]
    ms_mean, ms_med, kern_avg, ms_bracket = vals
    ms = ms_mean if flush else ms_bracket      # flushes sit between the per-step events
    strat = {1: "stream", 2: "shuffled"}.get(h.last_strategy, str(h.last_strategy))
    exch = {0: None, 1: "dense", 2: "sparse"}.get(h.last_exchange)
    parity = None if (args.profile or args.no_gate) else gate(S, h, wl, ts, src, dst, nb, nets, lens, cx.rank,
                                                                cx.world, cx.dev)
    bw = load_peaks().get("hbm_gbs", 6554.2)
    alg = 24.0 * R + 32.0 * wl.nbins            # per GPU: records read once + bins written once
    kern = h.last_kernel
    summary = {
        "config": dict(describe(wl, cx.world, strat), exchange_used=exch),
        "value": wl.n / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms, "ms_median": ms_med,
        "ms_steps": [round(x, 4) for x in per],
        "roofline": {"bound": "hbm", "achieved": alg / (kern_avg * 1e-3) / 1e9, "peak": bw, "unit": "GB/s",
                     "frac": alg / (kern_avg * 1e-3) / 1e9 / bw, "traffic": ncu_traffic(wl, kern),
                     "kernel": kern, "kernel_ms": kern_avg, "alg_bytes_per_launch": alg,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)" if load_peaks() else "fallback 6554.2"},
        "step_roofline": {"achieved": alg / (ms * 1e-3) / 1e9, "frac": alg / (ms * 1e-3) / 1e9 / bw,
                          "note": "(24 B/record + 32 B/bin) per GPU / whole-step time"},
        "gpu_launches": launches, "clocks": clk, "parity_gate": parity,
    }
    if scrub is not None:
        del scrub
    return summary, h, nets, lens


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
    import paper_2106_12863_b200 as S  # noqa: F401  (fails loudly without libsinet.so)
    cx = Ctx(args, rank, world, local, dev)

    wl = main_workload(args, world)
    rec = make_inputs(wl, cx)
    main, h, nets, lens = measure(wl, cx, rec, args.steps, args.warmup)
    ts, src, dst, nb = rec["ts"], rec["src"], rec["dst"], rec["bytes"]

    comp = None      # NEXT-4 comparator: the paper's sort + reduce_by_key design on the same input
    if not args.no_comparator and not args.profile and world == 1:
        comp = run_comparator(h, ts, src, dst, nb, args, wl)
    parse = None     # NEXT-3: session-log text -> columns (the step before the path)
    if not args.no_parse and not args.profile and world == 1:
        parse = run_parse_leg(wl, args, dev)
    e2e = None       # end to end through the public API with host buffers, result read back
    if not args.no_e2e and not args.profile:
        e2e = run_e2e(h, ts, src, dst, nb, args, cx)
    h.close()
    del h
    torch.cuda.empty_cache()

    cpu = None       # CPU oracle baseline (rank 0, N == 1)
    if rank == 0 and world == 1 and not args.no_cpu and not args.profile:
        threads = len(os.sched_getaffinity(0))
        host = {"ts": ts.cpu(), "src": src.cpu(), "dst": dst.cpu(), "bytes": nb.cpu()}
        from synth.sinet_synth import to_numpy

        def cols_fn(a, b):
            return to_numpy({k: v[a:b] for k, v in host.items()})
        rate, n_s, el = oracle_rate(cols_fn, nets, lens, wl, args.cpu_target_s, threads)
        rate1, n_1, el_1 = oracle_rate(cols_fn, nets, lens, wl, min(5.0, args.cpu_target_s), 1)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "oracle", "cpu": cpu_model(),
               "sample": f"first {n_s:,} of the {wl.n:,} records (oracle/sinet_oracle.c, time-slab threads, "
                         f"pre-touched result), {el:.1f} s",
               "oracle_1t": {"value": rate1, "cores": 1, "sample": f"first {n_1:,} records, {el_1:.1f} s"}}
        del host
    del rec, ts, src, dst, nb
    torch.cuda.empty_cache()

    legs = {}
    for lw in leg_workloads(args, world):
        key = lw.name + ("" if lw.order == "stream" else "@" + lw.order)
        try:
            r = make_inputs(lw, cx)
            s, hl, _, _ = measure(lw, cx, r, args.steps, max(3, min(args.warmup, 3)))
            hl.close()
            del hl
        except (Exception, SystemExit) as e:   # a leg that fails its gate reports no timing
            s = {"error": f"{type(e).__name__}: {e}"[:300]}
        r = None
        torch.cuda.empty_cache()
        legs[key] = s

    if rank == 0:
        out = {
            "metric": METRIC, "value": main["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": main["ms_per_step"], "ms_median": main["ms_median"],
            "higher_is_better": True, "scaling": "weak" if world == 1 else "strong",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": main["config"], "roofline": main["roofline"], "step_roofline": main["step_roofline"],
            "cpu_baseline": cpu, "e2e": e2e, "comparator": comp, "next3_parse": parse,
            "gpu_launches": main["gpu_launches"], "clocks": main["clocks"], "parity_gate": main["parity_gate"],
            "ms_steps": main["ms_steps"], "legs": legs,
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


def ncu_traffic(wl, kernel):
    """DRAM bytes per launch of the dominant kernel from a committed ncu --set full capture
    (profiles/ncu_traffic.json, keyed workload/order/kernel), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        e = d.get(f"{wl.name}/{wl.order}/{kernel}")
        return e.get("dram_bytes_per_launch") if e else None
    except Exception:
        return None


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


def run_parse_leg(wl, args, dev, n_lines=5_000_000):
    """NEXT-3 on this GPU: PA-7080 text (Table 1 lines, ~280 B each, synth/sinet_text.py) parsed
    into the four columns by k_parse_text; checked against the generator's records, timed with
    CUDA events.  Roofline bytes = text read once + 24 B per valid record written."""
    import torch
    import paper_2106_12863_b200 as S
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
           "note": "sinet_parse_text (k_parse_text), 5 M generated Table-1 lines (JST, tz +540 min), "
                   "includes the result read-back sync"}
    del text, out, wsb, rec
    torch.cuda.empty_cache()
    return res


def run_e2e(h, ts, src, dst, nb, args, cx):
    """The same metric through the public API from pinned host columns: per step the
    host->device copy of the records (overlapped with the kernel by sinet_classify_histogram_host),
    the merge, and the device->host read-back of the whole owned histogram (both directions,
    count and bytes: sinet_read_bins_raw) and of the totals.  PCIe-bound by design: the step
    moves 24 B/record in and 32 B/bin out over the host link."""
    import torch
    pin = [x.cpu().pin_memory() for x in (ts, src, dst, nb)]
    R = ts.numel()
    k = max(1, min(args.steps, 3))
    lo, hi = h.owned_range()
    out = torch.empty((hi - lo, 2, 2), dtype=torch.int64).pin_memory()

    def step():
        h.reset()
        h.classify_host(*pin, chunk_records=1 << 24)
        h.reduce()
        h.read_bins_raw(out)
        return h.read_totals()

    step()
    cx.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        step()
    torch.cuda.synchronize()
    el = (time.perf_counter() - t0) / k
    if cx.world > 1:
        import torch.distributed as dist
        t = torch.tensor([el], dtype=torch.float64, device=cx.dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t[0])
    total = R * cx.world
    d2h = 32 * (hi - lo) + 96
    del pin, out
    return {"value": total / el, "unit": UNIT, "h2d_bytes_per_step": 24 * R, "d2h_bytes_per_step": d2h,
            "ms_per_step": el * 1e3, "steps": k,
            "host_link_gbs": (24 * R + d2h) / el / 1e9,
            "path": "sinet_classify_histogram_host (pinned host columns -> 2x16M-record staging, copies overlapped "
                    "with the kernel) + sinet_reduce + sinet_read_bins_raw (whole owned histogram to pinned host) "
                    "+ sinet_read_totals; wall clock, host link (PCIe) bound"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
