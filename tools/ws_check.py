#!/usr/bin/env python
"""Quick A/B of the stream kernels on one GPU: parity vs the oracle on small cases, then
C2-shaped timing of k_hist_stream (knob stream_kernel=1) and k_hist_ws (=2)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2106_12863_b200 as S  # noqa: E402
from oracle import core as oracle  # noqa: E402
from synth import WORKLOADS, prefix_table, records  # noqa: E402
from synth.sinet_synth import records_into, to_numpy  # noqa: E402


def run(wl, rec, kern, steps=0):
    nets, lens = prefix_table(wl)
    h = S.SinetHistogram(nets, lens, wl.window_start_ms, wl.window_ms, wl.bin_width_ms, order=S.ORDER_STREAM)
    h.set_knob("stream_kernel", kern)
    args = (rec["ts"], rec["src"], rec["dst"], rec["bytes"])
    h.classify(*args)
    h.finalize()
    torch.cuda.synchronize()
    ms = None
    if steps:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(3):
            h.reset(); h.classify(*args); h.finalize()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(steps):
            h.reset(); h.classify(*args); h.finalize()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
    return h, ms


for name, n in (("c1", 300_000), ("c2", 3_000_000), ("c4", 3_000_000), ("c5", 2_000_000)):
    wl = WORKLOADS[name].with_(n=n, window_ms=3_600_000 if name != "c1" else 3_600_000)
    rec = records(wl, device="cuda")
    nets, lens = prefix_table(wl)
    o = oracle.classify_histogram(*to_numpy({k: v.cpu() for k, v in rec.items()}), nets, lens,
                                  wl.window_start_ms, wl.window_ms, 1, threads=8)
    for kern in (1, 2):
        t0 = time.time()
        h, _ = run(wl, rec, kern)
        c = np.stack([h.read_bins(d, 0) for d in (0, 1)])
        b = np.stack([h.read_bins(d, 1) for d in (0, 1)])
        ok = np.array_equal(c, o.count) and np.array_equal(b, o.bytes) and np.array_equal(h.read_totals(), o.totals)
        print(f"parity {name} n={n} kernel={kern} ({h.last_kernel}): {'OK' if ok else 'MISMATCH'} {time.time()-t0:.1f}s",
              flush=True)
        h.close()
import ctypes
from paper_2106_12863_b200 import _native as N
N.lib.sinet_debug_counters.argtypes = [ctypes.c_void_p, ctypes.c_int]
dbg = (ctypes.c_ulonglong * 12)()
for name in ("c2",):
    wl = WORKLOADS[name].with_(n=100_000_000)
    rec = records_into(wl, 0, wl.n, "cuda")
    nets, lens = prefix_table(wl)
    h = S.SinetHistogram(nets, lens, wl.window_start_ms, wl.window_ms, order=S.ORDER_STREAM)
    h.set_knob("stream_kernel", 2)
    h.set_knob("debug_counters", 1)
    N.lib.sinet_debug_counters(None, 1)
    h.classify(rec["ts"], rec["src"], rec["dst"], rec["bytes"])
    torch.cuda.synchronize()
    N.lib.sinet_debug_counters(dbg, 1)
    print("debug", name, "late, early, hi, batches, tiles, idle polls, chunks, hot chunks, wait heads, wait handshake, sum(tile-top) early, max head spread =", list(dbg), flush=True)
    h.close()
    del rec
    torch.cuda.empty_cache()
for name in ("c2", "c4", "c5"):
    wl = WORKLOADS[name]
    if name == "c4":
        wl = wl.with_(n=400_000_000)
    rec = records_into(wl, 0, wl.n, "cuda")
    for kern in (1, 2):
        h, ms = run(wl, rec, kern, steps=10)
        alg = 24 * wl.n + 32 * wl.nbins
        print(f"time {name} n={wl.n:,} kernel={kern} ({h.last_kernel}): {ms:.3f} ms/step "
              f"(classify+finalize), {alg / ms / 1e6:.0f} GB/s", flush=True)
        h.close()
    del rec
    torch.cuda.empty_cache()
