#!/usr/bin/env python
"""A/B of k_hist_stream performance knobs on one GPU (results must stay identical):
per config, time classify+finalize for each knob set and compare every bin and total with the
default run.  Usage: python tools/ab_stream.py [c2 c4 c5]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2106_12863_b200 as S  # noqa: E402
from synth import WORKLOADS, prefix_table  # noqa: E402
from synth.sinet_synth import records_into  # noqa: E402

VARIANTS = [{}]


def timed(h, args, steps=10):
    for _ in range(3):
        h.reset(); h.classify(*args); h.finalize()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        h.reset(); h.classify(*args); h.finalize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


for name in (sys.argv[1:] or ["c2", "c4", "c5"]):
    wl = WORKLOADS[name]
    nets, lens = prefix_table(wl)
    rec = records_into(wl, 0, wl.n, "cuda")
    args = (rec["ts"], rec["src"], rec["dst"], rec["bytes"])
    ref = None
    for knobs in VARIANTS:
        h = S.SinetHistogram(nets, lens, wl.window_start_ms, wl.window_ms, order=S.ORDER_STREAM)
        for k, v in knobs.items():
            h.set_knob(k, v)
        ms = timed(h, args)
        bins = h.bins_view()[: wl.nbins].clone()
        tot = h.read_totals()
        same = None
        if ref is None:
            ref = (bins, tot)
        else:
            same = bool(torch.equal(bins, ref[0])) and (tot == ref[1]).all()
        alg = 24 * wl.n + 32 * wl.nbins
        print(f"{name} {knobs or 'default'}: {ms:.3f} ms, {alg / ms / 1e6:.0f} GB/s, kernel {h.last_kernel}, "
              f"identical to default: {same}", flush=True)
        h.close()
        del bins
    del rec, args, ref
    torch.cuda.empty_cache()
