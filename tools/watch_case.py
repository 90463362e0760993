"""Watchlist repro for compute-sanitizer."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2106_12863_b200 as S
from synth import WORKLOADS, prefix_table, records
from synth.sinet_synth import to_numpy

wl = WORKLOADS["c1"].with_(n=400_000)
nets, lens = prefix_table(wl)
rec = records(wl, device="cuda")
cols = to_numpy({k: v.cpu() for k, v in rec.items()})
rng = np.random.default_rng(300)
listed = np.concatenate([rng.choice(cols[1], 150), rng.choice(cols[2], 150),
                         rng.integers(0, 1 << 32, 577, dtype=np.uint64).astype(np.uint32)])
for strat in (1, 2):
    h = S.SinetHistogram(nets, lens, wl.window_start_ms, wl.window_ms, order=strat)
    h.set_watchlist(listed)
    h.classify(rec["ts"], rec["src"], rec["dst"], rec["bytes"])
    print(strat, h.read_totals()[:4])
    h.classify_sortreduce(rec["ts"], rec["src"], rec["dst"], rec["bytes"])
    print(strat, "sr", h.read_totals()[:4])
