"""Small stream/atomic/series cases for compute-sanitizer (memcheck, racecheck, synccheck)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2106_12863_b200 as S
from synth import WORKLOADS, prefix_table, records

wl = WORKLOADS["c1"].with_(n=60_000, window_ms=600_000)
nets, lens = prefix_table(wl)
for order in ("stream", "shuffled"):
    rec = records(wl.with_(order=order), device="cuda")
    for strat, groups in ((1, 1), (1, 2), (2, 0)):
        h = S.SinetHistogram(nets, lens, wl.window_start_ms, wl.window_ms, order=strat)
        h.set_tuning(groups, -1)
        tags = torch.empty(wl.n, dtype=torch.uint8, device="cuda")
        h.classify(rec["ts"][1:], rec["src"][1:], rec["dst"][1:], rec["bytes"][1:], tags=tags[1:])
        h.reduce()
        t = h.read_totals()
        r = h.rebin(1000)
        (ts, c, b), n = h.export_sparse(0)
        h.close()
        print(order, strat, groups, int(t[:4].sum()), int(r.sum()), n)
torch.cuda.synchronize()
print("sanitize case done")
