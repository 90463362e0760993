"""Dense stream case for compute-sanitizer (racecheck / memcheck): C2-like density (1.6 records
per ms, 2 s disorder), both group layouts, checked bit-exact against the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2106_12863_b200 as S
from oracle import core as oracle
from synth import WORKLOADS, prefix_table, records
from synth.sinet_synth import to_numpy

wl = WORKLOADS["c2"].with_(n=400_000, window_ms=250_000)
nets, lens = prefix_table(wl)
rec = records(wl, device="cuda")
cols = to_numpy({k: v.cpu() for k, v in rec.items() if k != "cls"})
o = oracle.classify_histogram(*cols, nets, lens, wl.window_start_ms, wl.window_ms, 1)
for groups in (2, 1):
    h = S.SinetHistogram(nets, lens, wl.window_start_ms, wl.window_ms, order=S.ORDER_STREAM)
    h.set_tuning(groups, -1)
    h.classify(rec["ts"], rec["src"], rec["dst"], rec["bytes"])
    h.reduce()
    ok = (np.array_equal(np.stack([h.read_bins(d, S.METRIC_COUNT) for d in (0, 1)]), o.count) and
          np.array_equal(np.stack([h.read_bins(d, S.METRIC_BYTES) for d in (0, 1)]), o.bytes) and
          np.array_equal(h.read_totals(), o.totals))
    h.close()
    print("dense groups", groups, "bit-exact" if ok else "MISMATCH")
    assert ok
print("sanitize dense case done")
