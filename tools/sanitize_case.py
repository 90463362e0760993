"""Small stream/atomic/partition/series cases for compute-sanitizer (memcheck, racecheck, synccheck).

Kernel variants: (strategy, layout) = STREAM with k_hist_stream (1 or 2 rings), STREAM with
k_hist_ws ("ws"), SHUFFLED with L2 atomics (no scratch) and SHUFFLED partition-then-bin ("part")."""
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
    for strat, groups in ((1, 1), (1, 2), (1, "ws"), (2, 0), (2, "part")):
        h = S.SinetHistogram(nets, lens, wl.window_start_ms, wl.window_ms, order=strat)
        if groups == "ws":
            h.set_knob("stream_kernel", 2)
        elif groups == "part":
            h.set_scratch(1 << 16)
        else:
            h.set_knob("stream_kernel", 1)
            h.set_tuning(groups, -1)
        tags = torch.empty(wl.n, dtype=torch.uint8, device="cuda")
        h.classify(rec["ts"][1:], rec["src"][1:], rec["dst"][1:], rec["bytes"][1:], tags=tags[1:])
        h.reduce()
        t = h.read_totals()
        r = h.rebin(1000)
        (ts, c, b), n = h.export_sparse(0)
        h.close()
        print(order, strat, groups, int(t[:4].sum()), int(r.sum()), n)
# every lookup-table encoding on a /8-/32 list, records with > 2^32 bytes (the ring's high-word spill)
n5, l5 = prefix_table(WORKLOADS["c5"])
for tab_nets, tab_lens in ((n5[:100], l5[:100]), (n5, l5)):
    rec = records(wl.with_(order="stream"), device="cuda")
    big = rec["bytes"].clone()
    big[::97] = big[::97] + (1 << 33)
    for tab in (0, 1, 2, 3):
        for kern in (1, 2):
            h = S.SinetHistogram(tab_nets, tab_lens, wl.window_start_ms, wl.window_ms, order=1)
            h.set_table_mode(tab)
            h.set_knob("stream_kernel", kern)
            h.classify(rec["ts"], rec["src"], rec["dst"], big)
            t = h.read_totals()
            h.close()
            print("table", len(tab_nets), tab, kern, int(t[:4].sum()))
# NEXT-3 parser: several 16 KB chunks, malformed lines, look-back across chunks
from synth.sinet_text import session_text_batched
pw = WORKLOADS["c1"].with_(n=3000)
prec = records(pw, device="cuda")
text, _ = session_text_batched(pw, prec, bad_per_million=20_000)
cols, st, info = S.parse_text(text, 540, status=True)
print("parse", info["lines"], info["valid"])
torch.cuda.synchronize()
print("sanitize case done")
