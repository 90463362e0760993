#!/usr/bin/env python
"""Top source lines of an ncu --page source export (--print-source=cuda,sass) by stall samples."""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows = list(csv.reader(open(path)))
cur_file = None
hdr = None
out = []
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or not r or r[0] in ("", "Function Name"):
        continue
    d = dict(zip(hdr, r))
    try:
        samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        inst = int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    stalls = {k: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit()}
    st = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
    out.append((samp, inst, cur_file, r[0], r[1][:90], st))
tot_s = sum(o[0] for o in out) or 1
tot_i = sum(o[1] for o in out) or 1
print(f"total samples {tot_s}, total warp instructions {tot_i}")
for samp, inst, f, ln, src, st in sorted(out, key=lambda o: -o[0])[:top]:
    print(f"{100*samp/tot_s:5.1f}% s {100*inst/tot_i:5.1f}% i {f}:{ln:>4} {src:90s} {st}")
