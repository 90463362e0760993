#!/usr/bin/env python
"""Attribute ncu per-SASS-instruction counters to CUDA source lines (run here, on the CPU box).

ncu's CSV source page of this ncu version carries the counters only at SASS level, so this
joins it with `nvdisasm -g` line info of the same cubin (instructions in the same order):

  ncu -i rep.ncu-rep --page source --csv --print-source=sass > sass.csv
  cuobjdump -xelf all libsinet.so ; nvdisasm -g -c sinet_stream.sm_100a.cubin > all.sass
  python tools/sass_lines.py sass.csv all.sass [top]
"""
import csv
import re
import sys
from collections import defaultdict


def kernel_and_rows(path):
    rows = list(csv.reader(open(path, encoding="utf-8", errors="replace")))
    name = rows[0][1]
    hdr = rows[1]
    body = [dict(zip(hdr, r)) for r in rows[2:] if len(r) >= len(hdr)]
    return name, body


def mangled_match(name, sass_path):
    """The .text section whose mangled template arguments match ncu's demangled kernel name."""
    if re.search(r"::(\w+)<", name) is None:   # not a template: the section naming the function
        base = re.search(r"(\w+)\(", name).group(1)
        secs = re.findall(r"^\.text\.(\S+):$", open(sass_path).read(), re.M)
        for s in secs:
            if base in s:
                return s
        raise SystemExit(f"no section for {name}")
    args = re.search(r"<(.*)>", name).group(1).split(",")
    want = "I" + "E".join(("Lb" if "(bool)" in a else "Li") + a.split(")")[-1].strip() for a in args) + "E"
    base = re.search(r"::(\w+)<", name).group(1)
    secs = re.findall(r"^\.text\.(\S+):$", open(sass_path).read(), re.M)
    for s in secs:
        if base in s and want in s:
            return s
    raise SystemExit(f"no section for {name} ({want})")


def sass_lines(sass_path, section):
    out, cur, on = [], None, False
    for line in open(sass_path):
        if line.startswith(".text."):
            on = line.strip() == f".text.{section}:"
            continue
        if not on:
            continue
        m = re.match(r'\s*//## File "([^"]+)", line (\d+)', line)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        if re.match(r"\s*/\*[0-9a-f]{4,}\*/", line):
            out.append(cur)
    return out


def main():
    csv_path, sass_path = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    name, body = kernel_and_rows(csv_path)
    sec = mangled_match(name, sass_path)
    lines = sass_lines(sass_path, sec)
    if len(lines) != len(body):
        print(f"warning: {len(lines)} disassembled vs {len(body)} profiled instructions")
    src_cache = {}
    agg_s, agg_i = defaultdict(int), defaultdict(int)
    for loc, r in zip(lines, body):
        try:
            agg_s[loc] += int(r["Warp Stall Sampling (All Samples)"] or 0)
            agg_i[loc] += int(r["Instructions Executed"] or 0)
        except ValueError:
            pass
    ts, ti = sum(agg_s.values()) or 1, sum(agg_i.values()) or 1
    print(f"{name}\ntotal samples {ts}, warp instructions {ti}")
    for loc in sorted(agg_s, key=lambda k: -agg_s[k])[:top]:
        f, ln = loc if loc else ("?", 0)
        if f not in src_cache:
            import glob
            cand = glob.glob(f"/root/repo/**/{f}", recursive=True)
            src_cache[f] = open(cand[0]).read().splitlines() if cand else []
        text = src_cache[f][ln - 1].strip()[:80] if 0 < ln <= len(src_cache[f]) else ""
        print(f"{100 * agg_s[loc] / ts:5.1f}% s {100 * agg_i[loc] / ti:5.1f}% i {f}:{ln:<4} {text}")


if __name__ == "__main__":
    main()
