#!/usr/bin/env python
"""Full-size oracle digests of the BASELINE configs (C1-C5) -> tests/golden/digests.json.

Calls only ``oracle/`` (the CPU oracle) and ``synth/`` (the seeded generator); nothing from
the CUDA path.  The histogram is a function of the records as a multiset (integer sums,
"both associative and commutative"), so the records are generated chunk by chunk
in draw order (``synth.draw_records``), which over [0, N) is the same multiset as the stream
and shuffled orders the GPU tests and the bench use; one digest per config serves both.

Membership: the oracle's literal linear scan (``oracle_classify_histogram_mt``) for the
16/64-entry lists; for C5's 4096-entry list the grouped-by-Z evaluation of the same Alg. 1
test (``oracle_member_bylen_batch``, pinned equal to the linear scan in
tests/test_oracle_pins.py) followed by ``oracle_histogram_members``.

Planes (u64 little endian, B = window / width bins each): out_count, out_bytes, in_count,
in_bytes; SHA-256 of each, plus the 12 totals (layout of sinet_oracle.c).

  python tools/oracle_digests.py c1 c2 c3 c4 c5 [--threads 8] [--chunk 33554432]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import core as oracle  # noqa: E402
from synth import WORKLOADS, prefix_table  # noqa: E402
from synth.sinet_synth import draw_records, to_numpy  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "digests.json")
PLANES = ("out_count", "out_bytes", "in_count", "in_bytes")


def plane_arrays(res):
    return {"out_count": res.count[0], "out_bytes": res.bytes[0], "in_count": res.count[1], "in_bytes": res.bytes[1]}


def digest_config(name: str, threads: int, chunk: int, log=print):
    wl = WORKLOADS[name]
    nets, lens = prefix_table(wl)
    res = oracle.OracleResult(wl.nbins)
    bylen = len(nets) > 256
    t0 = time.time()
    for lo in range(0, wl.n, chunk):
        hi = min(wl.n, lo + chunk)
        ts, src, dst, nb = to_numpy(draw_records(wl, lo, hi))[:4]
        if bylen:
            s_in = oracle.member_bylen(src, nets, lens, threads=threads)
            d_in = oracle.member_bylen(dst, nets, lens, threads=threads)
            oracle.histogram_members(ts, s_in, d_in, nb, wl.window_start_ms, wl.window_ms, wl.bin_width_ms, into=res)
        else:
            oracle.classify_histogram(ts, src, dst, nb, nets, lens, wl.window_start_ms, wl.window_ms,
                                      wl.bin_width_ms, threads=threads, into=res)
        log(f"  {name}: {hi:,}/{wl.n:,} records, {time.time() - t0:.0f} s")
    planes = plane_arrays(res)
    return {
        "n": wl.n, "nbins": wl.nbins, "window_start_ms": wl.window_start_ms, "window_ms": wl.window_ms,
        "bin_width_ms": wl.bin_width_ms, "prefixes": len(nets), "ts_mode": wl.ts_mode, "seed": wl.seed,
        "membership": "grouped by Z (oracle_member_bylen_batch)" if bylen else "linear scan (oracle_classify_histogram_mt)",
        "totals": [int(x) for x in res.totals],
        "sha256": {k: hashlib.sha256(np.ascontiguousarray(v).astype("<u8").tobytes()).hexdigest() for k, v in planes.items()},
        "nonzero_count_bins": {k: int(np.count_nonzero(planes[k])) for k in ("out_count", "in_count")},
        "oracle_seconds": round(time.time() - t0, 1),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--threads", type=int, default=len(os.sched_getaffinity(0)))
    ap.add_argument("--chunk", type=int, default=1 << 25)
    ap.add_argument("--out", default=OUT)
    a = ap.parse_args()
    torch.set_num_threads(a.threads)
    oracle.build()
    for name in a.configs:
        d = digest_config(name, a.threads, a.chunk)
        allv = {}
        if os.path.exists(a.out):
            with open(a.out) as f:
                allv = json.load(f)
        allv[name] = d
        allv["_about"] = ("SHA-256 of the oracle's full-size planes (u64 LE) and its 12 totals per BASELINE "
                          "config, written by tools/oracle_digests.py (oracle/ + synth/ only); order independent")
        tmp = a.out + ".tmp"
        with open(tmp, "w") as f:
            json.dump(allv, f, indent=1, sort_keys=True)
        os.replace(tmp, a.out)
        print(name, json.dumps(d["sha256"]), flush=True)


if __name__ == "__main__":
    main()
