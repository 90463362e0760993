"""Small test-side helpers (parsing fixtures).  Holds none of the method's arithmetic."""
import ipaddress
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def ip(s: str) -> int:
    return int(ipaddress.IPv4Address(s))


def cidr(s: str):
    addr, z = s.split("/")
    return ip(addr), int(z)


def load_f0():
    with open(os.path.join(GOLDEN, "f0.json")) as f:
        g = json.load(f)
    start = g["window_start_ms"]
    tab = [cidr(c) for c in g["table"]]
    nets = np.array([t[0] for t in tab], dtype=np.uint32)
    lens = np.array([t[1] for t in tab], dtype=np.uint8)
    recs = g["records"]
    ts = np.array([start + r[0] for r in recs], dtype=np.uint64)
    src = np.array([ip(r[1]) for r in recs], dtype=np.uint32)
    dst = np.array([ip(r[2]) for r in recs], dtype=np.uint32)
    nb = np.array([r[3] for r in recs], dtype=np.uint64)
    return g, nets, lens, ts, src, dst, nb


def dense_from_sparse(sparse: dict, nbins: int):
    c = np.zeros(nbins, dtype=np.uint64)
    b = np.zeros(nbins, dtype=np.uint64)
    for k, (cnt, byt) in sparse.items():
        c[int(k)] = cnt
        b[int(k)] = byt
    return c, b


def edge_addresses(nets, lens):
    """Every table interval's first/last address and their +-1 neighbours (generation only)."""
    out = []
    for n, z in zip(nets.tolist(), lens.tolist()):
        size = 1 << (32 - z)
        first = n
        last = n + size - 1
        for a in (first - 1, first, first + 1, last - 1, last, last + 1):
            if 0 <= a <= 0xFFFFFFFF:
                out.append(a)
    out += [0, 1, 0x7FFFFFFF, 0x80000000, 0xFFFFFFFE, 0xFFFFFFFF]
    return np.array(sorted(set(out)), dtype=np.uint32)
