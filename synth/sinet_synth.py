"""Counter-based synthetic session-record generator (torch, CPU or CUDA; bit-identical on both).

Recipe:
  * every random draw is splitmix64(key(seed, stream) + GOLDEN * global_index), so
    any shard [lo, hi) of a workload can be generated alone, on any device;
  * record columns are the four Table 1 fields the path reads: capture_time
    (epoch ms), source_ip / destination_ip (u32, first
    octet most significant), bytes;
  * timestamps: "uniform" over the window or "bursty" (diurnal base + Zipf
    bursts + one hot millisecond); "stream" order = sorted by arrival key with a
    U{0..2000} ms capture delay (records approximately time ordered, as day log
    files processed chunk by chunk), or "shuffled" = a seeded
    permutation of the stream order (Feistel bijection, computable per shard);
  * endpoint classes: OUT-external 45.6 %, OUT-internal 2.4 %, IN 47 %,
    NEITHER 5 %; an inside address is a uniformly chosen table entry plus
    uniform host bits, an outside address lies in a /8 that holds no table
    entry (by construction of the table), so the intended class is ground truth;
  * bytes: 5 % zero, else an integer lognormal(7, 2) quantile table, plus
    ceil(N * 1e-7) "elephants" in [2^32, 2^40).
Floating point is used only while building small integer tables in pure
Python (identical on every x86 box); all per-record arithmetic is int64.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace
from statistics import NormalDist

import numpy as np
import torch

SEED_BASE = 2106128630
M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
DAY_START_JST = 1613660400000   # 2021-02-19 00:00 JST, Table 2's 1,632,300,495-session day
DAY_MS = 86_400_000             # 60*60*24*1000

# streams (independent draw families)
(S_KEY, S_DELAY, S_CLASS, S_SPFX, S_SHOST, S_DPFX, S_DHOST, S_BYTES, S_BYTES2, S_ELE,
 S_PERM, S_TABLE, S_BURST) = range(1, 14)

# first octets: table entries live only in HOME_8, outside addresses only in OUTSIDE_8
HOME_8 = [o for o in range(1, 127) if o != 10] + [133]
OUTSIDE_8 = [o for o in range(128, 224) if o != 133]


def _s64(x: int) -> int:
    x &= M64
    return x - (1 << 64) if x >= (1 << 63) else x


def _splitmix_int(z: int) -> int:
    z &= M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def _stream_key(seed: int, stream: int) -> int:
    return _splitmix_int(_splitmix_int(seed) ^ (stream * 0xD1B54A32D192ED03))


_C1 = _s64(0xBF58476D1CE4E5B9)
_C2 = _s64(0x94D049BB133111EB)
_G = _s64(GOLDEN)


def _srl(x: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of int64 bit patterns."""
    return (x >> k) & ((1 << (64 - k)) - 1)


def rand64(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    """splitmix64(key + GOLDEN*idx) as int64 bit patterns (wrapping arithmetic)."""
    z = idx * _G + _s64(_stream_key(seed, stream))
    z = (z ^ _srl(z, 30)) * _C1
    z = (z ^ _srl(z, 27)) * _C2
    return z ^ _srl(z, 31)


def _below(r: torch.Tensor, m) -> torch.Tensor:
    """Uniform integer in [0, m) from a 64-bit draw, m <= 2^31 (scalar or tensor)."""
    return (_srl(r, 33) * m) >> 31


class _PyRng:
    """Scalar splitmix64 sequence for building tables in pure Python."""

    def __init__(self, seed: int, stream: int):
        self.k = _stream_key(seed, stream)
        self.i = 0

    def next(self) -> int:
        v = _splitmix_int(self.k + GOLDEN * self.i)
        self.i += 1
        return v

    def below(self, m: int) -> int:
        return ((self.next() >> 33) * m) >> 31


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    window_ms: int
    n_prefixes: int
    table: str = "sinet"          # "sinet" | "mixed"
    ts_mode: str = "uniform"      # "uniform" | "bursty"
    order: str = "stream"         # "stream" | "shuffled"
    bin_width_ms: int = 1
    window_start_ms: int = DAY_START_JST
    disorder_ms: int = 2000
    seed: int = SEED_BASE

    def with_(self, **kw) -> "Workload":
        return replace(self, **kw)

    @property
    def nbins(self) -> int:
        return self.window_ms // self.bin_width_ms


# BASELINE.json configs[0..4]
WORKLOADS = {
    "c1": Workload("c1", 1_000_000, 3_600_000, 16, seed=SEED_BASE + 1),
    "c2": Workload("c2", 100_000_000, DAY_MS, 64, seed=SEED_BASE + 2),
    "c3": Workload("c3", 1_200_000_000, DAY_MS, 64, seed=SEED_BASE + 3),
    "c4": Workload("c4", 1_600_000_000, DAY_MS, 64, ts_mode="bursty", seed=SEED_BASE + 4),
    "c5": Workload("c5", 400_000_000, DAY_MS, 4096, table="mixed", seed=SEED_BASE + 5),
}


def window_of(wl: Workload):
    return wl.window_start_ms, wl.window_ms, wl.bin_width_ms


# --------------------------------------------------------------------------- prefix tables
def _host_clear(net: int, ln: int) -> int:
    # generation-side helper: the entry is stored normalised (host bits zero)
    return net & ~((1 << (32 - ln)) - 1) & 0xFFFFFFFF if ln < 32 else net


def prefix_table(wl: Workload):
    """Returns (nets uint32[P], lens uint8[P]); deterministic from wl.seed."""
    rng = _PyRng(wl.seed, S_TABLE)
    seen = set()
    nets, lens = [], []
    if wl.table == "sinet":
        # lengths 50% /16, 25% /17-/20, 15% /21-/24, 10% /12-/15; 60% inside 133/8
        while len(nets) < wl.n_prefixes:
            u = rng.below(100)
            if u < 50:
                ln = 16
            elif u < 75:
                ln = 17 + rng.below(4)
            elif u < 90:
                ln = 21 + rng.below(4)
            else:
                ln = 12 + rng.below(4)
            if rng.below(100) < 60:
                o8 = 133
            else:
                o8 = HOME_8[rng.below(len(HOME_8) - 1)]   # excludes the trailing 133
            net = _host_clear((o8 << 24) | (rng.next() >> 40), ln)
            if (net, ln) in seen:
                continue
            seen.add((net, ln))
            nets.append(net)
            lens.append(ln)
    elif wl.table == "mixed":
        # lengths uniform /8-/32, /8-/11 capped at 2 each, 30% nested in an earlier shorter entry
        cap = {8: 2, 9: 2, 10: 2, 11: 2}
        used = {k: 0 for k in cap}
        while len(nets) < wl.n_prefixes:
            ln = 8 + rng.below(25)
            if ln in cap and used[ln] >= cap[ln]:
                continue
            parents = None
            if nets and rng.below(100) < 30:
                j = rng.below(len(nets))
                if lens[j] < ln:
                    parents = j
            if parents is not None:
                pn, pl = nets[parents], lens[parents]
                host = (rng.next() >> 32) & ((1 << (32 - pl)) - 1)
                net = _host_clear(pn | host, ln)
            else:
                o8 = HOME_8[rng.below(len(HOME_8))]
                net = _host_clear((o8 << 24) | (rng.next() >> 40), ln)
            if (net, ln) in seen:
                continue
            if ln in cap:
                used[ln] += 1
            seen.add((net, ln))
            nets.append(net)
            lens.append(ln)
    else:
        raise ValueError(wl.table)
    return np.asarray(nets, dtype=np.uint32), np.asarray(lens, dtype=np.uint8)


# --------------------------------------------------------------------------- integer tables
def _lognormal_table(k: int = 1024, mu: float = 7.0, sigma: float = 2.0):
    nd = NormalDist(mu, sigma)
    q = []
    for i in range(k + 1):
        p = min(max(i / k, 1e-9), 1 - 1e-9)
        v = int(math.floor(math.exp(nd.inv_cdf(p))))
        q.append(min(max(v, 1), (1 << 40) - 1))
    return q


_LOGN = _lognormal_table()


def _diurnal_weights():
    # hourly weight 1 + 0.8 sin(2 pi (h - 8) / 24): peak ~14:00 JST (cf. P:L324 diurnal pattern)
    return [int(round(1e6 * (1 + 0.8 * math.sin(2 * math.pi * (h - 8) / 24)))) for h in range(24)]


def _bursts(wl: Workload, nb: int = 1024):
    rng = _PyRng(wl.seed, S_BURST)
    w = [1.0 / ((i + 1) ** 1.1) for i in range(nb)]
    tot = sum(w)
    cw = []
    acc = 0
    for x in w:
        acc += int(round((1 << 30) * x / tot))
        cw.append(acc)
    centers, widths = [], []
    for _ in range(nb):
        centers.append(rng.below(wl.window_ms))
        widths.append(max(1, int(math.floor(10 ** (4 * (rng.next() >> 11) / float(1 << 53))))))
    hot = rng.below(wl.window_ms)
    return cw, centers, widths, hot


def _ts_offsets(wl: Workload, idx: torch.Tensor) -> torch.Tensor:
    """Capture-time offset (ms from window start) of draw idx.

    uniform: U[-margin, W + margin) with a 1000 ms margin, so a sprinkle of
    records falls outside the window (log files overlap the day boundary).
    bursty: 60 % diurnal base, 39 % in 1024 Zipf(1.1) bursts, 1 % in one hot ms.
    """
    r = rand64(wl.seed, S_KEY, idx)
    if wl.ts_mode == "uniform":
        return _below(r, wl.window_ms + 2 * _MARGIN) - _MARGIN
    if wl.ts_mode != "bursty":
        raise ValueError(wl.ts_mode)
    dev = idx.device
    comp = _below(r, 1000)
    r2 = rand64(wl.seed, S_KEY + 100, idx)
    # diurnal base: hour by integer cumulative weights, then uniform ms inside the hour
    cdw = torch.tensor(np.cumsum(_diurnal_weights()), dtype=torch.int64, device=dev)
    hour_ms = wl.window_ms // 24
    hour = torch.searchsorted(cdw, _below(r2, int(cdw[-1].item())), right=True).clamp_(max=23)
    base = hour * hour_ms + _below(rand64(wl.seed, S_KEY + 101, idx), hour_ms)
    cw, centers, widths, hot = _bursts(wl)
    cwt = torch.tensor(cw, dtype=torch.int64, device=dev)
    b = torch.searchsorted(cwt, _below(r2, int(cw[-1])), right=True).clamp_(max=len(cw) - 1)
    ct = torch.tensor(centers, dtype=torch.int64, device=dev)[b]
    wt = torch.tensor(widths, dtype=torch.int64, device=dev)[b]
    burst = (ct + _below(rand64(wl.seed, S_KEY + 102, idx), wt) - wt // 2).clamp_(0, wl.window_ms - 1)
    return torch.where(comp < 600, base, torch.where(comp < 990, burst, torch.full_like(base, hot)))


_MARGIN = 1000
_CHUNK = 1 << 26


def stream_order(wl: Workload, device) -> torch.Tensor:
    """Draw index at each stream position: draws sorted by arrival = capture + delay,
    delay ~ U{0..disorder}, ties by draw index (packed sort key, unique)."""
    assert wl.n < (1 << 32)
    parts = []
    for lo in range(0, wl.n, _CHUNK):
        idx = torch.arange(lo, min(wl.n, lo + _CHUNK), dtype=torch.int64, device=device)
        arrival = _ts_offsets(wl, idx) + _MARGIN + _below(rand64(wl.seed, S_DELAY, idx), wl.disorder_ms + 1)
        parts.append((arrival << 32) | idx)
    packed = torch.cat(parts) if len(parts) > 1 else parts[0]
    del parts
    packed = torch.sort(packed).values
    return packed & 0xFFFFFFFF


def _feistel_perm(j: torch.Tensor, n: int, seed: int) -> torch.Tensor:
    """Seeded bijection of [0, n) (balanced Feistel on 2*h bits + cycle walking)."""
    bits = max(2, (n - 1).bit_length())
    bits += bits & 1
    h = bits // 2
    hm = (1 << h) - 1
    x = j.clone()
    todo = torch.ones_like(x, dtype=torch.bool)
    out = x.clone()
    for _ in range(512):   # (1 - n / 2^bits)^512 < 1e-70: every element has left the cycle walk
        l, r = x >> h, x & hm
        for rnd in range(4):
            f = rand64(seed, S_PERM + 1000 * rnd, r) & hm
            l, r = r, l ^ f
        y = (l << h) | r
        done_now = todo & (y < n)
        out = torch.where(done_now, y, out)
        todo = todo & ~done_now
        if not bool(todo.any()):
            return out
        x = torch.where(todo, y, x)
    raise RuntimeError("feistel cycle walk did not terminate")


def _to_u32_bits(x: torch.Tensor) -> torch.Tensor:
    return torch.where(x >= (1 << 31), x - (1 << 32), x).to(torch.int32)


def records(wl: Workload, lo: int = 0, hi: int | None = None, device="cpu", order=None):
    """Records at stream/shuffled positions [lo, hi) of workload ``wl``.

    Returns dict of tensors on ``device``: ts int64 (epoch ms), src/dst int32
    (u32 bit patterns), bytes int64 (u64 bit patterns), cls uint8 (intended
    s_in*2 + d_in, ground truth by construction).
    """
    hi = wl.n if hi is None else hi
    assert 0 <= lo <= hi <= wl.n
    device = torch.device(device)
    if order is None:
        order = stream_order(wl, device)
    pos = torch.arange(lo, hi, dtype=torch.int64, device=device)
    if wl.order == "shuffled":
        pos = _feistel_perm(pos, wl.n, wl.seed)
    i = order[pos].to(torch.int64)     # draw index; every per-record draw is keyed by it
    return _records_of_draws(wl, i)


def records_into(wl: Workload, lo: int, hi: int, device, order=None, chunk: int = _CHUNK):
    """``records(wl, lo, hi)`` without the ``cls`` column, generated ``chunk`` records at a time
    into preallocated columns, so a 1.6 B-record shard needs ~its 24 B/record plus one chunk of
    temporaries (the one-shot ``records()`` holds a dozen N-sized int64 temporaries)."""
    device = torch.device(device)
    if order is None:
        order = stream_order(wl, device)
    n = hi - lo
    out = {"ts": torch.empty(n, dtype=torch.int64, device=device),
           "src": torch.empty(n, dtype=torch.int32, device=device),
           "dst": torch.empty(n, dtype=torch.int32, device=device),
           "bytes": torch.empty(n, dtype=torch.int64, device=device)}
    for a in range(lo, hi, chunk):
        b = min(hi, a + chunk)
        r = records(wl, a, b, device=device, order=order)
        for k in out:
            out[k][a - lo:b - lo].copy_(r[k])
        del r
    return out


def draw_records(wl: Workload, lo: int, hi: int, device="cpu"):
    """Records of draws [lo, hi) in draw order (no arrival sort).  Over [0, N) this is the
    same multiset of records as ``records()`` in either order, so order-independent results
    (the histogram) can be produced chunk by chunk without the global sort."""
    assert 0 <= lo <= hi <= wl.n
    return _records_of_draws(wl, torch.arange(lo, hi, dtype=torch.int64, device=torch.device(device)))


def _records_of_draws(wl: Workload, i: torch.Tensor):
    device = i.device
    ts = wl.window_start_ms + _ts_offsets(wl, i)

    # endpoint classes
    u = _below(rand64(wl.seed, S_CLASS, i), 1000)
    s_in = (u < 480).to(torch.int64)                                   # 45.6 % + 2.4 %
    d_in = ((u >= 456) & (u < 950)).to(torch.int64)                    # 2.4 % + 47 %
    nets, lens = prefix_table(wl)
    nets_t = torch.tensor(nets.astype(np.int64), device=device)
    lens_t = torch.tensor(lens.astype(np.int64), device=device)
    out8 = torch.tensor(OUTSIDE_8, dtype=torch.int64, device=device)

    def addr(inside, s_pfx, s_host):
        rp = rand64(wl.seed, s_pfx, i)
        k = _below(rp, len(nets))
        host = _srl(rand64(wl.seed, s_host, i), 32)
        ln = lens_t[k]
        hostmask = (torch.ones_like(ln) << (32 - ln)) - 1
        a_in = nets_t[k] | (host & hostmask)
        a_out = (out8[_below(rp, len(OUTSIDE_8))] << 24) | (host & 0xFFFFFF)
        return torch.where(inside.bool(), a_in, a_out)

    src = addr(s_in, S_SPFX, S_SHOST)
    dst = addr(d_in, S_DPFX, S_DHOST)

    # bytes
    rb = rand64(wl.seed, S_BYTES, i)
    zero = _below(rb, 1000) < 50
    q = torch.tensor(_LOGN, dtype=torch.int64, device=device)
    r2 = rand64(wl.seed, S_BYTES2, i)
    kq = _srl(r2, 54)                       # 10 bits -> quantile cell
    frac = _srl(r2, 33) & ((1 << 20) - 1)   # 20-bit interpolation
    lo_q, hi_q = q[kq], q[kq + 1]
    nb = lo_q + (((hi_q - lo_q) * frac) >> 20)
    n_ele = -(-wl.n // 10_000_000)          # ceil(N * 1e-7)
    is_ele = ((i + 1) * n_ele) // wl.n > (i * n_ele) // wl.n
    ele = (1 << 32) + _below(rand64(wl.seed, S_ELE, i), 1 << 31) * 510   # in [2^32, 2^40)
    nbytes = torch.where(is_ele, ele, torch.where(zero, torch.zeros_like(nb), nb))

    cls = (s_in * 2 + d_in).to(torch.uint8)
    return {"ts": ts, "src": _to_u32_bits(src), "dst": _to_u32_bits(dst), "bytes": nbytes, "cls": cls}


def to_numpy(rec):
    """Host numpy views with the oracle's dtypes (u64 / u32 / u32 / u64)."""
    return (rec["ts"].cpu().numpy().view(np.uint64), rec["src"].cpu().numpy().view(np.uint32),
            rec["dst"].cpu().numpy().view(np.uint32), rec["bytes"].cpu().numpy().view(np.uint64))
