"""ctypes wrapper of oracle/sinet_oracle.c.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Every function here is marshalling only; the arithmetic lives in the C file,
which cites the paper passage each step follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sinet_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

# direction-LUT presets, index s_in*2 + d_in -> 0 OUT, 1 IN, 2 NEITHER (A1/A2)
OUT, IN, NEITHER = 0, 1, 2
LUT_ALG1 = (IN, IN, OUT, OUT)              # Alg. 1 literal: source decides
LUT_SRC_PRIORITY = (NEITHER, IN, OUT, OUT)  # default
LUT_STRICT = (NEITHER, IN, OUT, NEITHER)


def build(force: bool = False) -> str:
    """Compile sinet_oracle.c with plain gcc (no CUDA, no product headers)."""
    with _lock:
        if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
            tmp = _LIB + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread",
                                   "-Wall", "-Wextra", "-o", tmp, _SRC])
            os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        u64p = ctypes.POINTER(ctypes.c_uint64)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        u8p = ctypes.POINTER(ctypes.c_uint8)
        lib.oracle_mask.argtypes = [ctypes.c_uint32]
        lib.oracle_mask.restype = ctypes.c_uint32
        lib.oracle_bitmask.argtypes = [ctypes.c_uint32, ctypes.c_uint32]
        lib.oracle_bitmask.restype = ctypes.c_uint32
        lib.oracle_member.argtypes = [ctypes.c_uint32, u32p, u8p, ctypes.c_uint32]
        lib.oracle_member.restype = ctypes.c_int
        common = [u64p, u32p, u32p, u64p, ctypes.c_uint64, u32p, u8p, ctypes.c_uint32,
                  ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, u8p, u64p, u64p, u64p]
        lib.oracle_classify_histogram.argtypes = common
        lib.oracle_classify_histogram.restype = None
        lib.oracle_classify_histogram_mt.argtypes = common + [ctypes.c_int]
        lib.oracle_classify_histogram_mt.restype = ctypes.c_int
        lib.oracle_tags.argtypes = [u64p, u32p, u32p, ctypes.c_uint64, u32p, u8p, ctypes.c_uint32,
                                    ctypes.c_uint64, ctypes.c_uint64, u8p]
        lib.oracle_tags.restype = None
        lib.oracle_histogram_members.argtypes = [u64p, u8p, u8p, u64p, ctypes.c_uint64, ctypes.c_uint64,
                                                 ctypes.c_uint64, ctypes.c_uint32, u8p, u64p, u64p, u64p]
        lib.oracle_histogram_members.restype = None
        lib.oracle_member_bylen_batch.argtypes = [u32p, ctypes.c_uint64, u32p, u8p, ctypes.c_uint32, u8p,
                                                  ctypes.c_int]
        lib.oracle_member_bylen_batch.restype = ctypes.c_int
        lib.oracle_member_lpm_batch.argtypes = [u32p, ctypes.c_uint64, u32p, u8p, u8p, ctypes.c_uint32, u8p]
        lib.oracle_member_lpm_batch.restype = None
        lib.oracle_watch_filter.argtypes = [u32p, u32p, ctypes.c_uint64, u32p, ctypes.c_uint32, u64p]
        lib.oracle_watch_filter.restype = ctypes.c_uint64
        lib.oracle_rebin.argtypes = [u64p, ctypes.c_uint64, ctypes.c_uint64, u64p]
        lib.oracle_rebin.restype = None
        lib.oracle_sparse.argtypes = [u64p, u64p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32,
                                      u64p, u64p, u64p, ctypes.c_uint64]
        lib.oracle_sparse.restype = ctypes.c_uint64
        lib.oracle_parse_text.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_int32, u64p, u32p, u32p,
                                          u64p, u8p, u64p]
        lib.oracle_parse_text.restype = None
        lib.oracle_parse_line.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_int32, u64p, u32p, u32p,
                                          u64p]
        lib.oracle_parse_line.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def mask(z: int) -> int:
    return int(_load().oracle_mask(z))


def bitmask(addr: int, z: int) -> int:
    return int(_load().oracle_bitmask(addr, z))


def _table(nets, lens):
    nets = np.ascontiguousarray(np.asarray(nets, dtype=np.uint32))
    lens = np.ascontiguousarray(np.asarray(lens, dtype=np.uint8))
    assert nets.shape == lens.shape
    return nets, lens


def member(ip: int, nets, lens) -> bool:
    nets, lens = _table(nets, lens)
    return bool(_load().oracle_member(ip, _ptr(nets, ctypes.c_uint32), _ptr(lens, ctypes.c_uint8), len(nets)))


class OracleResult:
    """count[dir][bin], bytes[dir][bin] (u64, dir 0 = OUT, 1 = IN) and totals[12]."""

    def __init__(self, nbins: int):
        self.nbins = nbins
        self.count = np.zeros((2, nbins), dtype=np.uint64)
        self.bytes = np.zeros((2, nbins), dtype=np.uint64)
        self.totals = np.zeros(12, dtype=np.uint64)

    # named views of the totals vector (layout documented in sinet_oracle.c)
    @property
    def m_count(self):
        return self.totals[0:4]

    @property
    def m_bytes(self):
        return self.totals[4:8]

    @property
    def oow_count(self):
        return self.totals[8:10]

    @property
    def oow_bytes(self):
        return self.totals[10:12]


def classify_histogram(ts, src, dst, nbytes, nets, lens, start: int, window: int, width: int,
                       lut=LUT_SRC_PRIORITY, threads: int = 1, into: OracleResult | None = None) -> OracleResult:
    """Run the oracle over one batch of records; accumulate into ``into`` if given."""
    lib = _load()
    ts = np.ascontiguousarray(ts, dtype=np.uint64)
    src = np.ascontiguousarray(src, dtype=np.uint32)
    dst = np.ascontiguousarray(dst, dtype=np.uint32)
    nbytes = np.ascontiguousarray(nbytes, dtype=np.uint64)
    n = len(ts)
    assert len(src) == n and len(dst) == n and len(nbytes) == n
    assert width >= 1 and window % width == 0
    nets, lens = _table(nets, lens)
    lut_a = np.ascontiguousarray(np.asarray(lut, dtype=np.uint8))
    res = into if into is not None else OracleResult(window // width)
    assert res.nbins == window // width
    args = (_ptr(ts, ctypes.c_uint64), _ptr(src, ctypes.c_uint32), _ptr(dst, ctypes.c_uint32),
            _ptr(nbytes, ctypes.c_uint64), n, _ptr(nets, ctypes.c_uint32), _ptr(lens, ctypes.c_uint8),
            len(nets), start, window, width, _ptr(lut_a, ctypes.c_uint8),
            _ptr(res.count, ctypes.c_uint64), _ptr(res.bytes, ctypes.c_uint64),
            _ptr(res.totals, ctypes.c_uint64))
    if threads <= 1:
        lib.oracle_classify_histogram(*args)
    else:
        rc = lib.oracle_classify_histogram_mt(*args, int(threads))
        if rc != 0:
            raise RuntimeError("oracle_classify_histogram_mt failed")
    return res


def tags(ts, src, dst, nets, lens, start: int, window: int) -> np.ndarray:
    lib = _load()
    ts = np.ascontiguousarray(ts, dtype=np.uint64)
    src = np.ascontiguousarray(src, dtype=np.uint32)
    dst = np.ascontiguousarray(dst, dtype=np.uint32)
    nets, lens = _table(nets, lens)
    out = np.zeros(len(ts), dtype=np.uint8)
    lib.oracle_tags(_ptr(ts, ctypes.c_uint64), _ptr(src, ctypes.c_uint32), _ptr(dst, ctypes.c_uint32),
                    len(ts), _ptr(nets, ctypes.c_uint32), _ptr(lens, ctypes.c_uint8), len(nets),
                    start, window, _ptr(out, ctypes.c_uint8))
    return out


def rebin(fine, factor: int) -> np.ndarray:
    """NEXT-1: coarse[k] = sum of fine[k*factor:(k+1)*factor] (u64, wraps)."""
    fine = np.ascontiguousarray(fine, dtype=np.uint64)
    out = np.zeros((len(fine) + factor - 1) // factor, dtype=np.uint64)
    _load().oracle_rebin(_ptr(fine, ctypes.c_uint64), len(fine), factor, _ptr(out, ctypes.c_uint64))
    return out


def sparse(count, nbytes, start: int, width: int):
    """NEXT-1: (bin start ms, count, bytes) of every nonzero-count bin, ascending."""
    count = np.ascontiguousarray(count, dtype=np.uint64)
    nbytes = np.ascontiguousarray(nbytes, dtype=np.uint64)
    cap = int(np.count_nonzero(count))
    t = np.zeros(cap, np.uint64)
    c = np.zeros(cap, np.uint64)
    b = np.zeros(cap, np.uint64)
    k = _load().oracle_sparse(_ptr(count, ctypes.c_uint64), _ptr(nbytes, ctypes.c_uint64), len(count), start, width,
                              _ptr(t, ctypes.c_uint64), _ptr(c, ctypes.c_uint64), _ptr(b, ctypes.c_uint64), cap)
    assert k == cap
    return t, c, b


def watch_filter(src, dst, watchlist) -> np.ndarray:
    """NEXT-2: indices of the records whose source or destination is listed (order kept)."""
    src = np.ascontiguousarray(src, dtype=np.uint32)
    dst = np.ascontiguousarray(dst, dtype=np.uint32)
    wl = np.ascontiguousarray(np.asarray(watchlist, dtype=np.uint32))
    keep = np.zeros(len(src), dtype=np.uint64)
    k = _load().oracle_watch_filter(_ptr(src, ctypes.c_uint32), _ptr(dst, ctypes.c_uint32), len(src),
                                    _ptr(wl, ctypes.c_uint32), len(wl), _ptr(keep, ctypes.c_uint64))
    return keep[:k].astype(np.int64)


def classify_histogram_watched(ts, src, dst, nbytes, nets, lens, watchlist, start, window, width,
                               lut=LUT_SRC_PRIORITY, threads: int = 1) -> OracleResult:
    """Filter by the watchlist (either endpoint), then the unchanged histogram."""
    keep = watch_filter(src, dst, watchlist)
    cols = [np.ascontiguousarray(np.asarray(c)[keep]) for c in (ts, src, dst, nbytes)]
    return classify_histogram(*cols, nets, lens, start, window, width, lut=lut, threads=threads)


def member_bylen(ips, nets, lens, threads: int = 1) -> np.ndarray:
    """Membership of every address (0/1), Alg. 1 l.4-9 grouped by Z (oracle_member_bylen_batch)."""
    ips = np.ascontiguousarray(np.asarray(ips, dtype=np.uint32))
    nets, lens = _table(nets, lens)
    out = np.zeros(len(ips), np.uint8)
    rc = _load().oracle_member_bylen_batch(_ptr(ips, ctypes.c_uint32), len(ips), _ptr(nets, ctypes.c_uint32),
                                           _ptr(lens, ctypes.c_uint8), len(nets), _ptr(out, ctypes.c_uint8),
                                           int(threads))
    if rc != 0:
        raise RuntimeError("oracle_member_bylen_batch failed")
    return out


def histogram_members(ts, s_in, d_in, nbytes, start: int, window: int, width: int, lut=LUT_SRC_PRIORITY,
                      into: OracleResult | None = None) -> OracleResult:
    """The histogram steps after discrimination with the memberships given per record
    (oracle_histogram_members); accumulates into ``into`` if given."""
    ts = np.ascontiguousarray(ts, dtype=np.uint64)
    nbytes = np.ascontiguousarray(nbytes, dtype=np.uint64)
    s_in = np.ascontiguousarray(s_in, dtype=np.uint8)
    d_in = np.ascontiguousarray(d_in, dtype=np.uint8)
    assert len(ts) == len(s_in) == len(d_in) == len(nbytes)
    res = into if into is not None else OracleResult(window // width)
    assert res.nbins == window // width
    lut_a = np.ascontiguousarray(np.asarray(lut, dtype=np.uint8))
    _load().oracle_histogram_members(_ptr(ts, ctypes.c_uint64), _ptr(s_in, ctypes.c_uint8), _ptr(d_in, ctypes.c_uint8),
                                     _ptr(nbytes, ctypes.c_uint64), len(ts), start, window, width,
                                     _ptr(lut_a, ctypes.c_uint8), _ptr(res.count, ctypes.c_uint64),
                                     _ptr(res.bytes, ctypes.c_uint64), _ptr(res.totals, ctypes.c_uint64))
    return res


def member_lpm(ips, nets, lens, labels) -> np.ndarray:
    """NEXT-4: membership under a labelled table (longest matching prefix decides)."""
    ips = np.ascontiguousarray(np.asarray(ips, dtype=np.uint32))
    nets, lens = _table(nets, lens)
    lab = np.ascontiguousarray(np.asarray(labels, dtype=np.uint8))
    out = np.zeros(len(ips), np.uint8)
    _load().oracle_member_lpm_batch(_ptr(ips, ctypes.c_uint32), len(ips), _ptr(nets, ctypes.c_uint32),
                                    _ptr(lens, ctypes.c_uint8), _ptr(lab, ctypes.c_uint8), len(nets),
                                    _ptr(out, ctypes.c_uint8))
    return out


def classify_histogram_lpm(ts, src, dst, nbytes, nets, lens, labels, start, window, width,
                           lut=LUT_SRC_PRIORITY) -> OracleResult:
    """NEXT-4: the histogram with membership decided by the labelled longest-prefix match."""
    ts = np.ascontiguousarray(ts, dtype=np.uint64)
    nbytes = np.ascontiguousarray(nbytes, dtype=np.uint64)
    s_in = member_lpm(src, nets, lens, labels)
    d_in = member_lpm(dst, nets, lens, labels)
    res = OracleResult(window // width)
    lut_a = np.ascontiguousarray(np.asarray(lut, dtype=np.uint8))
    _load().oracle_histogram_members(_ptr(ts, ctypes.c_uint64), _ptr(s_in, ctypes.c_uint8), _ptr(d_in, ctypes.c_uint8),
                                     _ptr(nbytes, ctypes.c_uint64), len(ts), start, window, width,
                                     _ptr(lut_a, ctypes.c_uint8), _ptr(res.count, ctypes.c_uint64),
                                     _ptr(res.bytes, ctypes.c_uint64), _ptr(res.totals, ctypes.c_uint64))
    return res


# NEXT-3 line status codes (readings A27-A31)
PARSE_OK, PARSE_LONG, PARSE_COLUMNS, PARSE_TIME, PARSE_SRC, PARSE_DST, PARSE_BYTES = range(7)


class ParseResult:
    def __init__(self, ts, src, dst, nbytes, status):
        self.ts, self.src, self.dst, self.bytes, self.status = ts, src, dst, nbytes, status

    @property
    def n_lines(self):
        return len(self.status)

    @property
    def n_valid(self):
        return len(self.ts)


def parse_text(text: bytes, tz_offset_min: int = 0) -> ParseResult:
    """NEXT-3: PA-7080 session-log text (Table 1) -> (ts, src, dst, bytes) of the
    valid lines in line order + a status per line."""
    text = bytes(text)
    cap = text.count(b"\n") + 1
    ts = np.zeros(cap, np.uint64)
    src = np.zeros(cap, np.uint32)
    dst = np.zeros(cap, np.uint32)
    nb = np.zeros(cap, np.uint64)
    st = np.zeros(cap, np.uint8)
    out = np.zeros(2, np.uint64)
    _load().oracle_parse_text(text, len(text), tz_offset_min, _ptr(ts, ctypes.c_uint64), _ptr(src, ctypes.c_uint32),
                              _ptr(dst, ctypes.c_uint32), _ptr(nb, ctypes.c_uint64), _ptr(st, ctypes.c_uint8),
                              _ptr(out, ctypes.c_uint64))
    n, v = int(out[0]), int(out[1])
    return ParseResult(ts[:v], src[:v], dst[:v], nb[:v], st[:n])


def parse_line(line: bytes, tz_offset_min: int = 0):
    """One line's (status, ts, src, dst, bytes)."""
    ts, nb = ctypes.c_uint64(0), ctypes.c_uint64(0)
    s, d = ctypes.c_uint32(0), ctypes.c_uint32(0)
    st = _load().oracle_parse_line(bytes(line), len(line), tz_offset_min, ctypes.byref(ts), ctypes.byref(s),
                                   ctypes.byref(d), ctypes.byref(nb))
    return st, ts.value, s.value, d.value, nb.value
