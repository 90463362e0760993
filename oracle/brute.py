"""Second, independent oracle (O2) in pure Python.  TEST INFRASTRUCTURE ONLY.

Used to pin oracle/sinet_oracle.c on small inputs by methods that share none
of its arithmetic:
  * membership by comparing the first Z characters of 32-character binary
    strings (the "32-bit sequence" of P:L174-175, compared bit by bit);
  * membership by Python's ``ipaddress`` library (``ip in ip_network(c, strict=False)``);
  * histograms with ``collections.Counter`` keyed by (dir, ms bin) (P:L217's
    key-value namespaces X1<timestamp>, X1<count>, X2<bytes>), Python ints
    reduced mod 2^64 only at the end.
"""
from __future__ import annotations

import ipaddress
from collections import Counter

M64 = (1 << 64) - 1


def bits32(x: int) -> str:
    return format(x, "032b")


def member_bitstring(ip: int, nets, lens) -> bool:
    """Any CIDR whose first Z bits equal the address's first Z bits (reading A3)."""
    s = bits32(ip)
    return any(s[:z] == bits32(int(n))[:z] for n, z in zip(nets, lens))


def member_ipaddress(ip: int, nets, lens) -> bool:
    a = ipaddress.IPv4Address(int(ip))
    return any(a in ipaddress.IPv4Network((int(n), int(z)), strict=False) for n, z in zip(nets, lens))


def histogram_counter(ts, src, dst, nbytes, nets, lens, start, window, width, lut):
    """Returns (count Counter, bytes Counter keyed by (dir, bin)), m_count, m_bytes, oow_count, oow_bytes."""
    cnt, byt = Counter(), Counter()
    m_count, m_bytes = [0] * 4, [0] * 4
    oow_c, oow_b = [0, 0], [0, 0]
    memo = {}

    def mem(ip):
        if ip not in memo:
            memo[ip] = member_bitstring(ip, nets, lens)
        return memo[ip]

    for t, s, d, b in zip(ts, src, dst, nbytes):
        t, s, d, b = int(t), int(s), int(d), int(b)
        cell = 2 * int(mem(s)) + int(mem(d))
        m_count[cell] += 1
        m_bytes[cell] += b
        direction = lut[cell]
        if direction not in (0, 1):
            continue
        off = t - start
        if off < 0 or off >= window:
            oow_c[direction] += 1
            oow_b[direction] += b
            continue
        key = (direction, off // width)
        cnt[key] += 1
        byt[key] += b
    byt = Counter({k: v & M64 for k, v in byt.items()})
    return (cnt, byt, [c & M64 for c in m_count], [c & M64 for c in m_bytes],
            [c & M64 for c in oow_c], [c & M64 for c in oow_b])


def member_lpm_bitstring(ip: int, nets, lens, labels) -> bool:
    """Longest matching prefix (by bit strings) decides; no match -> outside."""
    s = bits32(ip)
    best, lab = -1, False
    for n, z, l in zip(nets, lens, labels):
        z = int(z)
        if s[:z] == bits32(int(n))[:z] and z >= best:
            best, lab = z, bool(l)
    return lab


# ----------------------------------------------------------------------------- NEXT-3
_TIME_RE = None


def parse_line_python(line: bytes, tz_offset_min: int = 0):
    """PA-7080 line (Table 1) by Python's own libraries: str.split, a regular
    expression for the capture_time shape, datetime (calendar validity), calendar.timegm
    (epoch seconds), ipaddress.IPv4Address (dotted quad), int() (bytes).  Returns
    (status, ts_ms, src, dst, bytes) with the status codes of oracle/core.py."""
    import calendar
    import datetime
    import re
    global _TIME_RE
    if _TIME_RE is None:
        _TIME_RE = re.compile(rb"(\d{4})/(\d{2})/(\d{2}) (\d{2}):(\d{2}):(\d{2})\.(\d{3})")
    if len(line) > 2047:
        return 1, 0, 0, 0, 0
    if line.endswith(b"\r"):
        line = line[:-1]
    f = line.split(b",")
    if len(f) != 24:
        return 2, 0, 0, 0, 0
    m = _TIME_RE.fullmatch(f[0])
    ts = None
    if m:
        try:
            Y, M, D, h, mi, s, ms = (int(x) for x in m.groups())
            dt = datetime.datetime(Y, M, D, h, mi, s)
            if Y >= 1970:
                ts = (calendar.timegm(dt.timetuple()) * 1000 + ms) - tz_offset_min * 60000
                if ts < 0:
                    ts = None
        except ValueError:
            ts = None
    if ts is None:
        return 3, 0, 0, 0, 0
    ips = []
    for k, code in ((4, 4), (7, 5)):
        try:
            txt = f[k].decode("ascii")
            if not all(c in "0123456789." for c in txt):
                raise ValueError
            ips.append(int(ipaddress.IPv4Address(txt)))
        except (ValueError, UnicodeDecodeError):
            return code, 0, 0, 0, 0
    b = f[20]
    if not (1 <= len(b) <= 20 and all(48 <= c <= 57 for c in b)) or int(b) > M64:
        return 6, 0, 0, 0, 0
    return 0, ts, ips[0], ips[1], int(b)


def parse_text_python(text: bytes, tz_offset_min: int = 0):
    """Lines = text.split(b"\\n") without the empty piece after a final newline."""
    lines = text.split(b"\n")
    if lines and lines[-1] == b"":
        lines.pop()
    return [parse_line_python(l, tz_offset_min) for l in lines]
