"""Seeded PA-7080 session-log text (Table 1) for the NEXT-3 parser.

Input generation only: it renders records from ``synth.records`` as comma-separated
lines of the 24 Table 1 items and can inject malformed lines whose intended line
status is recorded (ground truth by construction).  It holds none of the parser's
arithmetic: calendar dates come from Python's ``datetime`` (one string per distinct
second of the window, looked up per record), numbers are rendered digit by digit.
Runs on any torch device (GPU generation keeps bench-size text off the host).
"""
from __future__ import annotations

import datetime

import numpy as np
import torch

from .sinet_synth import Workload, _below, _srl, rand64

# streams of the text draws (disjoint from sinet_synth's 1..13)
S_PORT, S_PORT2, S_CC, S_MISC, S_PKT, S_ELAPSED, S_BAD, S_BADKIND = range(40, 48)

# intended line status (the parser's codes, A27-A31)
OK, LONG, COLUMNS, TIME, SRC, DST, BYTES = range(7)

_CC = [b"JP", b"US", b"CN", b"DE", b"GB", b"KR", b"FR", b"NL", b"SG", b"NA"]
_PROTO = [b"tcp", b"udp", b"icmp"]
_APP = [b"ssl", b"web-browsing", b"dns", b"incomplete", b"quic", b"ntp", b"ms-update",
        b"google-base", b"insufficient-data", b"smtp", b"ssh", b"not-applicable"]
_SUBTYPE = [b"end", b"start", b"drop", b"deny"]
_ACTION = [b"allow", b"deny", b"drop", b"reset-both"]
_REASON = [b"tcp-fin", b"aged-out", b"tcp-rst-from-client", b"tcp-rst-from-server", b"policy-deny",
           b"threat", b"n/a"]
_CATEGORY = [b"computer-and-internet-info", b"search-engines", b"business-and-economy", b"content-delivery-networks",
             b"unknown", b"any", b"educational-institutions", b"internet-communications-and-telephony"]
_DEVICE = [b"PA-7080-SINET-TOKYO-01", b"PA-7080-SINET-OSAKA-01", b"PA-7080-SINET-TOKYO-02"]


class _Piece:
    """A column of variable-length byte strings: chars (n, w) uint8 + lengths (n,)."""

    def __init__(self, chars: torch.Tensor, lens: torch.Tensor):
        self.chars, self.lens = chars, lens


def _vocab(words, idx: torch.Tensor) -> _Piece:
    w = max(len(x) for x in words)
    tab = torch.zeros(len(words), w, dtype=torch.uint8)
    ln = torch.tensor([len(x) for x in words], dtype=torch.int64)
    for i, x in enumerate(words):
        if x:
            tab[i, :len(x)] = torch.tensor(list(x), dtype=torch.uint8)
    tab, ln = tab.to(idx.device), ln.to(idx.device)
    return _Piece(tab[idx], ln[idx])


def _decimal(x: torch.Tensor, width: int = 20) -> _Piece:
    """Non-negative int64 -> shortest decimal digits (0 -> "0")."""
    n = x.shape[0]
    d = torch.empty(n, width, dtype=torch.uint8, device=x.device)
    v = x.clone()
    for k in range(width - 1, -1, -1):       # least significant digit last
        d[:, k] = (v % 10).to(torch.uint8) + 48
        v = v // 10
    nd = torch.ones(n, dtype=torch.int64, device=x.device)
    p = 10
    for k in range(1, width):
        nd += (x >= p).to(torch.int64)
        if p > (1 << 62) // 10:
            break
        p *= 10
    # left-align: shift the nd significant digits to the front
    cols = torch.arange(width, device=x.device).unsqueeze(0) + (width - nd).unsqueeze(1)
    cols = cols.clamp(max=width - 1)
    return _Piece(torch.gather(d, 1, cols), nd)


def _concat(pieces, sep: int | None = None) -> _Piece:
    n = pieces[0].lens.shape[0]
    w = sum(p.chars.shape[1] for p in pieces) + (len(pieces) - 1 if sep is not None else 0)
    dev = pieces[0].lens.device
    out = torch.zeros(n, w, dtype=torch.uint8, device=dev)
    pos = torch.zeros(n, dtype=torch.int64, device=dev)
    rows = torch.arange(n, device=dev).unsqueeze(1)
    for i, p in enumerate(pieces):
        if i and sep is not None:
            out[torch.arange(n, device=dev), pos] = sep
            pos = pos + 1
        pw = p.chars.shape[1]
        j = torch.arange(pw, device=dev).unsqueeze(0)
        m = j < p.lens.unsqueeze(1)
        cols = (pos.unsqueeze(1) + j).clamp(max=w - 1)
        out[rows.expand(-1, pw)[m], cols[m]] = p.chars[m]
        pos = pos + p.lens
    return _Piece(out, pos)


def _ipv4(a: torch.Tensor) -> _Piece:
    """u32 bit patterns (int32/int64 tensor) -> dotted quad."""
    a = a.to(torch.int64) & 0xFFFFFFFF
    octs = [_decimal((a >> s) & 255, 3) for s in (24, 16, 8, 0)]
    return _concat(octs, sep=ord("."))


def _second_table(lo_s: int, hi_s: int, tz_offset_min: int):
    """"YYYY/MM/DD HH:MM:SS" of every second in [lo_s, hi_s] (local time), via datetime."""
    tz = datetime.timezone(datetime.timedelta(minutes=tz_offset_min))
    rows = []
    for s in range(lo_s, hi_s + 1):
        t = datetime.datetime.fromtimestamp(s, tz)
        rows.append(t.strftime("%Y/%m/%d %H:%M:%S").encode())
    tab = np.frombuffer(b"".join(rows), dtype=np.uint8).reshape(len(rows), 19)
    return torch.from_numpy(tab.copy())


def session_text(wl: Workload, rec: dict, tz_offset_min: int = 540, bad_per_million: int = 0,
                 crlf: bool = False, salt: int = 0):
    """Render records (dict from synth.records, same device) as PA-7080 lines.

    Returns (text uint8 tensor, intended status uint8 per line).  With
    ``bad_per_million`` > 0 that share of lines is made malformed in one of six ways
    (each with its intended status); the others parse to exactly the record's
    (ts, src, dst, bytes).  tz_offset_min: the local time of the log (JST = +540).
    """
    ts = rec["ts"]
    n = ts.shape[0]
    dev = ts.device
    idx = torch.arange(n, dtype=torch.int64, device=dev) + salt * 1_000_003
    seed = wl.seed

    # capture_time: per-second strings from datetime + ".mmm"
    local = ts + tz_offset_min * 60_000
    sec = torch.div(ts, 1000, rounding_mode="floor")
    lo_s, hi_s = int(sec.min()) - 7200, int(sec.max()) + 60
    tab = _second_table(lo_s, hi_s, tz_offset_min).to(dev)
    ms = local - torch.div(local, 1000, rounding_mode="floor") * 1000
    cap = torch.cat([tab[sec - lo_s], torch.full((n, 1), ord("."), dtype=torch.uint8, device=dev),
                     _decimal(ms + 1000, 4).chars[:, 1:4]], dim=1)
    capture = _Piece(cap, torch.full((n,), 23, dtype=torch.int64, device=dev))
    elapsed = _below(rand64(seed, S_ELAPSED, idx), 120)
    gen = _Piece(tab[(sec - lo_s + 1).clamp(max=hi_s - lo_s)], torch.full((n,), 19, dtype=torch.int64, device=dev))
    start = _Piece(tab[sec - lo_s - elapsed], torch.full((n,), 19, dtype=torch.int64, device=dev))

    r_port = rand64(seed, S_PORT, idx)
    r_port2 = rand64(seed, S_PORT2, idx)
    r_cc = rand64(seed, S_CC, idx)
    r_misc = rand64(seed, S_MISC, idx)

    def pick(words, k):     # an independent draw per vocabulary column
        return _vocab(words, _below(rand64(seed, S_MISC + 16 + k, idx), len(words)))
    r_pkt = rand64(seed, S_PKT, idx)
    nbytes = rec["bytes"]
    pk = 1 + (torch.div(nbytes, 900, rounding_mode="floor").clamp(max=1 << 40)) + _below(r_pkt, 3)
    sent = torch.div(nbytes, 5, rounding_mode="floor") * 2
    fields = [
        capture, gen, start, _decimal(elapsed, 4),
        _ipv4(rec["src"]), _decimal(_below(r_port, 65536), 5), _vocab(_CC, _below(r_cc, len(_CC))),
        _ipv4(rec["dst"]), _decimal(_below(r_port2, 1024) * (_below(r_port2 >> 10, 4) != 0), 5),
        pick(_CC, 0), pick(_PROTO, 1), pick(_APP, 2), pick(_SUBTYPE, 3), pick(_ACTION, 4), pick(_REASON, 5),
        _decimal(1 + _below(r_misc, 2), 1), pick(_CATEGORY, 6),
        _decimal(pk, 20), _decimal(torch.div(pk + 1, 2, rounding_mode="floor"), 20),
        _decimal(torch.div(pk, 2, rounding_mode="floor"), 20),
        _decimal(nbytes, 20), _decimal(sent.clamp(min=0), 20), _decimal((nbytes - sent).clamp(min=0), 20),
        pick(_DEVICE, 7),
    ]
    status = torch.zeros(n, dtype=torch.uint8, device=dev)
    if bad_per_million:
        bad = _below(rand64(seed, S_BAD, idx), 1_000_000) < bad_per_million
        kind = _below(rand64(seed, S_BADKIND, idx), 7)
        # 0: bytes "NA"              -> BYTES
        # 1: 23 fields (drop No. 24)  -> COLUMNS
        # 2: source octet 256         -> SRC
        # 3: destination "01" octet   -> DST
        # 4: month 13                 -> TIME
        # 5: line > 2047 bytes        -> LONG
        # 6: 25 fields                -> COLUMNS
        na = _vocab([b"NA"], torch.zeros(n, dtype=torch.int64, device=dev))
        k0 = bad & (kind == 0)
        fields[20] = _Piece(torch.where(k0.unsqueeze(1), torch.nn.functional.pad(na.chars, (0, 18)), fields[20].chars),
                            torch.where(k0, na.lens, fields[20].lens))
        k2 = bad & (kind == 2)
        f4 = fields[4].chars.clone()
        f4[k2, 0:3] = torch.tensor(list(b"256"), dtype=torch.uint8, device=dev)
        f4[k2, 3] = ord(".")
        fields[4] = _Piece(f4, torch.where(k2, torch.clamp(fields[4].lens, min=4), fields[4].lens))
        k3 = bad & (kind == 3)
        f7 = torch.nn.functional.pad(fields[7].chars, (1, 0))
        f7[:, 0] = ord("0")
        f7[~k3] = torch.nn.functional.pad(fields[7].chars, (0, 1))[~k3]
        fields[7] = _Piece(f7, fields[7].lens + k3.to(torch.int64))
        k4 = bad & (kind == 4)
        c = fields[0].chars.clone()
        c[k4, 5] = ord("1")
        c[k4, 6] = ord("3")
        fields[0] = _Piece(c, fields[0].lens)
        k5 = bad & (kind == 5)
        pad = torch.full((n, 2100), ord("x"), dtype=torch.uint8, device=dev)
        fields[23] = _Piece(torch.cat([fields[23].chars, pad], 1), fields[23].lens + k5.to(torch.int64) * 2100)
        k1 = bad & (kind == 1)
        k6 = bad & (kind == 6)
        status[k0] = BYTES
        status[k1 | k6] = COLUMNS
        status[k2] = SRC
        status[k3] = DST
        status[k4] = TIME
        status[k5] = LONG
        body = _concat(fields[:23], sep=ord(","))
        last = fields[23]
        # kind 1: the last field and its comma disappear; kind 6: an extra ",x" field
        extra = _vocab([b"", b",x"], k6.to(torch.int64))
        tail = _concat([_Piece(torch.full((n, 1), ord(","), dtype=torch.uint8, device=dev),
                               (~k1).to(torch.int64)),
                        _Piece(last.chars, torch.where(k1, torch.zeros_like(last.lens), last.lens)), extra])
        line = _concat([body, tail])
    else:
        line = _concat(fields, sep=ord(","))
    eol = _vocab([b"\r\n"] if crlf else [b"\n"], torch.zeros(n, dtype=torch.int64, device=dev))
    line = _concat([line, eol])
    # flatten the rows
    w = line.chars.shape[1]
    m = torch.arange(w, device=dev).unsqueeze(0) < line.lens.unsqueeze(1)
    return line.chars[m].contiguous(), status


def session_text_batched(wl: Workload, rec: dict, batch: int = 1 << 20, **kw):
    """session_text over record batches (bounded temporaries), concatenated."""
    n = rec["ts"].shape[0]
    texts, stats = [], []
    for lo in range(0, n, batch):
        sub = {k: v[lo:lo + batch] for k, v in rec.items()}
        t, s = session_text(wl, sub, salt=lo // batch, **kw)
        texts.append(t)
        stats.append(s)
    return torch.cat(texts), torch.cat(stats)
