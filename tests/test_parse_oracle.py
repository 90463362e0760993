"""Pins of the NEXT-3 text parser of the oracle (oracle_parse_text in oracle/sinet_oracle.c).

Expected values come from: Table 1's printed sample (tests/golden/table1_sample.json),
Python's own libraries (datetime / calendar.timegm for the calendar, ipaddress for dotted
quads, int() for decimals), the independent Python parser oracle/brute.parse_text_python,
and the generator's construction-time ground truth (synth/sinet_text.py renders dates with
datetime.strftime and records which lines it corrupted, and how).
"""
import calendar
import datetime
import ipaddress
import json
import os
import random

import numpy as np
import pytest

from oracle import brute
from oracle.core import (PARSE_BYTES, PARSE_COLUMNS, PARSE_DST, PARSE_LONG, PARSE_OK, PARSE_SRC, PARSE_TIME,
                         parse_line, parse_text)
from synth import WORKLOADS, records
from synth.sinet_synth import to_numpy
from synth.sinet_text import session_text
from tests.helpers import GOLDEN

M64 = (1 << 64) - 1


def table1_fields():
    with open(os.path.join(GOLDEN, "table1_sample.json")) as f:
        g = json.load(f)
    assert len(g["items"]) == len(g["values"]) == 24
    return [v.encode() for v in g["values"]]


def line_of(fields):
    return b",".join(fields)


def epoch_ms(y, mo, d, h=0, mi=0, s=0, ms=0, tz_min=0):
    return calendar.timegm(datetime.datetime(y, mo, d, h, mi, s).timetuple()) * 1000 + ms - tz_min * 60000


def test_table1_sample_as_printed_is_rejected_at_the_masked_source():
    # the paper masks the addresses ("xxx.xxx.xxx.xxx"): not a dotted quad -> SRC
    st, *_ = parse_line(line_of(table1_fields()))
    assert st == PARSE_SRC


def test_table1_sample_with_addresses():
    f = table1_fields()
    f[4], f[7] = b"192.168.1.7", b"10.0.0.1"      # S:L196 / S:L206 worked addresses
    st, ts, src, dst, nb = parse_line(line_of(f))
    assert st == PARSE_OK
    assert ts == epoch_ms(2018, 1, 1)              # calendar.timegm: 1514764800 s
    assert ts == 1514764800000
    assert src == int(ipaddress.IPv4Address("192.168.1.7")) == 3232235783
    assert dst == int(ipaddress.IPv4Address("10.0.0.1"))
    assert nb == 0                                  # Table 1 No. 21 sample value
    # JST logs: the same text is 9 h earlier in UTC
    assert parse_line(line_of(f), 540)[1] == 1514764800000 - 9 * 3600 * 1000


def _with(field_no, value, base=None):
    f = list(base or table1_fields())
    f[4], f[7] = b"1.2.3.4", b"5.6.7.8"
    f[field_no - 1] = value                         # Table 1 numbering is 1-based
    return line_of(f)


@pytest.mark.parametrize("text,ok", [
    (b"2020/02/29 12:34:56.789", True), (b"2021/02/29 00:00:00.000", False), (b"2000/02/29 00:00:00.000", True),
    (b"2100/02/29 00:00:00.000", False), (b"1969/12/31 23:59:59.999", False), (b"1970/01/01 00:00:00.000", True),
    (b"2021/02/19 24:00:00.000", False), (b"2021/02/19 23:60:00.000", False), (b"2021/02/19 23:59:60.000", False),
    (b"2021/02/19 23:59:59.999", True), (b"2021/02/19 23:59:59", False), (b"2021-02-19 00:00:00.000", False),
    (b"2021/13/01 00:00:00.000", False), (b"2021/00/01 00:00:00.000", False), (b"2021/04/31 00:00:00.000", False),
    (b"2021/02/19 00:00:00.0000", False), (b"2021/2/19 00:00:00.000", False), (b"9999/12/31 23:59:59.999", True),
    (b"2021/02/19T00:00:00.000", False), (b"NA", False), (b"", False),
])
def test_capture_time_against_datetime(text, ok):
    st, ts, *_ = parse_line(_with(1, text))
    assert st == (PARSE_OK if ok else PARSE_TIME)
    if ok:
        d, t = text.decode().split(" ")
        y, mo, dd = (int(x) for x in d.split("/"))
        hms, ms = t.split(".")
        h, mi, s = (int(x) for x in hms.split(":"))
        assert ts == epoch_ms(y, mo, dd, h, mi, s, int(ms))


def test_capture_time_random_days_against_timegm():
    rng = random.Random(7)
    for _ in range(3000):
        dt = datetime.datetime(1970, 1, 1) + datetime.timedelta(milliseconds=rng.randrange(0, 253402300799999))
        text = dt.strftime("%Y/%m/%d %H:%M:%S").encode() + b".%03d" % (dt.microsecond // 1000)
        tz = rng.choice([0, 540, -300, 330, 1440, -1440])
        st, ts, *_ = parse_line(_with(1, text), tz)
        want = calendar.timegm(dt.timetuple()) * 1000 + dt.microsecond // 1000 - tz * 60000
        if want < 0:
            assert st == PARSE_TIME
        else:
            assert (st, ts) == (PARSE_OK, want)


@pytest.mark.parametrize("text", [b"1.2.3.4", b"0.0.0.0", b"255.255.255.255", b"192.168.1.7", b"10.0.0.1",
                                  b"256.1.1.1", b"1.2.3", b"1.2.3.4.5", b"01.2.3.4", b"1.2.3.04", b"1..3.4",
                                  b" 1.2.3.4", b"1.2.3.4 ", b"+1.2.3.4", b"1.2.3.-4", b"xxx.xxx.xxx.xxx", b"",
                                  b"1.2.3.4/32", b"::1", b"1.2.3.1000", b"0x1.2.3.4"])
def test_dotted_quad_against_ipaddress(text):
    try:
        want = int(ipaddress.IPv4Address(text.decode()))
    except ValueError:
        want = None
    for field_no, code, k in ((5, PARSE_SRC, 2), (8, PARSE_DST, 3)):
        st, _, src, dst, _ = parse_line(_with(field_no, text))
        if want is None:
            assert st == code
        else:
            assert st == PARSE_OK and (src, dst)[k - 2] == want


@pytest.mark.parametrize("text,want", [
    (b"0", 0), (b"7", 7), (b"007", 7), (str(M64).encode(), M64), (str(M64 + 1).encode(), None),
    (b"99999999999999999999", None), (b"4294967301", 4294967301), (b"NA", None), (b"", None), (b"-1", None),
    (b"1e3", None), (b" 1", None), (b"000000000000000000001", None), (b"18446744073709551610", 18446744073709551610),
])
def test_bytes_against_int(text, want):
    st, *_, nb = parse_line(_with(21, text))
    if want is None:
        assert st == PARSE_BYTES
    else:
        assert (st, nb) == (PARSE_OK, want) and want == int(text)


def test_columns_long_and_priority():
    good = _with(1, b"2018/01/01 00:00:00.000")
    assert parse_line(good)[0] == PARSE_OK
    assert parse_line(good + b",extra")[0] == PARSE_COLUMNS
    assert parse_line(good.rsplit(b",", 1)[0])[0] == PARSE_COLUMNS
    assert parse_line(b"")[0] == PARSE_COLUMNS
    assert parse_line(good + b"\r")[0] == PARSE_OK                       # CRLF line
    pad = 2047 - len(good)
    exact = good[:-2] + b"x" * pad + good[-2:]                          # content of exactly 2047 bytes
    assert len(exact) == 2047 and parse_line(exact)[0] == PARSE_OK
    assert parse_line(exact[:-2] + b"xNA")[0] == PARSE_LONG              # 2048 bytes
    assert parse_line(exact + b"\r")[0] == PARSE_LONG                    # the limit counts the '\r'
    # the first failing check wins: TIME before SRC before DST before BYTES
    f = list(table1_fields())
    assert parse_line(line_of(f))[0] == PARSE_SRC
    f[0] = b"bad"
    assert parse_line(line_of(f))[0] == PARSE_TIME
    f = list(table1_fields())
    f[4], f[20] = b"1.2.3.4", b"NA"
    assert parse_line(line_of(f))[0] == PARSE_DST


def test_line_splitting():
    good = _with(1, b"2018/01/01 00:00:00.000")
    assert parse_text(b"").n_lines == 0
    assert list(parse_text(b"\n").status) == [PARSE_COLUMNS]
    assert list(parse_text(good).status) == [PARSE_OK]                   # no final newline
    assert list(parse_text(good + b"\n").status) == [PARSE_OK]
    r = parse_text(good + b"\n\n" + good + b"\r\n")
    assert list(r.status) == [PARSE_OK, PARSE_COLUMNS, PARSE_OK] and r.n_valid == 2


def _mutate(rng, line: bytes) -> bytes:
    b = bytearray(line)
    for _ in range(rng.randrange(1, 4)):
        op = rng.randrange(4)
        i = rng.randrange(len(b) + 1)
        if op == 0 and b:
            del b[min(i, len(b) - 1)]
        elif op == 1:
            b.insert(i, rng.choice(b"0123456789,./: xN\r"))
        elif op == 2 and b:
            b[min(i, len(b) - 1)] = rng.choice(b"0123456789,./: x")
        else:
            b[i:i] = b"9"
    return bytes(b).replace(b"\n", b"")


def test_generated_text_against_ground_truth_and_python_parser():
    wl = WORKLOADS["c1"].with_(n=3000)
    rec = records(wl)
    text, intended = session_text(wl, rec, bad_per_million=150_000)
    tb = bytes(text.numpy())
    r = parse_text(tb, 540)
    assert np.array_equal(r.status, intended.numpy())                    # construction-time ground truth
    ok = intended.numpy() == PARSE_OK
    for col, got in zip(to_numpy(rec), (r.ts, r.src, r.dst, r.bytes)):
        assert np.array_equal(col[ok], got)
    py = brute.parse_text_python(tb, 540)
    assert [p[0] for p in py] == list(r.status)


def test_fuzzed_lines_against_python_parser():
    wl = WORKLOADS["c1"].with_(n=400)
    text, _ = session_text(wl, records(wl))
    lines = bytes(text.numpy()).split(b"\n")[:-1]
    rng = random.Random(11)
    fuzz = [_mutate(rng, rng.choice(lines)) for _ in range(4000)]
    blob = b"\n".join(fuzz) + b"\n"
    r = parse_text(blob, 540)
    py = brute.parse_text_python(blob, 540)
    assert [p[0] for p in py] == list(r.status)
    okp = [p for p in py if p[0] == PARSE_OK]
    assert [p[1] for p in okp] == list(r.ts) and [p[4] for p in okp] == list(r.bytes)
    assert [p[2] for p in okp] == list(r.src) and [p[3] for p in okp] == list(r.dst)
    assert 0 < r.n_valid < r.n_lines
