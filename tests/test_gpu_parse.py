"""GPU parity of the NEXT-3 parser (sinet_parse_text through the C ABI) against the oracle's
parser (oracle_parse_text), element by element: line statuses, the compacted columns and the
counts, on generated PA-7080 text (Table 1) with injected malformed lines, fuzzed
lines, and the chunking edge cases of the kernel (48 KB chunks, 2 KB tail, look-back)."""
import random

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2106_12863_b200")
from oracle import core as oracle  # noqa: E402
from synth import WORKLOADS, records  # noqa: E402
from synth.sinet_text import session_text, session_text_batched  # noqa: E402

CHUNK = int(P._native.lib.sinet_parse_chunk_bytes())   # the kernel's chunk (look-back unit)


def gpu_parse(blob: bytes, tz=540, capacity=None):
    t = torch.frombuffer(bytearray(blob), dtype=torch.uint8).cuda() if blob else torch.empty(0, dtype=torch.uint8,
                                                                                              device="cuda")
    cols, st, info = P.parse_text(t, tz, capacity=capacity, status=True)
    torch.cuda.synchronize()
    return cols, st, info


def check_against_oracle(blob: bytes, tz=540):
    cols, st, info = gpu_parse(blob, tz)
    o = oracle.parse_text(blob, tz)
    assert info["lines"] == o.n_lines
    assert info["valid"] == o.n_valid
    assert np.array_equal(st.cpu().numpy(), o.status)
    assert np.array_equal(cols["ts"].cpu().numpy().view(np.uint64), o.ts)
    assert np.array_equal(cols["src"].cpu().numpy().view(np.uint32), o.src)
    assert np.array_equal(cols["dst"].cpu().numpy().view(np.uint32), o.dst)
    assert np.array_equal(cols["bytes"].cpu().numpy().view(np.uint64), o.bytes)
    assert info["by_status"] == np.bincount(o.status, minlength=7).tolist()
    bad = np.nonzero(o.status)[0]
    assert info["first_bad_line"] == (int(bad[0]) if len(bad) else (1 << 64) - 1)
    return info


def gen_text(n, bad=100_000, crlf=False, seed_off=0):
    wl = WORKLOADS["c1"].with_(n=n, seed=WORKLOADS["c1"].seed + seed_off)
    rec = records(wl, device="cuda")
    text, intended = session_text_batched(wl, rec, bad_per_million=bad, crlf=crlf)
    return bytes(text.cpu().numpy()), intended.cpu().numpy()


def test_generated_text_with_bad_lines():
    blob, intended = gen_text(200_003)
    info = check_against_oracle(blob)
    assert info["lines"] == len(intended) and info["by_status"][0] == int((intended == 0).sum())


def test_crlf_and_timezones():
    blob, _ = gen_text(20_000, crlf=True)
    for tz in (540, 0, -300):
        check_against_oracle(blob, tz)


def test_empty_and_tiny_texts():
    for blob in (b"", b"\n", b"\n\n", b"x", b"x\n", b"a,b\n,\n"):
        check_against_oracle(blob)


def test_many_tiny_lines_multi_round_chunks():
    # more lines in a chunk than one round parses: the count-then-rewrite path of the kernel
    rng = random.Random(3)
    good, _ = gen_text(50, bad=0)
    lines = good.split(b"\n")[:-1]
    parts = []
    for _ in range(60_000):
        parts.append(rng.choice(lines) if rng.random() < 0.05 else b"x" * rng.randrange(0, 40))
    check_against_oracle(b"\n".join(parts) + b"\n")
    check_against_oracle(b"\n" * (3 * CHUNK + 5))


def test_lines_across_chunk_boundaries_and_long_lines():
    good, _ = gen_text(2000, bad=0)
    lines = good.split(b"\n")[:-1]
    rng = random.Random(5)
    parts, pos = [], 0
    while pos < 6 * CHUNK:
        k = rng.random()
        if k < 0.1:      # pad a line's last field so that the line is 2046..2049 bytes long
            base = rng.choice(lines)
            want = rng.choice([2046, 2047, 2048, 2049, 2100])
            line = base + b"x" * max(0, want - len(base))
        elif k < 0.2:    # a newline exactly at the last byte of a chunk
            line = b"y" * ((CHUNK - (pos % CHUNK)) - 1)
        else:
            line = rng.choice(lines)
        parts.append(line)
        pos += len(line) + 1
    blob = b"\n".join(parts)
    for cut in (0, 1, 7, 15, 16):          # ragged text lengths, with and without a final newline
        check_against_oracle(blob[:len(blob) - cut])
        check_against_oracle(blob[:len(blob) - cut] + b"\n")


def test_unpacked_look_back():
    """Texts of 2 GiB or more scan lines and valid records in two look-back words per chunk
    (one packed word below that); the knob forces the two-word path on a small text."""
    from paper_2106_12863_b200 import _native as N
    assert N.lib.sinet_parse_set_knob(b"unpacked_look_back", 1) == 0
    try:
        blob, _ = gen_text(20_000, bad=50_000)
        check_against_oracle(blob)
        check_against_oracle(b"\n" * (3 * CHUNK + 5))
    finally:
        N.lib.sinet_parse_set_knob(b"unpacked_look_back", 0)


def test_fuzzed_lines():
    good, _ = gen_text(300, bad=0)
    lines = good.split(b"\n")[:-1]
    rng = random.Random(9)
    out = []
    for _ in range(30_000):
        b = bytearray(rng.choice(lines))
        for _ in range(rng.randrange(0, 3)):
            i = rng.randrange(len(b))
            op = rng.randrange(3)
            if op == 0:
                del b[i]
            elif op == 1:
                b.insert(i, rng.choice(b"0123456789,./: xN\r"))
            else:
                b[i] = rng.choice(b"0123456789,./: x")
        out.append(bytes(b))
    check_against_oracle(b"\n".join(out) + b"\n")


def test_capacity_overflow_is_reported():
    blob, intended = gen_text(5000, bad=0)
    with pytest.raises(P.SinetError) as e:
        gpu_parse(blob, capacity=100)
    assert "E_RANGE" in str(e.value)


def test_parse_then_histogram_equals_histogram_of_records():
    wl = WORKLOADS["c1"].with_(n=300_000)
    rec = records(wl, device="cuda")
    text, intended = session_text_batched(wl, rec, bad_per_million=0)
    cols, _, info = P.parse_text(text, 540)
    assert info["valid"] == wl.n
    nets, lens = __import__("synth").prefix_table(wl)
    out = []
    for c in (cols, rec):
        h = P.SinetHistogram(nets, lens, wl.window_start_ms, wl.window_ms)
        h.classify(c["ts"], c["src"], c["dst"], c["bytes"])
        h.reduce()
        out.append((h.read_bins(0, P.METRIC_COUNT), h.read_bins(1, P.METRIC_BYTES), h.read_totals()))
        h.close()
    for a, b in zip(*out):
        assert np.array_equal(a, b)


@pytest.mark.slow
def test_full_size_text_sample():
    """~1.4 GB of text (5 M lines) in one call, compared line by line with the oracle."""
    blob, _ = gen_text(5_000_000, bad=2000)
    check_against_oracle(blob)
