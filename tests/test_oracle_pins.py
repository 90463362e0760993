"""Pins of the CPU oracle (oracle/sinet_oracle.c) to things other than itself.

Each test names what fixes the expected value: a worked value of the paper's
operation, a brute-force bit-string comparison, Python's ipaddress library,
a Counter-based histogram, a closed form / invariant, or the generator's
construction-time ground truth.  No expected value comes from the CUDA path.
"""
import random

import numpy as np
import pytest

from oracle import brute
from oracle.core import LUT_ALG1, LUT_SRC_PRIORITY, LUT_STRICT
from synth import WORKLOADS, prefix_table, records
from synth.sinet_synth import to_numpy
from tests.helpers import dense_from_sparse, edge_addresses, ip, load_f0

M64 = (1 << 64) - 1


# ----------------------------------------------------------------------------- Alg. 1 l.6-7
def test_mask_is_leading_ones_bitstring(oracle_lib):
    # "translated to a 32-bit sequence": mask(Z) = Z ones then 32-Z zeros
    for z in range(33):
        assert oracle_lib.mask(z) == int("1" * z + "0" * (32 - z), 2)


def test_bitmask_worked_values(oracle_lib):
    # bitmask(192.168.1.7, 24) = 192.168.1.0 (the operation of Alg.1 l.6 P:L160)
    assert oracle_lib.bitmask(ip("192.168.1.7"), 24) == ip("192.168.1.0") == 3232235776
    # host bits of a CIDR are cleared by l.7: 192.168.1.77/24 -> 3232235776
    assert oracle_lib.bitmask(ip("192.168.1.77"), 24) == 3232235776
    assert oracle_lib.bitmask(ip("10.0.0.0"), 8) == 167772160
    rnd = random.Random(1)
    for _ in range(1000):
        a = rnd.getrandbits(32)
        assert oracle_lib.bitmask(a, 0) == 0            # /0 clears all bits
        assert oracle_lib.bitmask(a, 32) == a           # /32 is the identity
        z1 = rnd.randint(0, 32)
        z2 = rnd.randint(0, z1)
        # monotonicity bitmask(bitmask(a,z1),z2) == bitmask(a,z2) for z2 <= z1
        assert oracle_lib.bitmask(oracle_lib.bitmask(a, z1), z2) == oracle_lib.bitmask(a, z2)
        # bit-string truncation by hand
        s = format(a, "032b")
        assert oracle_lib.bitmask(a, z1) == int(s[:z1] + "0" * (32 - z1), 2)


# ----------------------------------------------------------------------------- Alg. 1 l.8-9
def test_member_worked_values(oracle_lib):
    nets, lens = [ip("192.168.1.0")], [24]
    assert oracle_lib.member(ip("192.168.1.7"), nets, lens)       # -> Outgoing
    assert not oracle_lib.member(ip("10.0.0.1"), nets, lens)      # -> Ingoing


def _random_case(rnd):
    p = rnd.randint(1, 6)
    nets, lens = [], []
    for _ in range(p):
        z = rnd.choice([0, 1, 31, 32, rnd.randint(0, 32), rnd.randint(8, 28)])
        nets.append(rnd.getrandbits(32))   # host bits deliberately left set (reading A9)
        lens.append(z)
    # bias the address to land near a table entry half the time
    if rnd.random() < 0.5:
        k = rnd.randrange(p)
        z = lens[k]
        a = (nets[k] & (int("1" * z + "0" * (32 - z), 2) if z else 0)) | (rnd.getrandbits(32) >> z if z < 32 else 0)
        a ^= rnd.choice([0, 0, 1 << rnd.randrange(32)])
    else:
        a = rnd.getrandbits(32)
    return a & 0xFFFFFFFF, nets, lens


def test_member_vs_bitstring_bruteforce(oracle_lib):
    # 10^5 random (ip, list) cases incl. Z in {0,1,31,32} vs 32-char bit-string prefixes
    rnd = random.Random(2106)
    for _ in range(100_000):
        a, nets, lens = _random_case(rnd)
        assert oracle_lib.member(a, nets, lens) == brute.member_bitstring(a, nets, lens)


def test_member_vs_ipaddress(oracle_lib):
    rnd = random.Random(12863)
    for _ in range(10_000):
        a, nets, lens = _random_case(rnd)
        assert oracle_lib.member(a, nets, lens) == brute.member_ipaddress(a, nets, lens)


def test_member_table_order_insensitive(oracle_lib):
    rnd = random.Random(7)
    for _ in range(2000):
        a, nets, lens = _random_case(rnd)
        perm = list(range(len(nets)))
        rnd.shuffle(perm)
        assert oracle_lib.member(a, nets, lens) == oracle_lib.member(
            a, [nets[i] for i in perm], [lens[i] for i in perm])


def test_member_bylen_vs_bitstring_bruteforce(oracle_lib):
    # the grouped-by-Z evaluation of the list (oracle_member_bylen_batch, used for the full-size
    # C5 digests) against the 32-char bit-string brute force on 2 x 10^4 random (ip, list) cases
    rnd = random.Random(4096)
    for _ in range(20_000):
        a, nets, lens = _random_case(rnd)
        got = oracle_lib.member_bylen(np.array([a], np.uint32), nets, lens)[0]
        assert got == brute.member_bitstring(a, nets, lens)


def test_member_bylen_equals_linear_scan_on_c5_table(oracle_lib):
    # C5's 4096-entry /8-/32 nested list: every interval edge +-1 and random addresses, both
    # evaluations of Alg. 1 l.4-9 (linear scan, grouped by Z) agree address by address
    nets, lens = prefix_table(WORKLOADS["c5"])
    rng = np.random.default_rng(5)
    ips = np.concatenate([edge_addresses(nets, lens), rng.integers(0, 1 << 32, 20_000, dtype=np.uint64).astype(np.uint32)])
    got = oracle_lib.member_bylen(ips, nets, lens, threads=4)
    want = np.array([oracle_lib.member(int(x), nets, lens) for x in ips], np.uint8)
    np.testing.assert_array_equal(got, want)
    assert 0 < int(got.sum()) < len(ips)


def test_histogram_members_equals_classify(oracle_lib):
    # memberships given per record, then the same post-discrimination steps: identical results
    wl = WORKLOADS["c1"].with_(n=50_000)
    nets, lens = prefix_table(wl)
    ts, src, dst, nb = to_numpy(records(wl))[:4]
    a = oracle_lib.classify_histogram(ts, src, dst, nb, nets, lens, wl.window_start_ms, wl.window_ms, 1)
    b = oracle_lib.histogram_members(ts, oracle_lib.member_bylen(src, nets, lens), oracle_lib.member_bylen(dst, nets, lens),
                                     nb, wl.window_start_ms, wl.window_ms, 1)
    np.testing.assert_array_equal(a.count, b.count)
    np.testing.assert_array_equal(a.bytes, b.bytes)
    np.testing.assert_array_equal(a.totals, b.totals)


# ----------------------------------------------------------------------------- worked fixture
@pytest.mark.parametrize("case", ["src_priority_w1", "alg1_w1", "strict_w1", "src_priority_w5"])
def test_f0_golden(oracle_lib, case):
    g, nets, lens, ts, src, dst, nb = load_f0()
    e = g["expected"][case]
    w = e["width"]
    res = oracle_lib.classify_histogram(ts, src, dst, nb, nets, lens, g["window_start_ms"],
                                        g["window_ms"], w, lut=tuple(e["lut"]))
    nbins = g["window_ms"] // w
    for d, key in ((0, "out"), (1, "in")):
        c, b = dense_from_sparse(e[key], nbins)
        np.testing.assert_array_equal(res.count[d], c)
        np.testing.assert_array_equal(res.bytes[d], b)
    assert res.m_count.tolist() == e["m_count"]
    assert res.m_bytes.tolist() == e["m_bytes"]
    assert res.oow_count.tolist() == e["oow_count"]
    assert res.oow_bytes.tolist() == e["oow_bytes"]
    assert int(res.m_bytes.sum()) == g["sum_bytes"]


def test_f0_tags(oracle_lib):
    g, nets, lens, ts, src, dst, nb = load_f0()
    t = oracle_lib.tags(ts, src, dst, nets, lens, g["window_start_ms"], g["window_ms"])
    cells = g["expected_cells"]
    for r, (s_in, d_in) in enumerate(cells):
        assert t[r] & 3 == s_in | (d_in << 1)
    assert [(int(x) >> 2) & 1 for x in t] == [0, 0, 0, 0, 0, 0, 1, 1, 0, 0]


# ----------------------------------------------------------------------------- map (§4.1)
def test_map_key_worked_values(oracle_lib):
    # capture_time 86399999 at width 3600000 -> key 82800000, i.e. hour bin 23
    nets, lens = np.array([0], np.uint32), np.array([0], np.uint8)   # /0: every source inside -> OUT
    one = lambda t, b: (np.array([t], np.uint64), np.array([1], np.uint32), np.array([2], np.uint32),
                        np.array([b], np.uint64))
    res = oracle_lib.classify_histogram(*one(86399999, 700), nets, lens, 0, 86_400_000, 3_600_000)
    assert res.count[0].tolist() == [0] * 23 + [1] and res.bytes[0][23] == 700
    # (0,(1,10)) and (999,(1,20)) at width 1000 -> [(0,(2,30))]
    ts = np.array([0, 999], np.uint64)
    res = oracle_lib.classify_histogram(ts, np.ones(2, np.uint32), np.ones(2, np.uint32),
                                        np.array([10, 20], np.uint64), nets, lens, 0, 2000, 1000)
    assert res.count[0].tolist() == [2, 0] and res.bytes[0].tolist() == [30, 0]


def test_empty_and_singleton(oracle_lib):
    nets, lens = prefix_table(WORKLOADS["c1"])
    e = np.zeros(0, np.uint64)
    res = oracle_lib.classify_histogram(e, e.astype(np.uint32), e.astype(np.uint32), e, nets, lens,
                                        1000, 100, 1)
    assert not res.count.any() and not res.bytes.any() and not res.totals.any()
    t = np.array([1042], np.uint64)
    res = oracle_lib.classify_histogram(t, np.array([nets[0]], np.uint32), np.array([ip("200.1.1.1")], np.uint32),
                                        np.array([5], np.uint64), nets, lens, 1000, 100, 1)
    assert res.count.sum() == 1 and res.count[0][42] == 1 and res.bytes[0][42] == 5


def test_u64_bytes_wrap_modulo(oracle_lib):
    # reading A18: u64 modular addition (closed form: (3 * (2^64 - 5)) mod 2^64)
    nets, lens = np.array([0], np.uint32), np.array([0], np.uint8)
    v = (1 << 64) - 5
    ts = np.array([7, 7, 7], np.uint64)
    res = oracle_lib.classify_histogram(ts, np.ones(3, np.uint32), np.ones(3, np.uint32),
                                        np.array([v] * 3, np.uint64), nets, lens, 0, 10, 1)
    assert int(res.bytes[0][7]) == (3 * v) & M64 and res.count[0][7] == 3


# ----------------------------------------------------------------------------- Counter oracle
def _adversarial_records(n, nets, lens, start, window, seed):
    rng = np.random.default_rng(seed)
    edges = edge_addresses(nets, lens)
    pick = lambda: np.where(rng.random(n) < 0.5, rng.choice(edges, n),
                            rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32))
    src, dst = pick(), pick()
    ts = (start + rng.integers(-50, window + 50, n)).astype(np.uint64)
    nb = rng.integers(0, 1 << 40, n, dtype=np.uint64)
    nb[rng.random(n) < 0.01] = rng.integers(1 << 63, (1 << 64) - 1, dtype=np.uint64, size=1)[0]
    return ts, src.astype(np.uint32), dst.astype(np.uint32), nb


@pytest.mark.parametrize("lut", [LUT_SRC_PRIORITY, LUT_ALG1, LUT_STRICT])
@pytest.mark.parametrize("width", [1, 7])
def test_oracle_vs_counter(oracle_lib, lut, width):
    nets, lens = prefix_table(WORKLOADS["c1"])
    start, window = 1_613_660_400_000, 7_000
    ts, src, dst, nb = _adversarial_records(20_000, nets, lens, start, window, seed=width * 10 + lut[0])
    res = oracle_lib.classify_histogram(ts, src, dst, nb, nets, lens, start, window, width, lut=lut)
    cnt, byt, mc, mb, oc, ob = brute.histogram_counter(ts, src, dst, nb, nets.tolist(), lens.tolist(),
                                                       start, window, width, lut)
    for d in (0, 1):
        exp_c = np.zeros(window // width, np.uint64)
        exp_b = np.zeros(window // width, np.uint64)
        for (dd, k), v in cnt.items():
            if dd == d:
                exp_c[k] = v
        for (dd, k), v in byt.items():
            if dd == d:
                exp_b[k] = v
        np.testing.assert_array_equal(res.count[d], exp_c)
        np.testing.assert_array_equal(res.bytes[d], exp_b)
    assert res.m_count.tolist() == mc and res.m_bytes.tolist() == mb
    assert res.oow_count.tolist() == oc and res.oow_bytes.tolist() == ob


# ----------------------------------------------------------------------------- invariants
def _c1_small(n=200_000, **kw):
    wl = WORKLOADS["c1"].with_(n=n, **kw)
    nets, lens = prefix_table(wl)
    rec = records(wl)
    return wl, nets, lens, rec


def _run(oracle_lib, wl, nets, lens, cols, lut=LUT_SRC_PRIORITY, threads=1, into=None):
    return oracle_lib.classify_histogram(*cols, nets, lens, wl.window_start_ms, wl.window_ms,
                                         wl.bin_width_ms, lut=lut, threads=threads, into=into)


def test_generator_ground_truth(oracle_lib):
    # the generator's intended (s_in, d_in) per record is correct by construction (synth docstring)
    wl, nets, lens, rec = _c1_small()
    cols = to_numpy(rec)
    res = _run(oracle_lib, wl, nets, lens, cols)
    intended = np.bincount(rec["cls"].numpy(), minlength=4)
    assert res.m_count.tolist() == intended.tolist()
    t = oracle_lib.tags(cols[0], cols[1], cols[2], nets, lens, wl.window_start_ms, wl.window_ms)
    np.testing.assert_array_equal(t & 3, (rec["cls"].numpy() >> 1) | ((rec["cls"].numpy() & 1) << 1))


@pytest.mark.parametrize("lut", [LUT_SRC_PRIORITY, LUT_ALG1, LUT_STRICT])
def test_conservation(oracle_lib, lut):
    wl, nets, lens, rec = _c1_small()
    cols = to_numpy(rec)
    res = _run(oracle_lib, wl, nets, lens, cols, lut=lut)
    assert int(res.m_count.sum()) == wl.n
    assert int(res.m_bytes.sum()) == int(cols[3].astype(object).sum()) & M64
    for d in (0, 1):
        cells = [k for k in range(4) if lut[k] == d]
        assert int(res.count[d].sum()) + int(res.oow_count[d]) == sum(int(res.m_count[k]) for k in cells)
        assert (int(res.bytes[d].astype(object).sum()) + int(res.oow_bytes[d])) & M64 == \
            sum(int(res.m_bytes[k]) for k in cells) & M64


def test_preset_relations(oracle_lib):
    wl, nets, lens, rec = _c1_small()
    cols = to_numpy(rec)
    sp = _run(oracle_lib, wl, nets, lens, cols, LUT_SRC_PRIORITY)
    a1 = _run(oracle_lib, wl, nets, lens, cols, LUT_ALG1)
    st = _run(oracle_lib, wl, nets, lens, cols, LUT_STRICT)
    np.testing.assert_array_equal(a1.count[0], sp.count[0])   # OUT identical (A1)
    np.testing.assert_array_equal(st.count[1], sp.count[1])   # IN identical
    assert int(a1.count[1].sum() + a1.oow_count[1]) == int(sp.count[1].sum() + sp.oow_count[1]) + int(sp.m_count[0])
    assert int(sp.count[0].sum() + sp.oow_count[0]) == int(st.count[0].sum() + st.oow_count[0]) + int(sp.m_count[3])


def test_all_sources_inside_gives_empty_in(oracle_lib):
    # every source inside -> ingoing series empty
    wl, nets, lens, rec = _c1_small(50_000)
    ts, src, dst, nb = to_numpy(rec)
    src = np.full_like(src, nets[0])
    res = _run(oracle_lib, wl, nets, lens, (ts, src, dst, nb))
    assert not res.count[1].any() and res.count[0].sum() + res.oow_count[0] == wl.n


def test_permutation_chunk_and_thread_invariance(oracle_lib):
    wl, nets, lens, rec = _c1_small()
    cols = to_numpy(rec)
    ref = _run(oracle_lib, wl, nets, lens, cols)
    perm = np.random.default_rng(3).permutation(wl.n)
    shuf = _run(oracle_lib, wl, nets, lens, tuple(c[perm] for c in cols))
    chunked = None
    for lo, hi in ((0, 1), (1, 777), (777, 100_000), (100_000, wl.n)):
        chunked = _run(oracle_lib, wl, nets, lens, tuple(c[lo:hi] for c in cols), into=chunked)
    mt = _run(oracle_lib, wl, nets, lens, cols, threads=5)
    for other in (shuf, chunked, mt):
        np.testing.assert_array_equal(other.count, ref.count)
        np.testing.assert_array_equal(other.bytes, ref.bytes)
        np.testing.assert_array_equal(other.totals, ref.totals)


def test_shuffled_generator_same_multiset(oracle_lib):
    wl, nets, lens, rec = _c1_small(100_000)
    ref = _run(oracle_lib, wl, nets, lens, to_numpy(rec))
    rs = records(wl.with_(order="shuffled"))
    sh = _run(oracle_lib, wl, nets, lens, to_numpy(rs))
    np.testing.assert_array_equal(sh.count, ref.count)
    np.testing.assert_array_equal(sh.bytes, ref.bytes)


# ----------------------------------------------------------------------------- NEXT-1 rebin / sparse
def test_rebin_worked_values_and_conservation(oracle_lib):
    # (0,(1,10)) and (999,(1,20)) rebinned to 1000 ms -> [(0,(2,30))]
    fine_c = np.zeros(2000, np.uint64)
    fine_b = np.zeros(2000, np.uint64)
    fine_c[[0, 999]] = 1
    fine_b[[0, 999]] = [10, 20]
    assert oracle_lib.rebin(fine_c, 1000).tolist() == [2, 0]
    assert oracle_lib.rebin(fine_b, 1000).tolist() == [30, 0]
    # 1 ms -> 10 min -> 1 h conserves totals and equals direct 1 h binning (S:L470 criterion 4)
    wl, nets, lens, rec = _c1_small(100_000)
    cols = to_numpy(rec)
    fine = _run(oracle_lib, wl, nets, lens, cols)
    hourly = oracle_lib.classify_histogram(*cols, nets, lens, wl.window_start_ms, wl.window_ms, 3_600_000)
    for d in (0, 1):
        ten = oracle_lib.rebin(fine.count[d], 600_000)
        assert int(ten.sum()) == int(fine.count[d].sum())
        np.testing.assert_array_equal(oracle_lib.rebin(ten, 6), hourly.count[d])
        np.testing.assert_array_equal(oracle_lib.rebin(fine.bytes[d], 3_600_000), hourly.bytes[d])
    # partial last coarse bin, and u64 wrap
    v = np.array([(1 << 64) - 1, 2, 5], np.uint64)
    assert oracle_lib.rebin(v, 2).tolist() == [1, 5]


def test_sparse_export_matches_definition(oracle_lib):
    c = np.array([0, 3, 0, 0, 1, 0], np.uint64)
    b = np.array([0, 30, 0, 0, 0, 0], np.uint64)
    t, cc, bb = oracle_lib.sparse(c, b, 1000, 5)
    assert t.tolist() == [1005, 1020] and cc.tolist() == [3, 1] and bb.tolist() == [30, 0]
    wl, nets, lens, rec = _c1_small(50_000)
    res = _run(oracle_lib, wl, nets, lens, to_numpy(rec))
    t, cc, bb = oracle_lib.sparse(res.count[0], res.bytes[0], wl.window_start_ms, 1)
    # sparse bound and conservation
    assert len(t) <= min(wl.n, wl.nbins) and int(cc.sum()) == int(res.count[0].sum())
    assert np.all(np.diff(t.astype(np.int64)) > 0)


# ----------------------------------------------------------------------------- NEXT-2 watchlist
def test_watch_filter_worked_values(oracle_lib):
    # empty list -> empty output; destination listed, source not -> retained
    src = np.array([ip("1.2.3.4"), ip("5.6.7.8"), ip("9.9.9.9")], np.uint32)
    dst = np.array([ip("8.8.8.8"), ip("1.2.3.4"), ip("7.7.7.7")], np.uint32)
    assert oracle_lib.watch_filter(src, dst, []).tolist() == []
    assert oracle_lib.watch_filter(src, dst, [ip("1.2.3.4")]).tolist() == [0, 1]
    assert oracle_lib.watch_filter(src, dst, [ip("7.7.7.7"), ip("7.7.7.7")]).tolist() == [2]   # set semantics


def test_watch_filter_vs_python_set_and_properties(oracle_lib):
    # 1000 synthetic records, exactly 10 touching listed IPs -> 10 kept; union
    # superset and idempotence; filter-then-histogram conservation
    rng = np.random.default_rng(877)
    listed = rng.choice(np.arange(200, 2_000_000, dtype=np.uint32), 877, replace=False)
    src = rng.integers(3_000_000, 1 << 32, 1000, dtype=np.uint64).astype(np.uint32)
    dst = rng.integers(3_000_000, 1 << 32, 1000, dtype=np.uint64).astype(np.uint32)
    hit = rng.choice(1000, 10, replace=False)
    for k, r in enumerate(hit):
        (src if k % 2 else dst)[r] = listed[k]
    keep = oracle_lib.watch_filter(src, dst, listed)
    assert sorted(keep.tolist()) == sorted(hit.tolist())
    lset = set(int(x) for x in listed[:400])
    ref = [i for i in range(1000) if int(src[i]) in lset or int(dst[i]) in lset]
    assert oracle_lib.watch_filter(src, dst, listed[:400]).tolist() == ref
    a = set(oracle_lib.watch_filter(src, dst, listed[:300]).tolist())
    assert a <= set(keep.tolist())
    k2 = oracle_lib.watch_filter(src[keep], dst[keep], listed)
    assert k2.tolist() == list(range(len(keep)))


def test_watched_histogram_equals_histogram_of_filtered(oracle_lib):
    wl, nets, lens, rec = _c1_small(100_000)
    ts, src, dst, nb = to_numpy(rec)
    listed = np.unique(np.concatenate([src[:150], dst[1000:1150]]))
    res = oracle_lib.classify_histogram_watched(ts, src, dst, nb, nets, lens, listed, wl.window_start_ms,
                                                wl.window_ms, 1)
    lset = set(int(x) for x in listed)
    m = np.array([int(s) in lset or int(d) in lset for s, d in zip(src, dst)])
    ref = oracle_lib.classify_histogram(ts[m], src[m], dst[m], nb[m], nets, lens, wl.window_start_ms,
                                        wl.window_ms, 1)
    np.testing.assert_array_equal(res.count, ref.count)
    np.testing.assert_array_equal(res.totals, ref.totals)
    assert int(res.m_count.sum()) == int(m.sum())


# ----------------------------------------------------------------------------- NEXT-4 labelled LPM
def test_lpm_worked_values_and_bruteforce(oracle_lib):
    nets = [ip("133.0.0.0"), ip("133.11.0.0"), ip("133.11.7.0"), ip("133.11.7.128")]
    lens = [8, 16, 24, 25]
    labs = [1, 0, 1, 0]          # 133/8 in, carve out 133.11/16, re-include 133.11.7/24, carve .128/25
    cases = {"133.1.2.3": 1, "133.11.2.3": 0, "133.11.7.5": 1, "133.11.7.200": 0, "8.8.8.8": 0}
    got = oracle_lib.member_lpm([ip(k) for k in cases], nets, lens, labs)
    assert got.tolist() == list(cases.values())
    # all labels 1 -> plain match-any membership (Alg. 1 over the list)
    rnd = random.Random(26)
    for _ in range(3000):
        a, n2, l2 = _random_case(rnd)
        lab = [rnd.randint(0, 1) for _ in n2]
        assert oracle_lib.member_lpm([a], n2, l2, [1] * len(n2))[0] == oracle_lib.member(a, n2, l2)
        assert bool(oracle_lib.member_lpm([a], n2, l2, lab)[0]) == brute.member_lpm_bitstring(a, n2, l2, lab)


def test_histogram_members_equals_histogram_when_all_inside(oracle_lib):
    # with every label 1 the LPM histogram is the plain histogram (same definition, given memberships)
    wl, nets, lens, rec = _c1_small(60_000)
    cols = to_numpy(rec)
    a = _run(oracle_lib, wl, nets, lens, cols)
    b = oracle_lib.classify_histogram_lpm(*cols, nets, lens, np.ones(len(nets), np.uint8), wl.window_start_ms,
                                          wl.window_ms, 1)
    np.testing.assert_array_equal(a.count, b.count)
    np.testing.assert_array_equal(a.bytes, b.bytes)
    np.testing.assert_array_equal(a.totals, b.totals)
