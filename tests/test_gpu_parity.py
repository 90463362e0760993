"""GPU parity: libsinet (through its C ABI) vs the CPU oracle, bit-exact.

All arithmetic on the path is integer, so the bar is exact equality of every
bin, every total and every tag.
"""
import numpy as np
import pytest
import torch

from oracle.core import LUT_ALG1, LUT_SRC_PRIORITY, LUT_STRICT
from synth import WORKLOADS, prefix_table, records
from synth.sinet_synth import to_numpy
from tests.helpers import edge_addresses, load_f0

pytestmark = pytest.mark.gpu

ORDERS = None


@pytest.fixture(scope="module")
def S():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_12863_b200 as S
    return S


def dev_cols(cols, device="cuda"):
    ts, src, dst, nb = cols
    return (torch.from_numpy(np.ascontiguousarray(ts).view(np.int64)).to(device),
            torch.from_numpy(np.ascontiguousarray(src).view(np.int32)).to(device),
            torch.from_numpy(np.ascontiguousarray(dst).view(np.int32)).to(device),
            torch.from_numpy(np.ascontiguousarray(nb).view(np.int64)).to(device))


def gpu_run(S, nets, lens, cols, start, window, width=1, lut=LUT_SRC_PRIORITY, order=0, chunks=None,
            tags=False, groups=0, agg=-1, tab=-1, scratch=None):
    """groups: 0 automatic kernel/layout, 1 / 2 = k_hist_stream with one / two rings per CTA,
    "ws" = the warp-specialised k_hist_ws (stream kernels; order 2 takes k_hist_atomic)."""
    h = S.SinetHistogram(nets, lens, start, window, width, lut=lut, order=order)
    if groups == "ws":
        h.set_knob("stream_kernel", 2)
        groups = 0
    elif groups in (1, 2):
        h.set_knob("stream_kernel", 1)
    h.set_tuning(groups, agg)
    h.set_table_mode(tab)
    if scratch:   # unordered batches: partition then bin, sub-batches of `scratch` records
        h.set_scratch(scratch)
    d = dev_cols(cols)
    n = d[0].numel()
    tg = torch.full((max(n, 4),), 0xEE, dtype=torch.uint8, device="cuda") if tags else None
    if chunks is None:
        h.classify(*d, tags=tg)
    else:
        for lo, hi in chunks:
            h.classify(*(c[lo:hi] for c in d), tags=None if tg is None else tg[lo:hi])
    out = {"count": np.stack([h.read_bins(k, S.METRIC_COUNT) for k in (0, 1)]),
           "bytes": np.stack([h.read_bins(k, S.METRIC_BYTES) for k in (0, 1)]),
           "totals": h.read_totals(), "h": h}
    if tags:
        out["tags"] = tg[:n].cpu().numpy()
    return out


def assert_parity(g, o):
    np.testing.assert_array_equal(g["count"], o.count)
    np.testing.assert_array_equal(g["bytes"], o.bytes)
    np.testing.assert_array_equal(g["totals"], o.totals)


@pytest.mark.parametrize("case", ["src_priority_w1", "alg1_w1", "strict_w1", "src_priority_w5"])
def test_f0_golden_on_gpu(S, oracle_lib, case):
    g, nets, lens, ts, src, dst, nb = load_f0()
    e = g["expected"][case]
    cols = (ts, src, dst, nb)
    res = gpu_run(S, nets, lens, cols, g["window_start_ms"], g["window_ms"], e["width"], tuple(e["lut"]),
                  tags=True)
    o = oracle_lib.classify_histogram(*cols, nets, lens, g["window_start_ms"], g["window_ms"], e["width"],
                                      lut=tuple(e["lut"]))
    assert_parity(res, o)
    np.testing.assert_array_equal(res["tags"], oracle_lib.tags(ts, src, dst, nets, lens, g["window_start_ms"],
                                                               g["window_ms"]))


def _adversarial(n, nets, lens, start, window, seed):
    rng = np.random.default_rng(seed)
    edges = edge_addresses(nets, lens)
    pick = lambda: np.where(rng.random(n) < 0.4, rng.choice(edges, n),
                            rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)).astype(np.uint32)
    ts = (start + rng.integers(-300, window + 300, n)).astype(np.uint64)
    nb = rng.integers(0, 1 << 40, n, dtype=np.uint64)
    big = rng.random(n) < 0.02
    nb[big] = rng.integers(1 << 62, 1 << 63, int(big.sum()), dtype=np.uint64) * np.uint64(2)
    return ts, pick(), pick(), nb


@pytest.mark.parametrize("order,groups", [(1, 1), (1, 2), (1, "ws"), (2, 0)])
@pytest.mark.parametrize("lut", [LUT_SRC_PRIORITY, LUT_ALG1, LUT_STRICT])
@pytest.mark.parametrize("width", [1, 3, 1000])
def test_adversarial_parity(S, oracle_lib, lut, width, order, groups):
    nets, lens = prefix_table(WORKLOADS["c1"])
    start, window = 1_613_660_400_000, 3_000_000
    for n in (1, 5, 127, 129, 40_001):   # ragged tails around the 4-record / 128-record groups
        cols = _adversarial(n, nets, lens, start, window, seed=n + width)
        g = gpu_run(S, nets, lens, cols, start, window, width, lut, order=order, tags=True, groups=groups)
        o = oracle_lib.classify_histogram(*cols, nets, lens, start, window, width, lut=lut)
        assert_parity(g, o)
        np.testing.assert_array_equal(g["tags"], oracle_lib.tags(cols[0], cols[1], cols[2], nets, lens,
                                                                 start, window))


@pytest.mark.parametrize("table", ["c1", "c5", "c5_first100"])
@pytest.mark.parametrize("tab", [0, 1, 2, 3])
def test_table_encodings_parity(S, oracle_lib, table, tab):
    """Every lookup-table encoding of the stream kernel (byte, packed, packed without level 2,
    global), on a SINET-like list, the 4096-entry /8-/32 list and a byte-sized /8-/32 list with
    prefixes longer than /24; records hit every interval edge +-1 and carry > 2^32 bytes (the
    ring's high-word spill).  An encoding that does not fit falls back to the automatic one."""
    nets, lens = prefix_table(WORKLOADS[table.split("_")[0]])
    if table.endswith("first100"):
        nets, lens = nets[:100], lens[:100]
    start, window = 1_613_660_400_000, 2_000_000
    for n in (129, 60_001):
        cols = _adversarial(n, nets, lens, start, window, seed=n + tab)
        cols = (np.sort(cols[0]),) + cols[1:]     # time ordered: the stream kernel's ring path
        for groups in (1, 2, "ws"):
            g = gpu_run(S, nets, lens, cols, start, window, order=1, tags=True, groups=groups, tab=tab)
            o = oracle_lib.classify_histogram(*cols, nets, lens, start, window, 1)
            assert_parity(g, o)
            np.testing.assert_array_equal(g["tags"], oracle_lib.tags(cols[0], cols[1], cols[2], nets, lens,
                                                                     start, window))
    # c5: no byte encoding (> 253 mixed /16 blocks) and its level 2 does not fit next to the ring
    assert g["h"].table_mode == (2 if table == "c5" and tab in (0, 1) else tab)


def _crowded_blocks_table():
    """Mixed /16 blocks with 1, 2, 3 (inline entry), 4-7 (second inline entry) and 8-20
    boundaries (boundary search) of the no-level-2 encoding, beside whole /16s and /8s."""
    nets, lens = [], []
    for b, k in enumerate((1, 2, 3, 4, 5, 6, 7, 8, 9, 20)):
        base = (133 << 24) | ((10 + b) << 16)
        # k boundaries: k // 2 separated /28s, plus one /28 running to the block end if k is odd
        for j in range(k // 2):
            nets.append(base | (j * 0x1000 + 0x20)); lens.append(28)
        if k % 2:
            nets.append(base | 0xFFF0); lens.append(28)
    nets += [(150 << 24) | (1 << 16), 10 << 24]; lens += [16, 8]
    return np.asarray(nets, np.uint32), np.asarray(lens, np.uint8)


@pytest.mark.parametrize("groups", [1, 2, "ws"])
def test_inline_block_entries_parity(S, oracle_lib, groups):
    """kTabPackedNoL2 forced: every inline-entry case bit-exact against the oracle (tags too)."""
    nets, lens = _crowded_blocks_table()
    start, window = 1_613_660_400_000, 1_000_000
    for n in (257, 80_003):
        cols = _adversarial(n, nets, lens, start, window, seed=n + (3 if groups == "ws" else groups))
        cols = (np.sort(cols[0]),) + cols[1:]
        g = gpu_run(S, nets, lens, cols, start, window, order=1, tags=True, groups=groups, tab=2)
        assert g["h"].table_mode == 2
        assert_parity(g, oracle_lib.classify_histogram(*cols, nets, lens, start, window, 1))
        np.testing.assert_array_equal(g["tags"], oracle_lib.tags(cols[0], cols[1], cols[2], nets, lens,
                                                                 start, window))


@pytest.mark.parametrize("wl_name,order", [("c1", "stream"), ("c1", "shuffled")])
def test_c1_full_parity(S, oracle_lib, wl_name, order):
    """BASELINE configs[0] at full size: 1M sessions, 1 h of 1 ms bins, 16 prefixes."""
    wl = WORKLOADS[wl_name].with_(order=order)
    nets, lens = prefix_table(wl)
    cols = to_numpy(records(wl))
    o = oracle_lib.classify_histogram(*cols, nets, lens, wl.window_start_ms, wl.window_ms, 1, threads=8)
    for strategy, groups, agg in ((0, 0, -1), (1, 1, 1), (1, 2, 1), (1, 2, 0), (1, "ws", -1), (2, 0, -1)):
        g = gpu_run(S, nets, lens, cols, wl.window_start_ms, wl.window_ms, order=strategy, groups=groups, agg=agg)
        assert_parity(g, o)


@pytest.mark.parametrize("groups", [1, 2, "ws"])
def test_dense_stream_both_layouts(S, oracle_lib, groups):
    """A dense stream (C2 density: ~1.2 records per ms) through both ring layouts."""
    wl = WORKLOADS["c2"].with_(n=4_000_000, window_ms=3_600_000)
    nets, lens = prefix_table(wl)
    cols = to_numpy(records(wl))
    o = oracle_lib.classify_histogram(*cols, nets, lens, wl.window_start_ms, wl.window_ms, 1, threads=8)
    g = gpu_run(S, nets, lens, cols, wl.window_start_ms, wl.window_ms, order=1, groups=groups, tags=True)
    assert_parity(g, o)
    np.testing.assert_array_equal(g["tags"], oracle_lib.tags(cols[0], cols[1], cols[2], nets, lens,
                                                             wl.window_start_ms, wl.window_ms))


@pytest.mark.parametrize("rpg", [0, 1, 64])
@pytest.mark.parametrize("groups", [1, 2])
@pytest.mark.parametrize("name", ["c2", "c4"])
def test_range_count_and_retire_parity(S, oracle_lib, name, groups, rpg):
    """Record ranges per ring group: automatic (~300 k records), one, and 64 (ranges of a few
    thousand records: many shared boundary tiles, initialised-by-another-CTA retires) over the
    dense uniform and the bursty shape, both ring layouts (one 512-thread group retires two
    tiles per round)."""
    wl = WORKLOADS[name].with_(n=6_000_000, window_ms=3_600_000)
    nets, lens = prefix_table(wl)
    cols = to_numpy(records(wl))
    o = oracle_lib.classify_histogram(*cols, nets, lens, wl.window_start_ms, wl.window_ms, 1, threads=8)
    h = S.SinetHistogram(nets, lens, wl.window_start_ms, wl.window_ms, 1, order=1)
    h.set_knob("stream_kernel", 1)
    h.set_tuning(groups, -1)
    h.set_knob("ranges_per_group", rpg)
    h.classify(*dev_cols(cols))
    g = {"count": np.stack([h.read_bins(k, S.METRIC_COUNT) for k in (0, 1)]),
         "bytes": np.stack([h.read_bins(k, S.METRIC_BYTES) for k in (0, 1)]), "totals": h.read_totals()}
    h.close()
    assert_parity(g, o)


@pytest.mark.parametrize("strategy,groups", [(1, 1), (1, 2), (1, "ws"), (2, 0)])
def test_bursty_hot_bins(S, oracle_lib, strategy, groups):
    """C4-shaped (diurnal + Zipf bursts + 1 % in one ms) and a degenerate all-in-one-ms batch."""
    wl = WORKLOADS["c4"].with_(n=2_000_000)
    nets, lens = prefix_table(wl)
    cols = to_numpy(records(wl))
    g = gpu_run(S, nets, lens, cols, wl.window_start_ms, wl.window_ms, order=strategy, groups=groups)
    o = oracle_lib.classify_histogram(*cols, nets, lens, wl.window_start_ms, wl.window_ms, 1, threads=8)
    assert_parity(g, o)
    ts, src, dst, nb = cols
    one = (np.full_like(ts, wl.window_start_ms + 43_200_000), src, dst, nb)
    g = gpu_run(S, nets, lens, one, wl.window_start_ms, wl.window_ms, order=strategy, groups=groups)
    o = oracle_lib.classify_histogram(*one, nets, lens, wl.window_start_ms, wl.window_ms, 1)
    assert_parity(g, o)


@pytest.mark.parametrize("strategy,groups", [(1, 1), (1, 2), (1, "ws"), (2, 0)])
def test_gaps_and_window_jumps(S, oracle_lib, strategy, groups):
    """Sparse records hours apart (window jumps), then a dense stretch, in one batch."""
    rng = np.random.default_rng(77)
    nets, lens = prefix_table(WORKLOADS["c2"])
    start, window = 1_613_660_400_000, 86_400_000
    sparse = np.sort(rng.integers(0, window, 3000))
    dense = 40_000_000 + np.sort(rng.integers(0, 60_000, 200_000))
    off = np.concatenate([sparse[:1500], dense, sparse[1500:]])
    n = len(off)
    ts = (start + off).astype(np.uint64)
    src = rng.choice(np.concatenate([nets, rng.integers(0, 1 << 32, 64).astype(np.uint32)]), n).astype(np.uint32)
    dst = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    nb = rng.integers(0, 1 << 34, n, dtype=np.uint64)
    cols = (ts, src, dst, nb)
    g = gpu_run(S, nets, lens, cols, start, window, order=strategy, groups=groups)
    o = oracle_lib.classify_histogram(*cols, nets, lens, start, window, 1)
    assert_parity(g, o)


# ----------------------------------------------------------------------------- partition then bin
@pytest.mark.parametrize("width", [1, 3, 1000])
@pytest.mark.parametrize("lut", [LUT_SRC_PRIORITY, LUT_ALG1])
def test_partitioned_adversarial_parity(S, oracle_lib, lut, width):
    """Unordered input through partition-then-bin (forced SHUFFLED + scratch): ragged sizes,
    edge addresses, u64 bytes near 2^63 (the high-word accumulator), tags; scratch of 2^16
    records makes the 200 k batch run as 4 sub-batches that add onto each other's tiles."""
    nets, lens = prefix_table(WORKLOADS["c1"])
    start, window = 1_613_660_400_000, 3_000_000
    for n in (1, 5, 2047, 2049, 200_001):
        cols = _adversarial(n, nets, lens, start, window, seed=3 * n + width)
        g = gpu_run(S, nets, lens, cols, start, window, width, lut, order=2, tags=True, scratch=1 << 16)
        assert g["h"].last_kernel.startswith("k_part")
        o = oracle_lib.classify_histogram(*cols, nets, lens, start, window, width, lut=lut)
        assert_parity(g, o)
        np.testing.assert_array_equal(g["tags"], oracle_lib.tags(cols[0], cols[1], cols[2], nets, lens,
                                                                 start, window))


@pytest.mark.parametrize("name", ["c1", "c4", "c5"])
def test_partitioned_workloads_parity(S, oracle_lib, name):
    """Shuffled C1 (1 h), C4-shaped bursts with the 1 % hot millisecond (one fine bucket holds
    ~1 % of all records: split into parts that add onto one tile) and the 4096-entry list."""
    wl = WORKLOADS[name].with_(n=3_000_000 if name != "c1" else 1_000_000, order="shuffled")
    nets, lens = prefix_table(wl)
    cols = to_numpy(records(wl))
    o = oracle_lib.classify_histogram(*cols, nets, lens, wl.window_start_ms, wl.window_ms, 1, threads=8)
    for strategy in (0, 2):   # AUTO (the probe finds the order) and forced SHUFFLED
        g = gpu_run(S, nets, lens, cols, wl.window_start_ms, wl.window_ms, order=strategy, scratch=1 << 22)
        assert g["h"].last_kernel.startswith("k_part"), g["h"].last_kernel
        assert_parity(g, o)
    ts, src, dst, nb = cols
    one = (np.full_like(ts, wl.window_start_ms + 1_800_000), src, dst, nb)   # every record in one ms
    g = gpu_run(S, nets, lens, one, wl.window_start_ms, wl.window_ms, order=2, scratch=1 << 20)
    assert_parity(g, oracle_lib.classify_histogram(*one, nets, lens, wl.window_start_ms, wl.window_ms, 1))


def test_partitioned_watchlist_and_fallback(S, oracle_lib):
    """NEXT-2 filter on the partitioned path; a window of more than 2^27 bins refuses scratch
    and keeps the L2-atomic kernel."""
    wl = WORKLOADS["c1"].with_(n=400_000, order="shuffled")
    nets, lens = prefix_table(wl)
    cols = to_numpy(records(wl))
    watch = np.unique(np.concatenate([cols[1][::97], cols[2][::89]]))
    o = oracle_lib.classify_histogram_watched(*cols, nets, lens, watch, wl.window_start_ms, wl.window_ms, 1)
    h = S.SinetHistogram(nets, lens, wl.window_start_ms, wl.window_ms, order=2)
    h.set_scratch(1 << 17)
    h.set_watchlist(watch)
    h.classify(*dev_cols(cols))
    assert h.last_kernel.startswith("k_part")
    np.testing.assert_array_equal(np.stack([h.read_bins(k, 0) for k in (0, 1)]), o.count)
    np.testing.assert_array_equal(np.stack([h.read_bins(k, 1) for k in (0, 1)]), o.bytes)
    np.testing.assert_array_equal(h.read_totals(), o.totals)
    big = S.SinetHistogram(nets, lens, wl.window_start_ms, (1 << 27) + 8192, order=2)
    with pytest.raises(S.SinetError):
        big.set_scratch(1 << 16)


def test_chunked_accumulation_and_reset(S, oracle_lib):
    wl = WORKLOADS["c1"].with_(n=300_000)
    nets, lens = prefix_table(wl)
    cols = to_numpy(records(wl))
    o = oracle_lib.classify_histogram(*cols, nets, lens, wl.window_start_ms, wl.window_ms, 1)
    g = gpu_run(S, nets, lens, cols, wl.window_start_ms, wl.window_ms,
                chunks=[(0, 4), (4, 1001), (1001, 1001), (1001, 250_000), (250_000, 300_000)])
    assert_parity(g, o)
    h = g["h"]
    # reset: a new epoch starts empty; re-running gives the same result (bins not re-zeroed by memset)
    h.reset()
    z = h.read_totals()
    assert not z.any()
    assert not h.read_bins(0, 0).any() and not h.read_bins(1, 1).any()
    d = dev_cols(cols)
    for _ in range(2):
        h.reset()
        h.classify(*d)
    np.testing.assert_array_equal(np.stack([h.read_bins(k, 0) for k in (0, 1)]), o.count)
    np.testing.assert_array_equal(h.read_totals(), o.totals)


def test_empty_input_and_errors(S):
    nets, lens = prefix_table(WORKLOADS["c1"])
    h = S.SinetHistogram(nets, lens, 1000, 100, 1)
    e64 = torch.empty(0, dtype=torch.int64, device="cuda")
    e32 = torch.empty(0, dtype=torch.int32, device="cuda")
    h.classify(e64, e32, e32, e64)
    assert not h.read_totals().any() and not h.read_bins(0, 0).any()
    x64 = torch.zeros(9, dtype=torch.int64, device="cuda")
    x32 = torch.zeros(9, dtype=torch.int32, device="cuda")
    with pytest.raises(S.SinetError) as ei:
        h.classify(x64[1:], x32[:8], x32[:8], x64[1:])   # columns at different record offsets
    assert ei.value.code == -2
    h.classify(x64[1:], x32[1:], x32[1:], x64[1:])       # same offset (a slice): accepted
    with pytest.raises(S.SinetError) as ei:
        h.read_bins(0, 0, first=50, n=51)
    assert ei.value.code == -3
    h.reduce()
    with pytest.raises(S.SinetError) as ei:
        h.classify(x64[:8], x32[:8], x32[:8], x64[:8])
    assert ei.value.code == -6
    h.reset()
    h.classify(x64[:8], x32[:8], x32[:8], x64[:8])


def test_host_streaming_path(S, oracle_lib):
    wl = WORKLOADS["c1"].with_(n=500_000)
    nets, lens = prefix_table(wl)
    rec = records(wl)
    cols = to_numpy(rec)
    o = oracle_lib.classify_histogram(*cols, nets, lens, wl.window_start_ms, wl.window_ms, 1)
    h = S.SinetHistogram(nets, lens, wl.window_start_ms, wl.window_ms)
    pin = [rec[k].pin_memory() for k in ("ts", "src", "dst", "bytes")]
    h.classify_host(*pin, chunk_records=65_536 + 4)
    np.testing.assert_array_equal(np.stack([h.read_bins(k, 1) for k in (0, 1)]), o.bytes)
    np.testing.assert_array_equal(h.read_totals(), o.totals)


def test_reduce_single_rank_is_identity(S, oracle_lib):
    wl = WORKLOADS["c1"].with_(n=100_000)
    nets, lens = prefix_table(wl)
    cols = to_numpy(records(wl))
    o = oracle_lib.classify_histogram(*cols, nets, lens, wl.window_start_ms, wl.window_ms, 1)
    h = S.SinetHistogram(nets, lens, wl.window_start_ms, wl.window_ms)
    h.classify(*dev_cols(cols))
    h.reduce()
    assert h.owned_range() == (0, wl.nbins)
    np.testing.assert_array_equal(np.stack([h.read_bins(k, 0) for k in (0, 1)]), o.count)


def test_generator_cpu_gpu_identical(S):
    for name in ("c1", "c4"):
        wl = WORKLOADS[name].with_(n=200_000)
        a = records(wl, 1000, 150_000, device="cpu")
        b = records(wl, 1000, 150_000, device="cuda")
        for k in a:
            assert torch.equal(a[k], b[k].cpu()), (name, k)


@pytest.mark.slow
@pytest.mark.parametrize("strategy", [0, 2])
def test_c2_full_size_parity(S, oracle_lib, strategy):
    """BASELINE configs[1] at full size (100M sessions, one day of 1 ms bins, 64
    prefixes), in the bench's launch configuration, every bin vs the oracle."""
    wl = WORKLOADS["c2"]
    nets, lens = prefix_table(wl)
    rec = records(wl, device="cuda")
    h = S.SinetHistogram(nets, lens, wl.window_start_ms, wl.window_ms, order=strategy)
    h.classify(rec["ts"], rec["src"], rec["dst"], rec["bytes"])
    h.finalize()
    cols = tuple(c for c in to_numpy({k: rec[k].cpu() for k in rec}))
    del rec
    torch.cuda.empty_cache()
    import os
    o = oracle_lib.classify_histogram(*cols, nets, lens, wl.window_start_ms, wl.window_ms, 1,
                                      threads=max(1, len(os.sched_getaffinity(0))))
    for d in (0, 1):
        np.testing.assert_array_equal(h.read_bins(d, 0), o.count[d])
        np.testing.assert_array_equal(h.read_bins(d, 1), o.bytes[d])
    np.testing.assert_array_equal(h.read_totals(), o.totals)


# ----------------------------------------------------------------------------- NEXT-1 series read-out
@pytest.mark.parametrize("factor", [1, 7, 1000, 600_000, 3_600_000])
def test_rebin_parity(S, oracle_lib, factor):
    wl = WORKLOADS["c1"].with_(n=400_000)
    nets, lens = prefix_table(wl)
    cols = to_numpy(records(wl))
    o = oracle_lib.classify_histogram(*cols, nets, lens, wl.window_start_ms, wl.window_ms, 1)
    g = gpu_run(S, nets, lens, cols, wl.window_start_ms, wl.window_ms)
    out = g["h"].rebin(factor).cpu().numpy().view(np.uint64)
    for d in (0, 1):
        np.testing.assert_array_equal(out[:, d, 0], oracle_lib.rebin(o.count[d], factor))
        np.testing.assert_array_equal(out[:, d, 1], oracle_lib.rebin(o.bytes[d], factor))


def test_sparse_export_parity(S, oracle_lib):
    wl = WORKLOADS["c1"].with_(n=300_000)
    nets, lens = prefix_table(wl)
    cols = to_numpy(records(wl))
    o = oracle_lib.classify_histogram(*cols, nets, lens, wl.window_start_ms, wl.window_ms, 1)
    g = gpu_run(S, nets, lens, cols, wl.window_start_ms, wl.window_ms)
    for d in (0, 1):
        (t, c, b), n = g["h"].export_sparse(d)
        et, ec, eb = oracle_lib.sparse(o.count[d], o.bytes[d], wl.window_start_ms, 1)
        assert n == len(et)
        np.testing.assert_array_equal(t.cpu().numpy().view(np.uint64), et)
        np.testing.assert_array_equal(c.cpu().numpy().view(np.uint64), ec)
        np.testing.assert_array_equal(b.cpu().numpy().view(np.uint64), eb)
        (t2, _, _), n2 = g["h"].export_sparse(d, capacity=100)   # truncated output keeps the first entries
        assert n2 == n and np.array_equal(t2.cpu().numpy().view(np.uint64), et[:100])


# ----------------------------------------------------------------------------- NEXT-4 comparator
@pytest.mark.parametrize("order", ["stream", "shuffled"])
def test_sortreduce_comparator_parity(S, oracle_lib, order):
    """The paper's sort + reduce_by_key design (CUB) gives the same bins as the oracle."""
    wl = WORKLOADS["c1"].with_(order=order)
    nets, lens = prefix_table(wl)
    cols = to_numpy(records(wl))
    o = oracle_lib.classify_histogram(*cols, nets, lens, wl.window_start_ms, wl.window_ms, 1, threads=8)
    h = S.SinetHistogram(nets, lens, wl.window_start_ms, wl.window_ms)
    d = dev_cols(cols)
    scratch = h.classify_sortreduce(*d)
    assert h.last_strategy == 3
    np.testing.assert_array_equal(np.stack([h.read_bins(k, 0) for k in (0, 1)]), o.count)
    np.testing.assert_array_equal(np.stack([h.read_bins(k, 1) for k in (0, 1)]), o.bytes)
    np.testing.assert_array_equal(h.read_totals(), o.totals)
    # accumulates like classify(): a second pass doubles every bin
    h.classify_sortreduce(*(c[1:] for c in d), scratch=scratch)
    h.classify(*(c[:1] for c in d))
    np.testing.assert_array_equal(np.stack([h.read_bins(k, 0) for k in (0, 1)]), o.count * np.uint64(2))


def test_nccl_reduce_single_rank(S, oracle_lib):
    """The NCCL merge path (run-time loaded libnccl, in-place u64 reduce-scatter +
    totals all-reduce) on a one-rank communicator: bins and totals unchanged."""
    wl = WORKLOADS["c1"].with_(n=200_000)
    nets, lens = prefix_table(wl)
    cols = to_numpy(records(wl))
    o = oracle_lib.classify_histogram(*cols, nets, lens, wl.window_start_ms, wl.window_ms, 1)
    import torch.distributed  # noqa: F401  (loads torch's libnccl.so.2 into the process)
    h = S.SinetHistogram(nets, lens, wl.window_start_ms, wl.window_ms)
    h.comm_init(S.SinetHistogram.new_unique_id())
    h.classify(*dev_cols(cols))
    h.reduce()
    assert h.owned_range() == (0, wl.nbins)
    np.testing.assert_array_equal(np.stack([h.read_bins(k, 1) for k in (0, 1)]), o.bytes)
    np.testing.assert_array_equal(h.read_totals(), o.totals)


# ----------------------------------------------------------------------------- NEXT-2 watchlist
@pytest.mark.parametrize("strategy", [1, 2])
def test_watchlist_parity(S, oracle_lib, strategy):
    """Filter by an exact-IP watchlist (either endpoint), then histogram, vs the oracle."""
    wl = WORKLOADS["c1"].with_(n=400_000)
    nets, lens = prefix_table(wl)
    cols = to_numpy(records(wl))
    rng = np.random.default_rng(300)
    listed = np.concatenate([rng.choice(cols[1], 150), rng.choice(cols[2], 150),
                             rng.integers(0, 1 << 32, 577, dtype=np.uint64).astype(np.uint32)])
    o = oracle_lib.classify_histogram_watched(*cols, nets, lens, listed, wl.window_start_ms, wl.window_ms, 1)
    for sr in (False, True):
        h = S.SinetHistogram(nets, lens, wl.window_start_ms, wl.window_ms, order=strategy)
        h.set_watchlist(listed)
        d = dev_cols(cols)
        if sr:
            h.classify_sortreduce(*d)
        else:
            h.classify(*d)
        np.testing.assert_array_equal(np.stack([h.read_bins(k, 0) for k in (0, 1)]), o.count)
        np.testing.assert_array_equal(np.stack([h.read_bins(k, 1) for k in (0, 1)]), o.bytes)
        np.testing.assert_array_equal(h.read_totals(), o.totals)
        h.set_watchlist(None)   # removing the filter restores the full histogram
        h.reset()
        h.classify(*d)
        assert int(h.read_totals()[:4].sum()) == wl.n


@pytest.mark.parametrize("strategy", [1, 2])
def test_touched_range_is_binned_extent(S, oracle_lib, strategy):
    """The extent the sparse multi-GPU exchange relies on: min/max bin with data."""
    wl = WORKLOADS["c1"].with_(n=200_000)
    nets, lens = prefix_table(wl)
    cols = to_numpy(records(wl))
    o = oracle_lib.classify_histogram(*cols, nets, lens, wl.window_start_ms, wl.window_ms, 1)
    nz = np.nonzero((o.count[0] + o.count[1]) > 0)[0]
    for sr in (False, True):
        h = S.SinetHistogram(nets, lens, wl.window_start_ms, wl.window_ms, order=strategy)
        d = dev_cols(cols)
        (h.classify_sortreduce if sr else h.classify)(*(c[5000:150_000] for c in d))
        sub = oracle_lib.classify_histogram(*(c[5000:150_000] for c in cols), nets, lens, wl.window_start_ms,
                                            wl.window_ms, 1)
        snz = np.nonzero((sub.count[0] + sub.count[1]) > 0)[0]
        assert h.touched_range() == (int(snz.min()), int(snz.max()))
        h.reset()
        assert h.touched_range() == (0xFFFFFFFF, 0)
        h.classify(*d)
        assert h.touched_range() == (int(nz.min()), int(nz.max()))


# ----------------------------------------------------------------------------- full-size configs
def _full_records(wl, device="cuda", chunk=200_000_000):
    """All records of a BASELINE config on the device, generated in chunks (bounded temporaries)."""
    from synth.sinet_synth import stream_order
    order = stream_order(wl, device)
    out = {"ts": torch.empty(wl.n, dtype=torch.int64, device=device),
           "src": torch.empty(wl.n, dtype=torch.int32, device=device),
           "dst": torch.empty(wl.n, dtype=torch.int32, device=device),
           "bytes": torch.empty(wl.n, dtype=torch.int64, device=device)}
    for lo in range(0, wl.n, chunk):
        hi = min(wl.n, lo + chunk)
        r = records(wl, lo, hi, device=device, order=order)
        for k in out:
            out[k][lo:hi] = r[k]
        del r
    del order
    torch.cuda.empty_cache()
    return out


def _plane_sha256(bins_cpu):
    """SHA-256 of each full (dir, metric) plane, u64 little endian (tools/oracle_digests.py layout)."""
    import hashlib
    a = bins_cpu.numpy().view(np.uint64)
    names = ("out_count", "out_bytes", "in_count", "in_bytes")
    return {names[2 * d + m]: hashlib.sha256(np.ascontiguousarray(a[:, d, m]).astype("<u8").tobytes()).hexdigest()
            for d in (0, 1) for m in (0, 1)}


def _golden_digests():
    import json
    import os
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "digests.json")) as f:
        return json.load(f)


@pytest.mark.slow
@pytest.mark.parametrize("order", ["stream", "shuffled"])
@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_full_size_digest_parity(S, name, order):
    """Every BASELINE config at full size on one GPU (1 M / 100 M / 1.2 B / 1.6 B bursty /
    400 M with the 4096-entry list), in both record orders, default strategy: the SHA-256 of
    each full (dir, metric) plane and the 12 totals equal the oracle's (tests/golden/digests.json,
    written by tools/oracle_digests.py from oracle/ + synth/ only).  The histogram is a
    function of the records as a multiset, so one digest serves both orders."""
    dg = _golden_digests()
    if name not in dg:
        pytest.skip(f"no committed oracle digest for {name}")
    exp = dg[name]
    wl = WORKLOADS[name].with_(order=order)
    assert exp["n"] == wl.n and exp["nbins"] == wl.nbins and exp["seed"] == wl.seed
    nets, lens = prefix_table(wl)
    rec = _full_records(wl)
    h = S.SinetHistogram(nets, lens, wl.window_start_ms, wl.window_ms)
    h.classify(rec["ts"], rec["src"], rec["dst"], rec["bytes"])
    h.finalize()
    del rec
    torch.cuda.empty_cache()
    assert [int(x) for x in h.read_totals()] == exp["totals"]
    assert _plane_sha256(h.bins_view()[: wl.nbins].cpu()) == exp["sha256"]
    h.close()


# ----------------------------------------------------------------------------- NEXT-4 labelled LPM
@pytest.mark.parametrize("strategy", [1, 2])
def test_labelled_lpm_parity(S, oracle_lib, strategy):
    """C5-shaped table (4096 nested /8-/32 entries) with 30 % carve-outs: longest match decides."""
    wl = WORKLOADS["c5"].with_(n=500_000, window_ms=3_600_000)
    nets, lens = prefix_table(wl)
    labels = (np.random.default_rng(5).random(len(nets)) < 0.7).astype(np.uint8)
    cols = to_numpy(records(wl))
    o = oracle_lib.classify_histogram_lpm(*cols, nets, lens, labels, wl.window_start_ms, wl.window_ms, 1)
    h = S.SinetHistogram(nets, lens, wl.window_start_ms, wl.window_ms, order=strategy, labels=labels)
    tg = torch.empty(wl.n, dtype=torch.uint8, device="cuda")
    h.classify(*dev_cols(cols), tags=tg)
    np.testing.assert_array_equal(np.stack([h.read_bins(k, 0) for k in (0, 1)]), o.count)
    np.testing.assert_array_equal(np.stack([h.read_bins(k, 1) for k in (0, 1)]), o.bytes)
    np.testing.assert_array_equal(h.read_totals(), o.totals)
    t = tg.cpu().numpy()
    np.testing.assert_array_equal(t & 1, oracle_lib.member_lpm(cols[1], nets, lens, labels))
    np.testing.assert_array_equal((t >> 1) & 1, oracle_lib.member_lpm(cols[2], nets, lens, labels))
