"""CPU-only checks of libsinet: it loads, exports every symbol include/sinet.h
declares, validates arguments, and its prefix compiler (evaluated on the host
with the kernels' lookup) agrees with the oracle.  No compute call needs a GPU."""
import ctypes

import numpy as np
import pytest

from paper_2106_12863_b200 import _native as N
from paper_2106_12863_b200 import owned_bin_range, padded_bins, shard_range, table_member_host
from synth import WORKLOADS, prefix_table
from tests.helpers import edge_addresses


def test_every_header_symbol_is_exported():
    names = N.header_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(N.lib, name), f"libsinet.so does not export {name}"
    assert N.lib.sinet_abi_version() == N._header_abi_version() == 3


def test_hub_create_validates_world():
    h = ctypes.c_void_p()
    assert N.lib.sinet_hub_create(ctypes.byref(h), 0) == N.E_INVAL
    assert N.lib.sinet_hub_create(ctypes.byref(h), 65) == N.E_INVAL
    assert N.lib.sinet_hub_create(None, 2) == N.E_INVAL
    assert N.lib.sinet_hub_create(ctypes.byref(h), 8) == N.OK and h.value
    N.lib.sinet_hub_destroy(h)
    N.lib.sinet_hub_destroy(None)
    assert N.lib.sinet_comm_init_hub(None, None) == N.E_INVAL
    assert N.lib.sinet_set_knob(None, b"stream_groups", 1) == N.E_INVAL


def _cfg(**kw):
    c = N.Config()
    c.window_start_ms = kw.get("start", 1613660400000)
    c.window_ms = kw.get("window", 86_400_000)
    c.bin_width_ms = kw.get("width", 1)
    for k, v in enumerate(kw.get("lut", N.LUT_SRC_PRIORITY)):
        c.dir_lut[k] = v
    c.world = kw.get("world", 1)
    c.rank = kw.get("rank", 0)
    return c


def test_sizing():
    t = N.lib.sinet_tile_bins()
    c = _cfg()
    assert N.lib.sinet_bins_bytes(ctypes.byref(c)) == 32 * padded_bins(86_400_000, 1, t)
    c8 = _cfg(world=8, rank=3)
    bp = padded_bins(86_400_000, 8, t)
    assert bp % (8 * t) == 0 and bp >= 86_400_000 and bp - 86_400_000 < 8 * t
    assert N.lib.sinet_bins_bytes(ctypes.byref(c8)) == 32 * bp
    assert N.lib.sinet_workspace_bytes(ctypes.byref(c), 64) > 65536 * 4
    assert N.lib.sinet_workspace_bytes(ctypes.byref(c), 0) == 0


@pytest.mark.parametrize("bad", [dict(window=0), dict(width=0), dict(window=10, width=3),
                                 dict(window=1 << 32), dict(world=0), dict(world=2, rank=2),
                                 dict(lut=(0, 1, 3, 0)), dict(start=(1 << 64) - 5, window=10)])
def test_invalid_config_rejected(bad):
    c = _cfg(**bad)
    assert N.lib.sinet_bins_bytes(ctypes.byref(c)) == 0
    ctx = ctypes.c_void_p()
    nets = np.array([1], np.uint32)
    lens = np.array([8], np.uint8)
    rc = N.lib.sinet_open(ctypes.byref(ctx), ctypes.byref(c), nets.ctypes.data_as(ctypes.c_void_p),
                          lens.ctypes.data_as(ctypes.c_void_p), 1, None, 0, None, 0)
    assert rc == N.E_INVAL and not ctx.value


def test_invalid_table_rejected():
    c = _cfg()
    ctx = ctypes.c_void_p()
    nets = np.array([1, 2], np.uint32)
    lens = np.array([8, 33], np.uint8)
    for n in (0, 2):   # empty list / prefix_len > 32
        rc = N.lib.sinet_open(ctypes.byref(ctx), ctypes.byref(c), nets.ctypes.data_as(ctypes.c_void_p),
                              lens.ctypes.data_as(ctypes.c_void_p), n, None, 0, None, 0)
        assert rc == N.E_INVAL
    with pytest.raises(N.SinetError):
        table_member_host([1], [40], [5])


@pytest.mark.parametrize("wl", ["c1", "c2", "c5", "c5_first100"])
def test_compiled_table_matches_oracle(oracle_lib, wl):
    """Prefix compiler (a1) + the kernels' lookups (every table encoding, checked against each
    other inside table_member_host) == the oracle's literal linear scan.  c5_first100: a
    /8-/32 list small enough for the byte encoding, with prefixes longer than /24."""
    nets, lens = prefix_table(WORKLOADS[wl.split("_")[0]])
    if wl.endswith("first100"):
        nets, lens = nets[:100], lens[:100]
    rng = np.random.default_rng(5)
    edges = edge_addresses(nets, lens)
    ips = np.concatenate([edges, rng.integers(0, 1 << 32, 20_000 if wl == "c5" else 200_000,
                                              dtype=np.uint64).astype(np.uint32)])
    got = table_member_host(nets, lens, ips)
    # oracle membership via its tags (bit 0 = s_in), one C call for the whole batch
    z = np.zeros(len(ips), np.uint64)
    exp = oracle_lib.tags(z, ips, ips, nets, lens, 0, 1) & 1
    np.testing.assert_array_equal(got, exp)


def test_compiled_table_random_lists_with_host_bits(oracle_lib):
    rng = np.random.default_rng(11)
    for trial in range(60):
        p = int(rng.integers(1, 40))
        nets = rng.integers(0, 1 << 32, p, dtype=np.uint64).astype(np.uint32)
        lens = rng.choice([0, 1, 2, 7, 8, 15, 16, 17, 23, 24, 31, 32], p).astype(np.uint8)
        if trial % 3 == 0:
            lens = np.maximum(lens, 12).astype(np.uint8)   # avoid /0 swallowing everything
        ips = np.concatenate([edge_addresses(nets & ~np.uint32(0), lens),
                              rng.integers(0, 1 << 32, 5000, dtype=np.uint64).astype(np.uint32)])
        got = table_member_host(nets, lens, ips)
        exp = oracle_lib.tags(np.zeros(len(ips), np.uint64), ips, ips, nets, lens, 0, 1) & 1
        np.testing.assert_array_equal(got, exp)


def test_shard_and_owned_ranges_partition():
    for n in (0, 1, 7, 1_000_003):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
    for nbins in (1, 3_600_000, 86_400_000):
        for world in (1, 2, 4, 8):
            own = [owned_bin_range(nbins, r, world) for r in range(world)]
            assert own[0][0] == 0 and own[-1][1] == nbins
            assert all(own[i][1] == own[i + 1][0] for i in range(world - 1))


def test_exchange_plan_edges():
    from paper_2106_12863_b200 import exchange_plan
    # rank 1 of 4 owns [250, 500) of B = 1000 (pad 1024 -> per 256: [256, 512))
    t = np.array([[0, 300], [200, 600], [0xFFFFFFFF, 0], [999, 999]], np.uint32)
    send, recv = exchange_plan(4, 1, 1000, 1024, t)
    assert send[1].tolist() == [0, 0]                      # nothing to myself
    assert send[0].tolist() == [200, 56]                   # my [200,600] ∩ own(0)=[0,256)
    assert send[2].tolist() == [512, 89]                   # ∩ own(2)=[512,768)
    assert recv[0].tolist() == [256, 45]                   # rank 0's [0,300] ∩ own(1)=[256,512)
    assert recv[2].tolist() == [0, 0] and recv[3].tolist() == [0, 0]   # empty / disjoint
    with pytest.raises(N.SinetError):
        exchange_plan(3, 0, 1000, 1024, t[:3])             # pad not a multiple of world


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_labelled_lpm_table_matches_oracle(oracle_lib, seed):
    """NEXT-4: the labelled table compiled to member intervals == the oracle's literal LPM scan."""
    rng = np.random.default_rng(seed)
    from synth import WORKLOADS, prefix_table
    nets, lens = prefix_table(WORKLOADS["c5"])          # nested /8-/32 entries
    nets, lens = nets[:3000], lens[:3000]
    labels = (rng.random(len(nets)) < 0.7).astype(np.uint8)
    ips = np.concatenate([edge_addresses(nets, lens),
                          rng.integers(0, 1 << 32, 30_000, dtype=np.uint64).astype(np.uint32)])
    got = table_member_host(nets, lens, ips, labels)
    np.testing.assert_array_equal(got, oracle_lib.member_lpm(ips, nets, lens, labels))
    # duplicates: the last equal entry wins
    n2 = np.array([ip_ for ip_ in (0x85000000, 0x85000000)], np.uint32)
    l2 = np.array([8, 8], np.uint8)
    assert table_member_host(n2, l2, [0x85010203], [1, 0]).tolist() == [0]
    assert table_member_host(n2, l2, [0x85010203], [0, 1]).tolist() == [1]


def test_compiled_table_crowded_blocks(oracle_lib):
    """Mixed /16 blocks with 1-9 and 20 boundaries: every inline-entry case of the no-level-2
    encoding (mirrored inside table_member_host) == the oracle's linear scan."""
    from tests.test_gpu_parity import _crowded_blocks_table
    nets, lens = _crowded_blocks_table()
    rng = np.random.default_rng(7)
    ips = np.concatenate([edge_addresses(nets, lens),
                          ((133 << 24) | rng.integers(0, 1 << 24, 50_000)).astype(np.uint32)])
    exp = oracle_lib.tags(np.zeros(len(ips), np.uint64), ips, ips, nets, lens, 0, 1) & 1
    np.testing.assert_array_equal(table_member_host(nets, lens, ips), exp)
