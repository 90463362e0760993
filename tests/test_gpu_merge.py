"""GPU parity of the cross-GPU merge (row a8: merge-scatter of per-GPU partials).

`world` ranks run on ONE B200 as `world` ctxs of one process, each fed its contiguous
record shard (one chunk per GPU thread), joined by the in-process hub
(sinet_comm_init_hub) and merged by `sinet_reduce` called concurrently from one host
thread per rank -- the same code as the NCCL path: touched-range all-gather, host plan,
partial materialisation, send/recv into staging + k_add_bins (sparse), or the dense
reduce-scatter (k_sum_peers over peer memory), and the totals all-reduce.  Every owner's
slice and the global totals must equal the single-process oracle bit for bit.
"""
import threading

import numpy as np
import pytest
import torch

from synth import WORKLOADS, prefix_table, records
from synth.sinet_synth import stream_order, to_numpy

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_12863_b200 as S
    return S


def _oracle_full(oracle_lib, wl, order):
    nets, lens = prefix_table(wl)
    cols = to_numpy(records(wl, order=order))[:4]
    return oracle_lib.classify_histogram(*cols, nets, lens, wl.window_start_ms, wl.window_ms, wl.bin_width_ms,
                                         threads=4)


def _run_world(S, wl, world, exchange, order_t, own_streams=True):
    nets, lens = prefix_table(wl)
    dev = torch.device("cuda", 0)
    rec = records(wl, device=dev, order=order_t)
    hub = S.SinetHub(world)
    hs, streams = [], []
    for r in range(world):
        st = torch.cuda.Stream(dev) if own_streams else torch.cuda.current_stream(dev)
        h = S.SinetHistogram(nets, lens, wl.window_start_ms, wl.window_ms, wl.bin_width_ms, device=0, rank=r,
                             world=world, stream=st)
        h.comm_init_hub(hub)
        if exchange is not None:
            h.set_exchange(exchange)
        hs.append(h)
        streams.append(st)
    torch.cuda.synchronize()
    for r, h in enumerate(hs):
        lo, hi = S.shard_range(wl.n, r, world)
        with torch.cuda.stream(streams[r]):
            h.classify(rec["ts"][lo:hi], rec["src"][lo:hi], rec["dst"][lo:hi], rec["bytes"][lo:hi])
    launches0 = [h.launches for h in hs]
    errs = [None] * world

    def reduce(r):
        try:
            hs[r].reduce()
        except Exception as e:  # noqa: BLE001
            errs[r] = e

    th = [threading.Thread(target=reduce, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not any(t.is_alive() for t in th), "hub merge did not finish"
    assert errs == [None] * world, errs
    torch.cuda.synchronize()
    return hs, hub, launches0


def _check_owned(S, hs, o, wl):
    covered = 0
    for h in hs:
        lo, hi = h.owned_range()
        assert (lo, hi) == S.owned_bin_range(wl.nbins, h.rank, h.world)
        covered += hi - lo
        for d in (0, 1):
            np.testing.assert_array_equal(h.read_bins(d, S.METRIC_COUNT), o.count[d, lo:hi])
            np.testing.assert_array_equal(h.read_bins(d, S.METRIC_BYTES), o.bytes[d, lo:hi])
        np.testing.assert_array_equal(h.read_totals(), o.totals)   # global totals on every rank
    assert covered == wl.nbins


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("exchange", [0, 1, 2])
def test_hub_merge_stream_shards(S, oracle_lib, world, exchange):
    # contiguous time-ordered shards: each rank touches about its own part of the hour, the
    # sparse exchange moves only the ~2 s boundary overlaps
    wl = WORKLOADS["c1"].with_(n=400_003)
    order = stream_order(wl, "cuda")
    o = _oracle_full(oracle_lib, wl, order.cpu())
    hs, hub, l0 = _run_world(S, wl, world, exchange, order)
    _check_owned(S, hs, o, wl)
    want = {0: 2, 1: 1, 2: 2}[exchange]     # auto picks sparse: it moves far less than half
    assert all(h.last_exchange == want for h in hs)
    if want == 2:
        # every owner whose range overlaps a neighbour's shard received and added partial bins
        assert sum(h.launches - a for h, a in zip(hs, l0)) >= world
    for h in hs:
        h.close()


@pytest.mark.parametrize("world", [2, 8])
@pytest.mark.parametrize("exchange", [0, 1, 2])
def test_hub_merge_shuffled_shards(S, oracle_lib, world, exchange):
    # shuffled records: every rank touches the whole window, sparse degrades to dense
    wl = WORKLOADS["c1"].with_(n=300_001, order="shuffled")
    order = stream_order(wl, "cuda")
    o = _oracle_full(oracle_lib, wl, order.cpu())
    hs, hub, _ = _run_world(S, wl, world, exchange, order)
    _check_owned(S, hs, o, wl)
    assert all(h.last_exchange == 1 for h in hs)   # staging too small for whole slices: dense
    for h in hs:
        h.close()


def test_hub_merge_sparse_overlapping_and_empty_ranks(S, oracle_lib):
    # ranks whose shards overlap in time heavily, and ranks with no records at all
    wl = WORKLOADS["c1"].with_(n=200_000)
    order = stream_order(wl, "cuda")
    o = _oracle_full(oracle_lib, wl, order.cpu())
    nets, lens = prefix_table(wl)
    rec = records(wl, device="cuda", order=order)
    world = 4
    hub = S.SinetHub(world)
    hs = []
    for r in range(world):
        h = S.SinetHistogram(nets, lens, wl.window_start_ms, wl.window_ms, device=0, rank=r, world=world,
                             stream=torch.cuda.Stream())
        h.comm_init_hub(hub)
        h.set_exchange(2)
        hs.append(h)
    torch.cuda.synchronize()
    # rank 0 and 2 take alternate records of the first half, rank 1 the second half, rank 3 nothing
    half = wl.n // 2
    idx0 = torch.arange(0, half, 2, device="cuda")
    idx2 = torch.arange(1, half, 2, device="cuda")
    parts = {0: idx0, 2: idx2, 1: torch.arange(half, wl.n, device="cuda")}
    for r, ix in parts.items():
        cols = [rec[k][ix].contiguous() for k in ("ts", "src", "dst", "bytes")]
        with torch.cuda.stream(hs[r].stream):
            hs[r].classify(*cols)
        torch.cuda.synchronize()
    errs = []
    th = [threading.Thread(target=lambda h=h: (errs.append(None), h.reduce()), daemon=True) for h in hs]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    torch.cuda.synchronize()
    _check_owned(S, hs, o, wl)
    for h in hs:
        h.close()


@pytest.mark.parametrize("world", [3, 8])
def test_hub_merge_then_rebin_frames(S, oracle_lib, world):
    # NEXT-1 after the merge: frames are aligned to the window start on every rank; a frame that
    # straddles two owned ranges is the sum of the two ranks' entries for it
    wl = WORKLOADS["c1"].with_(n=250_000)
    order = stream_order(wl, "cuda")
    o = _oracle_full(oracle_lib, wl, order.cpu())
    hs, hub, _ = _run_world(S, wl, world, 0, order)
    for factor in (600_000, 1000, 7):
        want_c = np.stack([oracle_lib.rebin(o.count[d], factor) for d in (0, 1)])
        want_b = np.stack([oracle_lib.rebin(o.bytes[d], factor) for d in (0, 1)])
        got = np.zeros((want_c.shape[1], 2, 2), np.uint64)
        for h in hs:
            f0, nf = h.rebin_frames(factor)
            part = h.rebin(factor).cpu().numpy().view(np.uint64)
            assert part.shape[0] == nf
            got[f0:f0 + nf] += part
        np.testing.assert_array_equal(got[:, :, 0].T, want_c)
        np.testing.assert_array_equal(got[:, :, 1].T, want_b)
    for h in hs:
        h.close()


def test_hub_repeated_days_same_ctxs(S, oracle_lib):
    # reset -> classify -> reduce twice on the same ctxs and hub (event parity across collectives)
    wl = WORKLOADS["c1"].with_(n=150_000)
    order = stream_order(wl, "cuda")
    o = _oracle_full(oracle_lib, wl, order.cpu())
    hs, hub, _ = _run_world(S, wl, 3, 0, order)
    _check_owned(S, hs, o, wl)
    rec = records(wl, device="cuda", order=order)
    for h in hs:
        h.reset()
    for r, h in enumerate(hs):
        lo, hi = S.shard_range(wl.n, r, 3)
        with torch.cuda.stream(h.stream):
            h.classify(rec["ts"][lo:hi], rec["src"][lo:hi], rec["dst"][lo:hi], rec["bytes"][lo:hi])
    th = [threading.Thread(target=h.reduce, daemon=True) for h in hs]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    torch.cuda.synchronize()
    _check_owned(S, hs, o, wl)
    for h in hs:
        h.close()
