"""World-size-2 CPU test (gloo) of the multi-GPU host logic: contiguous record
shards (P:L189 one chunk per GPU thread), per-rank partial histograms, the
additive merge (merge-scatter: associative + commutative) and the
per-rank owned bin ranges the NCCL reduce-scatter leaves behind.  The partial
histograms come from the oracle (the GPU path is covered by -m gpu tests)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

M64 = (1 << 64) - 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import core as oracle
    from paper_2106_12863_b200.histogram import owned_bin_range, shard_range
    from synth import WORKLOADS, prefix_table, records
    from synth.sinet_synth import stream_order, to_numpy

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    wl = WORKLOADS["c1"].with_(n=120_001)
    nets, lens = prefix_table(wl)
    order = stream_order(wl, "cpu")
    lo, hi = shard_range(wl.n, rank, world)
    cols = to_numpy(records(wl, lo, hi, order=order))
    part = oracle.classify_histogram(*cols, nets, lens, wl.window_start_ms, wl.window_ms, 1)
    # merge: u64 sums as int64 two's complement (wraps identically mod 2^64)
    flat = torch.from_numpy(np.concatenate([part.count.ravel(), part.bytes.ravel(), part.totals]).view(np.int64))
    dist.all_reduce(flat)
    merged = flat.numpy().view(np.uint64)
    B = wl.nbins
    cnt = merged[:2 * B].reshape(2, B)
    byt = merged[2 * B:4 * B].reshape(2, B)
    tot = merged[4 * B:]
    olo, ohi = owned_bin_range(B, rank, world)   # the library's tile (sinet_tile_bins)
    full = oracle.classify_histogram(*to_numpy(records(wl, order=order)), nets, lens, wl.window_start_ms,
                                     wl.window_ms, 1)
    ok = (np.array_equal(cnt[:, olo:ohi], full.count[:, olo:ohi]) and
          np.array_equal(byt[:, olo:ohi], full.bytes[:, olo:ohi]) and np.array_equal(tot, full.totals))
    sizes = torch.tensor([ohi - olo, hi - lo])
    dist.all_reduce(sizes)
    ok = ok and int(sizes[0]) == B and int(sizes[1]) == wl.n
    out[rank] = bool(ok)
    dist.destroy_process_group()


def test_two_rank_shard_merge_matches_single_oracle():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    assert all(p.exitcode == 0 for p in procs)
    assert out[0] and out[1]


def _sparse_worker(rank, world, port, out, order):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import core as oracle
    from paper_2106_12863_b200 import exchange_plan, owned_bin_range, padded_bins, shard_range
    from synth import WORKLOADS, prefix_table, records
    from synth.sinet_synth import stream_order, to_numpy

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    wl = WORKLOADS["c1"].with_(n=90_001, order=order)
    nets, lens = prefix_table(wl)
    so = stream_order(wl, "cpu")
    lo, hi = shard_range(wl.n, rank, world)
    part = oracle.classify_histogram(*to_numpy(records(wl, lo, hi, order=so)), nets, lens, wl.window_start_ms,
                                     wl.window_ms, 1)
    B = wl.nbins
    Bp = padded_bins(B, world, 256)
    # the bins buffer layout: [bin][dir][metric]
    mine = np.zeros((Bp, 4), np.uint64)
    mine[:B, 0], mine[:B, 1], mine[:B, 2], mine[:B, 3] = part.count[0], part.bytes[0], part.count[1], part.bytes[1]
    nz = np.nonzero((part.count[0] + part.count[1]) > 0)[0]
    t = torch.tensor([int(nz.min()), int(nz.max())] if len(nz) else [0xFFFFFFFF, 0], dtype=torch.int64)
    allt = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allt, t)
    touched = np.array([x.tolist() for x in allt], dtype=np.uint32)
    send, recv = exchange_plan(world, rank, B, Bp, touched)
    # the exchange: isend my slices, recv the others' into staging, then add into my owned range
    reqs = []
    for o in range(world):
        f, n = send[o]
        if n:
            reqs.append(dist.isend(torch.from_numpy(mine[f:f + n].view(np.int64).copy()), dst=o))
    olo, ohi = owned_bin_range(B, rank, world)
    result = mine[olo:ohi].copy()
    for r in range(world):
        f, n = recv[r]
        if n:
            buf = torch.zeros((n, 4), dtype=torch.int64)
            dist.recv(buf, src=r)
            assert olo <= f and f + n <= ohi
            result[f - olo:f - olo + n] += buf.numpy().view(np.uint64)
    for q in reqs:
        q.wait()
    full = oracle.classify_histogram(*to_numpy(records(wl, order=so)), nets, lens, wl.window_start_ms, wl.window_ms, 1)
    ok = (np.array_equal(result[:, 0], full.count[0][olo:ohi]) and np.array_equal(result[:, 1], full.bytes[0][olo:ohi])
          and np.array_equal(result[:, 2], full.count[1][olo:ohi]) and np.array_equal(result[:, 3], full.bytes[1][olo:ohi]))
    moved = int(recv[:, 1].sum())
    out[rank] = (bool(ok), moved)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,order", [(2, "stream"), (3, "stream"), (3, "shuffled")])
def test_sparse_exchange_plan_gives_global_sums(world, order):
    """The sparse touched-range exchange (the plan sinet_reduce executes with NCCL
    send/recv) leaves every owner the global sums; with contiguous time shards only
    the boundary overlaps move."""
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_sparse_worker, args=(r, world, port, out, order)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    assert all(p.exitcode == 0 for p in procs)
    assert all(out[r][0] for r in range(world))
    moved = sum(out[r][1] for r in range(world))
    if order == "stream":   # 1 h window split in `world` time slices: only ~2 s overlaps move
        assert moved < 3_600_000 // 20
