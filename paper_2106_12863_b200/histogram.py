"""User-facing Python API over libsinet (argument marshalling + torch-owned device memory).

Every step of the hot path runs in the CUDA library; this module only
allocates caller-owned buffers with torch, passes pointers and streams,
and converts results.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native as N
from ._native import check, lib

__all__ = ["SinetHistogram", "SinetHub", "shard_range", "owned_bin_range", "padded_bins"]


def shard_range(n: int, rank: int, world: int):
    """Contiguous record shard of rank `rank`: [rank*n//world, (rank+1)*n//world).

    One file chunk per GPU thread in the paper becomes one
    contiguous slice per rank."""
    return n * rank // world, n * (rank + 1) // world


def padded_bins(nbins: int, world: int, tile_bins: int | None = None) -> int:
    t = int(lib.sinet_tile_bins()) if tile_bins is None else tile_bins
    unit = world * t
    return (nbins + unit - 1) // unit * unit


def owned_bin_range(nbins: int, rank: int, world: int, tile_bins: int | None = None):
    """Bins rank `rank` holds after the reduce-scatter: [lo, hi) clipped to [0, nbins)."""
    per = padded_bins(nbins, world, tile_bins) // world
    lo, hi = min(per * rank, nbins), min(per * (rank + 1), nbins)
    return lo, hi


def _ptr(t: torch.Tensor | None):
    return ctypes.c_void_p(t.data_ptr() if t is not None else 0)


class SinetHub:
    """In-process rendezvous of `world` ranks (one host thread per GPU): ctxs that
    join it merge through peer memory instead of NCCL (sinet_hub_create).  Keep it alive
    while any joined SinetHistogram is open."""

    def __init__(self, world: int):
        h = ctypes.c_void_p()
        check(lib.sinet_hub_create(ctypes.byref(h), int(world)), None, "hub_create")
        self.handle, self.world = h, int(world)

    def close(self):
        if getattr(self, "handle", None):
            lib.sinet_hub_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class SinetHistogram:
    """One per (process, GPU): the compiled CIDR list, the bins and the totals.

    nets/lens: the CIDR list (Y.Y.Y.Y as u32, Z), Alg. 1 l.1,4.
    Bins: u64 [B_pad][2 dir][2 metric], one 32-byte sector per ms bin.
    """

    def __init__(self, nets, lens, window_start_ms: int, window_ms: int, bin_width_ms: int = 1,
                 lut=N.LUT_SRC_PRIORITY, device=None, rank: int = 0, world: int = 1,
                 stream: torch.cuda.Stream | None = None, order: int = N.ORDER_AUTO, labels=None):
        if not torch.cuda.is_available():
            raise RuntimeError("SinetHistogram needs a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else int(device))
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        cfg = N.Config()
        cfg.window_start_ms = int(window_start_ms)
        cfg.window_ms = int(window_ms)
        cfg.bin_width_ms = int(bin_width_ms)
        for k in range(4):
            cfg.dir_lut[k] = int(lut[k])
        cfg.device = self.device.index
        cfg.rank, cfg.world = int(rank), int(world)
        cfg.stream = ctypes.c_void_p(self.stream.cuda_stream)
        cfg.order_hint = int(order)
        self.cfg = cfg
        self.nbins = int(window_ms) // int(bin_width_ms)
        self.rank, self.world = int(rank), int(world)
        nets = np.ascontiguousarray(np.asarray(nets, dtype=np.uint32))
        lens = np.ascontiguousarray(np.asarray(lens, dtype=np.uint8))
        bb = lib.sinet_bins_bytes(ctypes.byref(cfg))
        wb = lib.sinet_workspace_bytes(ctypes.byref(cfg), len(nets))
        if bb == 0 or wb == 0:
            raise N.SinetError(N.E_INVAL, "invalid configuration or prefix count")
        self.B_pad = bb // 32
        with torch.cuda.device(self.device):
            self.bins = torch.empty(bb // 8, dtype=torch.int64, device=self.device)
            self.ws = torch.empty(wb, dtype=torch.uint8, device=self.device)
        ctx = ctypes.c_void_p()
        if labels is not None:   # NEXT-4: labelled longest-prefix match
            labs = np.ascontiguousarray(np.asarray(labels, dtype=np.uint8))
            assert labs.shape == nets.shape
            lab_p = labs.ctypes.data_as(ctypes.c_void_p)
        else:
            lab_p = None
        rc = lib.sinet_open_labelled(ctypes.byref(ctx), ctypes.byref(cfg), nets.ctypes.data_as(ctypes.c_void_p),
                                     lens.ctypes.data_as(ctypes.c_void_p), lab_p, len(nets), _ptr(self.bins), bb,
                                     _ptr(self.ws), wb)
        check(rc, None, "sinet_open")
        self.ctx = ctx
        self._staging = None

    # ------------------------------------------------------------------ lifecycle
    def close(self):
        if getattr(self, "ctx", None):
            lib.sinet_close(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def reset(self):
        check(lib.sinet_reset(self.ctx), self.ctx, "reset")

    # ------------------------------------------------------------------ hot path
    @staticmethod
    def _records(ts, src, dst, nbytes):
        n = ts.numel()
        assert src.numel() == n and dst.numel() == n and nbytes.numel() == n
        assert ts.element_size() == 8 and nbytes.element_size() == 8
        assert src.element_size() == 4 and dst.element_size() == 4
        for t in (ts, src, dst, nbytes):
            assert t.is_contiguous()
        return N.Records(ts.data_ptr(), src.data_ptr(), dst.data_ptr(), nbytes.data_ptr(), n)

    def classify(self, ts, src, dst, nbytes, tags: torch.Tensor | None = None):
        """Accumulate one batch of device-resident records (int64/int32 bit patterns)."""
        for t in (ts, src, dst, nbytes):
            assert t.device == self.device, "records must live on the ctx device"
        recs = self._records(ts, src, dst, nbytes)
        if tags is not None:
            assert tags.dtype == torch.uint8 and tags.numel() >= ts.numel() and tags.device == self.device
        check(lib.sinet_classify_histogram(self.ctx, ctypes.byref(recs), _ptr(tags)), self.ctx, "classify")

    def classify_host(self, ts, src, dst, nbytes, chunk_records: int = 1 << 24):
        """Accumulate host (ideally pinned) records, streamed through a device staging buffer."""
        for t in (ts, src, dst, nbytes):
            assert t.device.type == "cpu"
        need = lib.sinet_staging_bytes(chunk_records)
        if self._staging is None or self._staging.numel() < need:
            self._staging = torch.empty(need, dtype=torch.uint8, device=self.device)
        recs = self._records(ts, src, dst, nbytes)
        check(lib.sinet_classify_histogram_host(self.ctx, ctypes.byref(recs), _ptr(self._staging), need,
                                                chunk_records), self.ctx, "classify_host")

    def classify_sortreduce(self, ts, src, dst, nbytes, scratch: torch.Tensor | None = None):
        """NEXT-4 comparator: the paper's sort + reduce_by_key design (CUB), same result as classify()."""
        recs = self._records(ts, src, dst, nbytes)
        need = lib.sinet_sortreduce_scratch_bytes(ctypes.byref(self.cfg), recs.n)
        if scratch is None or scratch.numel() < need:
            scratch = torch.empty(max(need, 1), dtype=torch.uint8, device=self.device)
        check(lib.sinet_classify_histogram_sortreduce(self.ctx, ctypes.byref(recs), _ptr(scratch), need),
              self.ctx, "classify_sortreduce")
        return scratch

    def set_scratch(self, max_records: int | None = 1 << 27):
        """Register device scratch for unordered batches (partition then bin, sub-batches of
        `max_records`; ~24 B/record).  None removes it (unordered batches then take L2 atomics)."""
        if max_records is None:
            check(lib.sinet_set_scratch(self.ctx, None, 0), self.ctx, "set_scratch")
            self._scratch = None
            return
        need = lib.sinet_partition_scratch_bytes(ctypes.byref(self.cfg), int(max_records))
        if need == 0:
            raise N.SinetError(N.E_INVAL, "partitioned path unsupported for this window (> 2^27 bins) or size")
        self._scratch = torch.empty(need + 256, dtype=torch.uint8, device=self.device)
        off = (-self._scratch.data_ptr()) % 256
        check(lib.sinet_set_scratch(self.ctx, ctypes.c_void_p(self._scratch.data_ptr() + off), need), self.ctx,
              "set_scratch")

    def set_watchlist(self, ips):
        """NEXT-2: count only records with a listed source or destination (None/[] removes it)."""
        ips = np.ascontiguousarray(np.asarray([] if ips is None else ips, dtype=np.uint32))
        n = len(ips)
        if n == 0:
            check(lib.sinet_set_watchlist(self.ctx, None, 0, None, 0), self.ctx, "set_watchlist")
            self._watch = None
            return
        need = lib.sinet_watchlist_bytes(n)
        self._watch = torch.empty(need, dtype=torch.uint8, device=self.device)
        check(lib.sinet_set_watchlist(self.ctx, ips.ctypes.data_as(ctypes.c_void_p), n, _ptr(self._watch), need),
              self.ctx, "set_watchlist")

    def finalize(self):
        check(lib.sinet_finalize(self.ctx), self.ctx, "finalize")

    # ------------------------------------------------------------------ multi-GPU
    @staticmethod
    def new_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        check(lib.sinet_nccl_unique_id(buf), None, "nccl unique id")
        return buf.raw

    def comm_init(self, unique_id: bytes):
        assert len(unique_id) == 128
        buf = ctypes.create_string_buffer(unique_id, 128)
        check(lib.sinet_comm_init(self.ctx, buf), self.ctx, "comm_init")

    def comm_init_from_group(self, group=None):
        """Rank 0 creates the NCCL id; torch.distributed broadcasts it (plumbing only)."""
        import torch.distributed as dist
        obj = [self.new_unique_id() if self.rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        self.comm_init(obj[0])

    def comm_init_hub(self, hub: "SinetHub"):
        """Join an in-process hub (this ctx's rank/world must match it)."""
        assert hub.world == self.world
        check(lib.sinet_comm_init_hub(self.ctx, hub.handle), self.ctx, "comm_init_hub")
        self._hub = hub   # keep the hub alive at least as long as this ctx

    def reduce(self):
        check(lib.sinet_reduce(self.ctx), self.ctx, "reduce")

    def set_exchange(self, mode: int):
        """Multi-GPU merge: 0 auto, 1 dense reduce-scatter, 2 sparse touched-range exchange."""
        check(lib.sinet_set_exchange(self.ctx, mode), self.ctx, "set_exchange")

    def touched_range(self):
        """(min bin, max bin) written since the last reset; min > max if none."""
        a, b = ctypes.c_uint32(), ctypes.c_uint32()
        check(lib.sinet_touched_range(self.ctx, ctypes.byref(a), ctypes.byref(b)), self.ctx, "touched_range")
        return a.value, b.value

    @property
    def last_exchange(self) -> int:
        return int(lib.sinet_last_exchange(self.ctx))

    def owned_range(self):
        lo, n = ctypes.c_uint64(), ctypes.c_uint64()
        check(lib.sinet_owned_range(self.ctx, ctypes.byref(lo), ctypes.byref(n)), self.ctx, "owned_range")
        return lo.value, lo.value + n.value

    # ------------------------------------------------------------------ read-out
    def _take_over(self):
        """Buffers the caller allocated on its current stream: the ctx stream waits for it first."""
        cur = torch.cuda.current_stream(self.device)
        if cur != self.stream:
            self.stream.wait_stream(cur)

    def _hand_over(self, *tensors):
        """Device results written on the ctx stream: the caller's current stream waits for it,
        and the caching allocator keeps the buffers until the ctx stream is done with them."""
        cur = torch.cuda.current_stream(self.device)
        if cur != self.stream:
            cur.wait_stream(self.stream)
            for t in tensors:
                if t is not None and t.is_cuda:
                    t.record_stream(self.stream)

    def read_bins(self, direction: int, metric: int, first: int | None = None, n: int | None = None,
                  device: bool = False):
        """u64 plane slice [first, first + n) (default: the whole owned range) as numpy uint64
        (host) or a torch int64 tensor (device)."""
        lo, hi = self.owned_range()
        if first is None:
            first = lo
        if n is None:
            n = hi - first
        if device:
            out = torch.empty(n, dtype=torch.int64, device=self.device)
            self._take_over()
            ptr = _ptr(out)
        else:
            out = np.empty(n, dtype=np.uint64)
            ptr = out.ctypes.data_as(ctypes.c_void_p)
        check(lib.sinet_read_bins(self.ctx, direction, metric, first, n, ptr, 1 if device else 0),
              self.ctx, "read_bins")
        if device:
            self._hand_over(out)
        return out

    def read_bins_raw(self, out: torch.Tensor | None = None, first: int | None = None, n: int | None = None):
        """Owned bins [first, first + n) in the native layout, int64[n, 2 dir, 2 metric], copied with one
        sinet_read_bins_raw call into `out` (a device tensor, or a host tensor -- pinned for full speed)."""
        lo, hi = self.owned_range()
        first = lo if first is None else int(first)
        n = hi - first if n is None else int(n)
        if out is None:
            out = torch.empty((n, 2, 2), dtype=torch.int64)
        assert out.dtype == torch.int64 and out.is_contiguous() and out.numel() >= 4 * n
        dev = out.device.type == "cuda"
        if dev:
            self._take_over()
        check(lib.sinet_read_bins_raw(self.ctx, first, n, _ptr(out), 1 if dev else 0), self.ctx, "read_bins_raw")
        if dev:
            self._hand_over(out)
        return out

    def rebin_frames(self, factor: int):
        """(first frame, number of frames) the owned range meets; frame F = bins [F*factor, (F+1)*factor)."""
        f0, nf = ctypes.c_uint64(), ctypes.c_uint64()
        check(lib.sinet_rebin_frames(self.ctx, int(factor), ctypes.byref(f0), ctypes.byref(nf)), self.ctx,
              "rebin_frames")
        return f0.value, nf.value

    def rebin(self, factor: int) -> torch.Tensor:
        """Coarser frames (NEXT-1): int64[n_frames, 2 dir, 2 metric] on the device, entry k = the
        owned bins of frame rebin_frames()[0] + k (frames aligned to the window start)."""
        _, n_out = self.rebin_frames(factor)
        out = torch.empty((max(n_out, 1), 2, 2), dtype=torch.int64, device=self.device)
        self._take_over()
        check(lib.sinet_rebin(self.ctx, int(factor), _ptr(out), n_out), self.ctx, "rebin")
        self._hand_over(out)
        return out[:n_out]

    def set_knob(self, name: str, value: int):
        """Named performance knob of the library (results identical for every value)."""
        check(lib.sinet_set_knob(self.ctx, name.encode(), int(value)), self.ctx, "set_knob")

    def export_sparse(self, direction: int, capacity: int | None = None):
        """(bin start ms, count, bytes) of every nonzero-count bin of `direction`, ascending (NEXT-1)."""
        n = ctypes.c_uint64()
        if capacity is None:
            check(lib.sinet_export_sparse(self.ctx, direction, None, None, None, 0, ctypes.byref(n)),
                  self.ctx, "export_sparse")
            capacity = n.value
        bufs = [torch.empty(max(capacity, 1), dtype=torch.int64, device=self.device) for _ in range(3)]
        self._take_over()
        check(lib.sinet_export_sparse(self.ctx, direction, _ptr(bufs[0]), _ptr(bufs[1]), _ptr(bufs[2]), capacity,
                                      ctypes.byref(n)), self.ctx, "export_sparse")
        self._hand_over(*bufs)
        k = min(n.value, capacity)
        return tuple(b[:k] for b in bufs), n.value

    def read_totals(self) -> np.ndarray:
        """12 x u64: m_count[4], m_bytes[4], oow_count[2], oow_bytes[2] (oracle layout)."""
        t = N.Totals()
        check(lib.sinet_read_totals(self.ctx, ctypes.byref(t)), self.ctx, "read_totals")
        return np.array(list(t.m_count) + list(t.m_bytes) + list(t.oow_count) + list(t.oow_bytes),
                        dtype=np.uint64)

    def bins_view(self) -> torch.Tensor:
        """Device view int64[B_pad, 2, 2] of the bins buffer (after finalize/reduce)."""
        return self.bins.view(self.B_pad, 2, 2)

    # ------------------------------------------------------------------ introspection
    @property
    def launches(self) -> int:
        return int(lib.sinet_launch_count(self.ctx))

    @property
    def last_strategy(self) -> int:
        return int(lib.sinet_last_strategy(self.ctx))

    @property
    def last_kernel(self) -> str:
        return lib.sinet_last_kernel(self.ctx).decode()

    def set_tuning(self, stream_groups: int = 0, warp_aggregation: int = -1):
        """Stream-kernel layout (0 auto / 1 / 2 groups) and warp aggregation (1/0, -1 unchanged)."""
        check(lib.sinet_set_tuning(self.ctx, stream_groups, warp_aggregation), self.ctx, "set_tuning")

    def set_table_mode(self, mode: int = -1):
        """Stream-kernel lookup-table encoding: -1 auto, 0 byte, 1 packed, 2 packed w/o level 2, 3 global."""
        check(lib.sinet_set_table_mode(self.ctx, mode), self.ctx, "set_table_mode")

    @property
    def table_mode(self) -> int:
        return int(lib.sinet_table_mode(self.ctx))

    def set_kernel_timing(self, on: bool):
        check(lib.sinet_set_kernel_timing(self.ctx, 1 if on else 0), self.ctx, "timing")

    def kernel_time(self):
        ms, k = ctypes.c_double(), ctypes.c_uint64()
        check(lib.sinet_kernel_time(self.ctx, ctypes.byref(ms), ctypes.byref(k)), self.ctx, "kernel_time")
        return ms.value, k.value


def exchange_plan(world: int, rank: int, nbins: int, nbins_pad: int, touched):
    """Host plan of the sparse multi-GPU exchange: (send, recv) int arrays [world, 2] of (first bin, count)."""
    t = np.ascontiguousarray(np.asarray(touched, dtype=np.uint32).reshape(world * 2))
    send = np.zeros(world * 2, np.uint64)
    recv = np.zeros(world * 2, np.uint64)
    check(lib.sinet_exchange_plan(world, rank, nbins, nbins_pad, t.ctypes.data_as(ctypes.c_void_p),
                                  send.ctypes.data_as(ctypes.c_void_p), recv.ctypes.data_as(ctypes.c_void_p)),
          None, "exchange_plan")
    return send.reshape(world, 2).astype(np.int64), recv.reshape(world, 2).astype(np.int64)


def table_member_host(nets, lens, ips, labels=None) -> np.ndarray:
    """Host evaluation of the compiled lookup table (prefix compiler check, no GPU)."""
    nets = np.ascontiguousarray(np.asarray(nets, dtype=np.uint32))
    lens = np.ascontiguousarray(np.asarray(lens, dtype=np.uint8))
    ips = np.ascontiguousarray(np.asarray(ips, dtype=np.uint32))
    out = np.empty(len(ips), dtype=np.uint8)
    labs = None if labels is None else np.ascontiguousarray(np.asarray(labels, dtype=np.uint8))
    rc = lib.sinet_table_member_host_labelled(
        nets.ctypes.data_as(ctypes.c_void_p), lens.ctypes.data_as(ctypes.c_void_p),
        None if labs is None else labs.ctypes.data_as(ctypes.c_void_p), len(nets),
        ips.ctypes.data_as(ctypes.c_void_p), len(ips), out.ctypes.data_as(ctypes.c_void_p))
    check(rc, None, "table_member_host")
    return out


def parse_text(text: torch.Tensor, tz_offset_min: int = 0, capacity: int | None = None,
               status: bool = False, out: dict | None = None, workspace: torch.Tensor | None = None):
    """NEXT-3: PA-7080 session-log text (uint8 CUDA tensor, Table 1 lines) -> device columns.

    Marshals sinet_parse_text: returns (columns dict {ts, src, dst, bytes} of the valid lines
    in line order, trimmed to the valid count; per-line status uint8 tensor or None;
    the result counts as a dict).  Every step runs in libsinet.so.
    """
    assert text.is_cuda and text.dtype == torch.uint8 and text.is_contiguous()
    n = text.numel()
    dev = text.device
    if capacity is None:
        capacity = n // 62 + 1            # a valid line has >= 61 bytes + its newline
    if out is None:
        out = {"ts": torch.empty(capacity, dtype=torch.int64, device=dev),
               "src": torch.empty(capacity, dtype=torch.int32, device=dev),
               "dst": torch.empty(capacity, dtype=torch.int32, device=dev),
               "bytes": torch.empty(capacity, dtype=torch.int64, device=dev)}
    capacity = out["ts"].numel()
    cols = N.Columns(_ptr(out["ts"]), _ptr(out["src"]), _ptr(out["dst"]), _ptr(out["bytes"]), capacity)
    st = torch.empty(n + 1, dtype=torch.uint8, device=dev) if status else None
    wsb = N.lib.sinet_parse_workspace_bytes(n)
    if workspace is None or workspace.numel() < wsb:
        workspace = torch.empty(wsb, dtype=torch.uint8, device=dev)
    res = N.ParseResult()
    stream = torch.cuda.current_stream(dev).cuda_stream
    rc = N.lib.sinet_parse_text(_ptr(text), n, tz_offset_min, ctypes.byref(cols), _ptr(st), st.numel() if st is not None else 0,
                                _ptr(workspace), workspace.numel(), stream, ctypes.byref(res))
    if rc != N.OK:
        raise N.SinetError(rc, "parse_text: " + N.lib.sinet_parse_last_error().decode())
    v = res.valid
    cols_out = {k: t[:v] for k, t in out.items()}
    info = {"lines": res.lines, "valid": v, "first_bad_line": res.first_bad_line,
            "by_status": list(res.by_status)}
    return cols_out, (st[:res.lines] if st is not None else None), info
