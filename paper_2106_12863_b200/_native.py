"""ctypes binding of libsinet.so (include/sinet.h).  Argument marshalling only.

The product path has no CPU fallback: if the CUDA library is missing this
module raises at import time.
"""
from __future__ import annotations

import ctypes
import os
import re

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libsinet.so")
HEADER = os.path.join(os.path.dirname(_PKG), "include", "sinet.h")

if not os.path.exists(LIB_PATH) or os.environ.get("SINET_REBUILD") == "1":
    # Compile the CUDA library in-tree (nvcc, sm_100a); never substitute anything for it.
    from . import _build
    try:
        _build.build()
    except Exception as e:  # noqa: BLE001
        raise ImportError(f"libsinet.so not built at {LIB_PATH} and nvcc build failed ({e}): "
                          "run `python -c 'import __graft_entry__ as g; g.build()'`") from e

# A/B experiments only: SINET_LIB_VARIANT=x loads libsinet.x.so (built by tools/build_variant.py)
_variant = os.environ.get("SINET_LIB_VARIANT")
lib = ctypes.CDLL(os.path.join(_PKG, f"libsinet.{_variant}.so") if _variant else LIB_PATH)

OK, E_INVAL, E_ALIGN, E_RANGE, E_CUDA, E_NCCL, E_STATE = 0, -1, -2, -3, -4, -5, -6
ERR_NAMES = {E_INVAL: "E_INVAL", E_ALIGN: "E_ALIGN", E_RANGE: "E_RANGE", E_CUDA: "E_CUDA",
             E_NCCL: "E_NCCL", E_STATE: "E_STATE"}
DIR_OUT, DIR_IN, DIR_NEITHER = 0, 1, 2
METRIC_COUNT, METRIC_BYTES = 0, 1
ORDER_AUTO, ORDER_STREAM, ORDER_SHUFFLED = 0, 1, 2
LUT_SRC_PRIORITY = (DIR_NEITHER, DIR_IN, DIR_OUT, DIR_OUT)
LUT_ALG1 = (DIR_IN, DIR_IN, DIR_OUT, DIR_OUT)
LUT_STRICT = (DIR_NEITHER, DIR_IN, DIR_OUT, DIR_NEITHER)


class Records(ctypes.Structure):
    _fields_ = [("ts_ms", ctypes.c_void_p), ("src", ctypes.c_void_p), ("dst", ctypes.c_void_p),
                ("bytes", ctypes.c_void_p), ("n", ctypes.c_uint64)]


class Config(ctypes.Structure):
    _fields_ = [("window_start_ms", ctypes.c_uint64), ("window_ms", ctypes.c_uint64),
                ("bin_width_ms", ctypes.c_uint32), ("dir_lut", ctypes.c_uint8 * 4),
                ("device", ctypes.c_int32), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("stream", ctypes.c_void_p), ("order_hint", ctypes.c_uint32),
                ("reserved", ctypes.c_uint32 * 7)]


class Totals(ctypes.Structure):
    _fields_ = [("m_count", ctypes.c_uint64 * 4), ("m_bytes", ctypes.c_uint64 * 4),
                ("oow_count", ctypes.c_uint64 * 2), ("oow_bytes", ctypes.c_uint64 * 2)]


class Columns(ctypes.Structure):
    _fields_ = [("ts_ms", ctypes.c_void_p), ("src", ctypes.c_void_p), ("dst", ctypes.c_void_p),
                ("bytes", ctypes.c_void_p), ("capacity", ctypes.c_uint64)]


class ParseResult(ctypes.Structure):
    _fields_ = [("lines", ctypes.c_uint64), ("valid", ctypes.c_uint64), ("first_bad_line", ctypes.c_uint64),
                ("by_status", ctypes.c_uint64 * 7)]


LINE_OK, LINE_LONG, LINE_COLUMNS, LINE_TIME, LINE_SRC, LINE_DST, LINE_BYTES = range(7)

_vp, _u64, _u32, _i = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
_CP = ctypes.POINTER(Config)
_SIGS = {
    "sinet_abi_version": ([], _i),
    "sinet_tile_bins": ([], _u32),
    "sinet_parse_chunk_bytes": ([], _u32),
    "sinet_bins_bytes": ([_CP], ctypes.c_size_t),
    "sinet_workspace_bytes": ([_CP, _u32], ctypes.c_size_t),
    "sinet_staging_bytes": ([_u64], ctypes.c_size_t),
    "sinet_open": ([ctypes.POINTER(_vp), _CP, _vp, _vp, _u32, _vp, ctypes.c_size_t, _vp, ctypes.c_size_t], _i),
    "sinet_open_labelled": ([ctypes.POINTER(_vp), _CP, _vp, _vp, _vp, _u32, _vp, ctypes.c_size_t, _vp, ctypes.c_size_t], _i),
    "sinet_close": ([_vp], None),
    "sinet_reset": ([_vp], _i),
    "sinet_classify_histogram": ([_vp, ctypes.POINTER(Records), _vp], _i),
    "sinet_classify_histogram_host": ([_vp, ctypes.POINTER(Records), _vp, ctypes.c_size_t, _u64], _i),
    "sinet_finalize": ([_vp], _i),
    "sinet_comm_init": ([_vp, _vp], _i),
    "sinet_nccl_unique_id": ([_vp], _i),
    "sinet_reduce": ([_vp], _i),
    "sinet_owned_range": ([_vp, ctypes.POINTER(_u64), ctypes.POINTER(_u64)], _i),
    "sinet_read_bins": ([_vp, _i, _i, _u64, _u64, _vp, _i], _i),
    "sinet_read_bins_raw": ([_vp, _u64, _u64, _vp, _i], _i),
    "sinet_read_totals": ([_vp, ctypes.POINTER(Totals)], _i),
    "sinet_rebin": ([_vp, _u64, _vp, _u64], _i),
    "sinet_rebin_frames": ([_vp, _u64, ctypes.POINTER(_u64), ctypes.POINTER(_u64)], _i),
    "sinet_hub_create": ([ctypes.POINTER(_vp), ctypes.c_int32], _i),
    "sinet_hub_destroy": ([_vp], None),
    "sinet_comm_init_hub": ([_vp, _vp], _i),
    "sinet_set_knob": ([_vp, ctypes.c_char_p, ctypes.c_int64], _i),
    "sinet_sortreduce_scratch_bytes": ([_CP, _u64], ctypes.c_size_t),
    "sinet_partition_scratch_bytes": ([_CP, _u64], ctypes.c_size_t),
    "sinet_set_scratch": ([_vp, _vp, ctypes.c_size_t], _i),
    "sinet_classify_histogram_sortreduce": ([_vp, ctypes.POINTER(Records), _vp, ctypes.c_size_t], _i),
    "sinet_export_sparse": ([_vp, _i, _vp, _vp, _vp, _u64, ctypes.POINTER(_u64)], _i),
    "sinet_last_error": ([_vp], ctypes.c_char_p),
    "sinet_launch_count": ([_vp], _u64),
    "sinet_set_kernel_timing": ([_vp, _i], _i),
    "sinet_kernel_time": ([_vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_u64)], _i),
    "sinet_last_strategy": ([_vp], _i),
    "sinet_last_kernel": ([_vp], ctypes.c_char_p),
    "sinet_set_tuning": ([_vp, _i, _i], _i),
    "sinet_set_table_mode": ([_vp, _i], _i),
    "sinet_table_mode": ([_vp], _i),
    "sinet_watchlist_bytes": ([_u32], ctypes.c_size_t),
    "sinet_set_watchlist": ([_vp, _vp, _u32, _vp, ctypes.c_size_t], _i),
    "sinet_set_exchange": ([_vp, _i], _i),
    "sinet_last_exchange": ([_vp], _i),
    "sinet_touched_range": ([_vp, ctypes.POINTER(_u32), ctypes.POINTER(_u32)], _i),
    "sinet_exchange_plan": ([ctypes.c_int32, ctypes.c_int32, _u64, _u64, _vp, _vp, _vp], _i),
    "sinet_table_member_host": ([_vp, _vp, _u32, _vp, _u64, _vp], _i),
    "sinet_parse_workspace_bytes": ([_u64], ctypes.c_size_t),
    "sinet_parse_text": ([_vp, _u64, ctypes.c_int32, ctypes.POINTER(Columns), _vp, _u64, _vp, ctypes.c_size_t, _vp,
                          ctypes.POINTER(ParseResult)], _i),
    "sinet_parse_last_error": ([], ctypes.c_char_p),
    "sinet_parse_set_knob": ([ctypes.c_char_p, ctypes.c_int64], _i),
    "sinet_table_member_host_labelled": ([_vp, _vp, _vp, _u32, _vp, _u64, _vp], _i),
}
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _res


def _header_abi_version() -> int:
    with open(HEADER) as f:
        m = re.search(r"#define\s+SINET_ABI_VERSION\s+(\d+)", f.read())
    return int(m.group(1)) if m else -1


if int(lib.sinet_abi_version()) != _header_abi_version():
    raise ImportError(f"{LIB_PATH} has ABI {int(lib.sinet_abi_version())} but include/sinet.h declares "
                      f"{_header_abi_version()}: the library is stale, rebuild it (__graft_entry__.build())")


def header_functions():
    """Names of every function declared in include/sinet.h."""
    with open(HEADER) as f:
        txt = re.sub(r"/\*.*?\*/", "", f.read(), flags=re.S)
    return sorted(set(re.findall(r"\b(sinet_[a-z0-9_]+)\s*\(", txt)))


class SinetError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERR_NAMES.get(code, code)}: {msg}")
        self.code = code


def check(rc, ctx=None, what=""):
    if rc != OK:
        msg = lib.sinet_last_error(ctx).decode() if ctx else ""
        raise SinetError(rc, f"{what}: {msg}" if what else msg)
    return rc
