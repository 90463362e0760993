"""B200-native SINET session discrimination + millisecond histogram (arXiv 2106.12863).

The hot path: discriminate every session record against the
SINET CIDR list (Alg. 1, subnet-mask AND + network-address match of src and
dst) fused with the per-ms count/bytes histogram (§4 map-reduce), merged
across GPUs by an NCCL reduce-scatter.  All of it runs in libsinet.so
(paper_2106_12863_b200/csrc, C ABI in include/sinet.h); this package is the
thin Python binding.
"""
from ._native import (  # noqa: F401
    DIR_IN, DIR_NEITHER, DIR_OUT, LUT_ALG1, LUT_SRC_PRIORITY, LUT_STRICT, METRIC_BYTES,
    METRIC_COUNT, ORDER_AUTO, ORDER_SHUFFLED, ORDER_STREAM, SinetError,
)
from .histogram import (  # noqa: F401
    SinetHistogram, SinetHub, exchange_plan, owned_bin_range, padded_bins, parse_text, shard_range, table_member_host,
)

__version__ = "0.1.0"
