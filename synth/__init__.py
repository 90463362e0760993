"""Seeded synthetic SINET-shaped workloads (shared input generator).

This package is the ONLY code shared by the oracle side (tests) and the CUDA
side (bench, parity tests).  It holds none of the method's arithmetic: no
membership test, no direction rule, no binning -- only counter-based random
draws shaped like the paper's workloads.
"""
from .sinet_synth import (  # noqa: F401
    WORKLOADS, Workload, prefix_table, records, window_of, SEED_BASE,
)
