"""paper_1509_01149_b200 — B200-native MPPI (Williams, Aldrich & Theodorou, arXiv:1509.01149).

The hot path of one MPPI optimisation step in hand-written sm_100a CUDA kernels behind the
C ABI of include/mppi.h (libmppi_b200.so); this package is the thin Python binding.
"""
from ._capi import MppiError  # noqa: F401
from .mppi import MPPI, from_workload  # noqa: F401
from .dist import ShardedMPPI, shard_range  # noqa: F401
