"""B200-native replay engine for the AMPD (arXiv 2602.14516) plan search.

The hot path — replaying every (candidate deployment, trace replica) pair
through the reference simulator's cost model, adaptive incremental-prefill
routing, prefill-queue reordering and TTFT/ITL SLO scoring, then taking the
argmax plan — runs as hand-written CUDA for sm_100a behind the C-ABI in
include/pdsim_gpu.h (library: libpdsim_gpu.so). Python here is a ctypes
mirror of that ABI; see DESIGN.md.
"""
from . import abi  # noqa: F401

__all__ = ["abi", "native", "workloads"]
