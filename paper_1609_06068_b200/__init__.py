"""B200-native hot path of the chordally decomposed ADMM for sparse SDPs
(arXiv 1609.06068).  The compute lives in libchordal_sdp.so (C ABI declared in
include/chordal_sdp.h); this package is its thin Python binding.

    from paper_1609_06068_b200 import Solver, PsdPlan, chordal_cliques
    from paper_1609_06068_b200.sdpa import read_sdpa   # SDPA sparse (.dat-s) input
"""
from ._lib import (EXPORTED, LIB_PATH, LoopbackGroup, PsdPlan, SdpError, Solver, TorchAllocator,  # noqa: F401
                   chordal_cliques, lib, nccl_unique_id, schur_inverse_host, shard_plan)

__all__ = ["Solver", "PsdPlan", "LoopbackGroup", "TorchAllocator", "chordal_cliques", "shard_plan", "nccl_unique_id", "SdpError", "lib", "LIB_PATH",
           "EXPORTED"]
