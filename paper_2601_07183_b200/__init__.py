"""paper_2601_07183_b200 -- B200-native RAIRS search hot path (arXiv 2601.07183).

Batched k-NN over an IVF-PQ 4-bit fast-scan index with exact refine, RAIR
(AIR) redundant assignment and cell-major SEIL shared-cell lists. All compute
runs in librairs.so (hand-written sm_100a CUDA behind the C ABI in
include/rairs.h); this package only marshals arguments. There is no CPU
fallback: importing the binding fails if the library is missing.
"""
from ._lib import EXPORTED_SYMBOLS, LIB_PATH, RairsError, build_library, lib  # noqa: F401
from .index import Index, build_index, exact_knn, merge_topk, train  # noqa: F401

lib()  # load librairs.so now: no silent fallback if the CUDA library is missing

__all__ = ["Index", "build_index", "train", "merge_topk", "exact_knn", "build_library",
           "RairsError", "LIB_PATH", "EXPORTED_SYMBOLS"]
