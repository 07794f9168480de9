"""B200-native ADMM topology solver (hot path of arXiv 2512.07536 "BA-Topo").

The compute path is libtopoopt_b200.so (sm_100a CUDA + C ABI, see
include/topoopt_b200.h); ``topoopt`` mirrors the reference C++ API.
"""
from . import topoopt  # noqa: F401
from ._lib import LIB_PATH, load  # noqa: F401

__all__ = ["topoopt", "load", "LIB_PATH"]
