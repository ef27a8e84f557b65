"""B200-native kNN-graph construction (SOLANET hot path, arxiv/paper_2605_27691).

partition -> lock-free local NN-Descent -> remote refine (NVLink pulls +
greedy beam search) -> binary-tree kNN-list merge -> graph output, as sm_100a
CUDA kernels behind the C-ABI in include/knng_c.h.  This package is the host
mirror of the reference API (knng.py); the compute lives in libknng_b200.so.
"""
from .knng import *  # noqa: F401,F403
from .knng import (KnnGraph, NnDescentParams, NnDescentStats, RefineConfig, SearchParams, lib,
                   context)  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
