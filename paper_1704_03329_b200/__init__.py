"""B200-native Lennard-Jones PairLoop engine (hot path of arXiv 1704.03329, PPMD).

The compute path is libljmd.so (hand-written sm_100a CUDA behind the C ABI in
include/ljmd.h); this package only builds it and marshals arguments.
"""
from .ljmd import LJMD, LjmdError, Options, default_options, load, plan_cells, plan_slab, version  # noqa: F401

__all__ = ["LJMD", "LjmdError", "Options", "default_options", "load", "plan_cells", "plan_slab", "version"]
