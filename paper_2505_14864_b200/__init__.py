"""B200-native DynMo per-step rebalancing hot path (arXiv 2505.14864).

The product is ``libdynmo.so`` (C-ABI in ``include/dynmo.h``; CUDA kernels for
sm_100a in ``csrc/``).  ``paper_2505_14864_b200.dynmo`` is the thin Python
binding with the same call names.
"""
from . import _lib  # noqa: F401

__version__ = "0.1.0"
