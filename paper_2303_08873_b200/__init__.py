"""B200-native model-building engine behind ML-driven adaptive OpenMP (arXiv 2303.08873).

The engine is ``libadapt.so`` (hand-written sm_100a CUDA behind the C ABI of
``include/adapt.h``); this package is its thin ctypes binding.  See DESIGN.md.
"""
from . import _binding
from ._binding import *  # noqa: F401,F403  (the adapt_* names of include/adapt.h)
from ._binding import (AdaptError, KFOLD_DTYPE, NODE_DTYPE, SYMBOLS, LIB_PATH, lib,  # noqa: F401
                       __adapt_region_begin, __adapt_region_create, __adapt_region_end,
                       __adapt_region_get_policy, __adapt_region_set_feature,
                       __adapt_region_train)

__all__ = [n for n in dir(_binding) if n.startswith("adapt_") or n.startswith("ADAPT_")]
