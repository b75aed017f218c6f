"""B200-native (sm_100a) activation outlier-attribution pass of arXiv 2603.10444
(mean/spike/tail decomposition + top-0.1% rho attribution).

The compute lives in libavd.so (hand-written CUDA behind the C ABI of include/avd.h);
this package is a thin binding.  There is no CPU fallback.
"""
from .api import Decomposer, Result, decompose  # noqa: F401

__all__ = ["Decomposer", "Result", "decompose"]
