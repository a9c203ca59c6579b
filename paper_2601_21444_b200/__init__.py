"""paper_2601_21444_b200 -- B200-native Spava sequence-parallel prefill attention.

The product is the C-ABI library ``libspava_b200.so`` (include/spava_b200.h) built
from ``csrc/`` for sm_100a.  This package only loads it and offers a Python mirror
of the reference's ``seqpar`` operator API (partition.hpp / approx.hpp /
attention.hpp) over torch device tensors, for tests and bench.py.  There is no CPU
fallback: every compute call goes through the CUDA library and raises if it (or an
sm_100 device) is missing.
"""
from .spava import *  # noqa: F401,F403
from .spava import __all__  # noqa: F401
