"""B200-native segmented-decode serving for time-sensitive robotic agents (arxiv 2412.18695).

The product is the C-ABI library ``lib/librt_b200.so`` (sources in ``csrc/``,
header ``include/rt.h``); ``rt`` is its thin ctypes binding and ``metrics``
the host-side time-utility report of a segment log.
"""
from . import rt  # noqa: F401
from .rt import Engine  # noqa: F401
