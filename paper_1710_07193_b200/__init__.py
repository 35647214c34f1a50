"""B200-native DCT-domain block filter (arXiv 1710.07193), sm_100a.

The hot path — mask -> dense DCT-domain operator, batched block DCT, the
DCT-domain filter contraction and the fused u8 -> u8 pipeline — runs in
hand-written CUDA (libdctf_b200.so, C ABI in include/dctf.h). This package is
the Python mirror of the reference's C++ API over that ABI.
"""
from . import _lib  # noqa: F401  (fails loudly if the CUDA library is missing)
from .dctfilter import (  # noqa: F401
    DctBasis, Domain, FilterPlan, InvalidArgument, Mask, MultiPlan, NanEncountered, PaddingMode, Precision,
    Unsupported,
    filter_frames, filter_frames_host, filter_image, format_operator_dump, forward_2d, inverse_2d,
    operator_from_dump, row_symmetric)

__version__ = _lib.lib.dctf_version().decode()
