"""B200-native ParaMaP mapping-and-planning hot path.

Drop-in for the reference package's hot path (vp/mapping.py occupancy fusion,
exact EDT and distance query; vp/planner.py / vp/batch.py SMPC rollout,
softmin and weighted update) running as hand-written sm_100a CUDA kernels
behind the C ABI in include/vpb200.h.  There is no CPU fallback.
"""

__version__ = "0.1.0"

from .errors import (  # noqa: F401
    DegenerateRotation,
    DimensionMismatch,
    FrameMismatch,
    VolumeOutOfBounds,
    WeightMismatch,
)


def library_path():
    from ._lib import LIB_PATH

    return LIB_PATH
