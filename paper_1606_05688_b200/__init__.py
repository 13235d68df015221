"""B200-native sliding-window 3D ConvNet inference (the ZNNi hot path).

Layer primitives, transforms and the network forward run as hand-written
sm_100a CUDA kernels in libvxg.so (C-ABI: include/vxg.h); this package is the
Python mirror of the reference's interface (see voxin.py).  There is no CPU
fallback: without the built library the import fails.
"""
from ._lib import LIB_PATH, ParseError, ResourceExhausted, lib  # noqa: F401
from .voxin import *  # noqa: F401,F403
from . import bundled_nets  # noqa: F401

lib()  # fail loudly at import when the native library is missing
