"""B200-native AdaHOP MXFP4 linear (arXiv 2604.02525) — package root.

The compute lives in ``libadahop.so`` (hand-written sm_100a CUDA behind the C ABI in
include/adahop.h). This package is the thin Python binding over it; importing it fails
loudly if the library has not been built (there is no CPU fallback).
"""
from .adahop import *  # noqa: F401,F403
from .adahop import Params  # noqa: F401

__version__ = "0.1.0"
