"""B200-native VGICP matching-cost path (arXiv 2202.00242), a drop-in for limapper's
registration / preprocess / MatchingCostFactor API backed by hand-written sm_100a CUDA
(libvgicp.so, C-ABI in include/vgicp.h)."""

from ._lib import LIB_PATH, VgicpUnavailable, context, load_library, set_device

__all__ = ["LIB_PATH", "VgicpUnavailable", "context", "load_library", "set_device"]
__version__ = "0.1.0"
