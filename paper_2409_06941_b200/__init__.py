"""B200-native bubble-harvesting hot path of FreeRide (arXiv 2409.06941).

The product is one in-tree shared library, `_lib/libfreeride.so` (host C++ +
sm_100a CUDA, C-ABI declared in include/freeride.h).  `lib()` loads it and
raises if it is missing -- there is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# FR_LIB: load another build of the library (A/B experiments only)
LIB_PATH = os.environ.get("FR_LIB") or os.path.join(_HERE, "_lib", "libfreeride.so")
REPO_ROOT = os.path.dirname(_HERE)

_lock = threading.Lock()
_lib = None
_api = None


class ExtensionMissing(ImportError):
    pass


def lib() -> ctypes.CDLL:
    """The product library (loaded once).  Fails loudly when it was not built."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ExtensionMissing(
                    f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
                    " (there is no CPU fallback)")
            _lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        return _lib


def api():
    """`bubblesim.BubbleSim` bound to the product library."""
    global _api
    if _api is None:
        from .bubblesim import BubbleSim
        _api = BubbleSim(lib())
    return _api
