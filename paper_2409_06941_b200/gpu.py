"""Python front end of include/freeride_gpu.h (side-task steps on sm_100a).

Device buffers are torch tensors (plumbing only); every computation runs in
the product library's kernels.  Calls are asynchronous on the given stream
(default: torch's current stream).  There is no CPU fallback: a missing
library or a non-CUDA tensor raises.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _abi as A
from . import lib as _load_lib

_glib = None


def glib() -> C.CDLL:
    global _glib
    if _glib is None:
        lib = _load_lib()
        A.bind(lib, A.HOST_PROTOTYPES)
        _glib = A.bind(lib, A.GPU_PROTOTYPES)
    return _glib


def check(rc: int):
    A.raise_for(glib(), rc)


def _ptr(t: torch.Tensor) -> int:
    if not t.is_cuda:
        raise ValueError("side-task buffers must be CUDA tensors (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError("side-task buffers must be contiguous")
    return t.data_ptr()


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


def low_priority_stream(device=None) -> torch.cuda.Stream:
    """The stream class side-task steps run in (lowest CUDA priority)."""
    lo, _hi = torch.cuda.Stream.priority_range()
    return torch.cuda.Stream(device=device, priority=lo)


# ------------------------------------------------------------------ K5 image
class ImagePlan:
    """fr_img_plan: one (src -> dst) resize shape."""

    GENERAL, TMA_2X = 0, 1

    def __init__(self, sw: int, sh: int, dw: int, dh: int):
        self.sw, self.sh, self.dw, self.dh = sw, sh, dw, dh
        h = C.c_void_p()
        check(glib().fr_img_plan_create(sw, sh, dw, dh, C.byref(h)))
        self._h = h

    @property
    def path(self) -> int:
        out = C.c_int32()
        check(glib().fr_img_plan_path(self._h, C.byref(out)))
        return out.value

    def run(self, src: torch.Tensor, dst: torch.Tensor, wm: torch.Tensor, stream=None):
        """dst[n,dh,dw,3] = blend(resize(src[n,sh,sw,3]), wm[dh,dw,4])."""
        n = src.shape[0]
        if tuple(src.shape[1:]) != (self.sh, self.sw, 3) or tuple(dst.shape) != (n, self.dh, self.dw, 3):
            raise ValueError("image shapes do not match the plan")
        if tuple(wm.shape) != (self.dh, self.dw, 4):
            raise ValueError("watermark must be [dh, dw, 4] RGBA")
        for t in (src, dst, wm):
            if t.dtype != torch.uint8:
                raise ValueError("images are uint8")
        check(glib().fr_img_resize_watermark(self._h, _ptr(src), _ptr(dst), _ptr(wm), n,
                                             _stream(stream)))
        return dst

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _glib is not None:
            _glib.fr_img_plan_destroy(h)
            self._h = None


def img_generate(n, w, h, channels=3, seed=1, first_index=0, device="cuda", stream=None):
    out = torch.empty((n, h, w, channels), dtype=torch.uint8, device=device)
    check(glib().fr_img_generate(_ptr(out), n, w, h, channels, seed, first_index, _stream(stream)))
    return out


def img_generate_watermark(w, h, seed=7, device="cuda", stream=None):
    out = torch.empty((h, w, 4), dtype=torch.uint8, device=device)
    check(glib().fr_img_generate_watermark(_ptr(out), w, h, seed, _stream(stream)))
    return out
