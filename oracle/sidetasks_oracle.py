"""ORACLE / TEST INFRASTRUCTURE ONLY -- numpy front end of oracle/sidetasks.c.

Loaded only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs, always as the checker or the timed CPU baseline,
never on the product path.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
DEFAULT_LIB = os.path.join(HERE, "_build", "liboracle_sidetasks.so")

u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


class SideTaskOracle:
    def __init__(self, path=DEFAULT_LIB):
        lib = C.CDLL(path)
        lib.orc_splitmix64.restype = C.c_uint64
        lib.orc_splitmix64.argtypes = [C.c_uint64]
        lib.orc_img_generate.argtypes = [u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int]
        lib.orc_img_generate_watermark.argtypes = [u8p, C.c_int, C.c_int, C.c_uint64, C.c_int]
        lib.orc_img_coeffs.argtypes = [C.c_int, C.c_int, i32p, i32p, i32p]
        lib.orc_img_resize_watermark.argtypes = [u8p, u8p, u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
        lib.orc_rmat_edges.argtypes = [C.c_int, C.c_int64, C.c_uint64, i32p, i32p, C.c_int]
        lib.orc_pr_run.argtypes = [C.c_int32, i32p, i32p, i32p, C.c_double, C.c_int, f64p, C.c_int]
        lib.orc_sgd_edges.argtypes = [C.c_int32, C.c_int64, C.c_uint64, i32p, i32p, f32p, C.c_int]
        lib.orc_sgd_group_by_user.argtypes = [C.c_int32, C.c_int64, C.c_int64, C.c_int, i32p, i32p, f32p]
        lib.orc_sgd_item_blocks.restype = C.c_int32
        lib.orc_sgd_item_blocks.argtypes = [C.c_int32, C.c_int]
        lib.orc_sgd_init.argtypes = [C.c_int32, C.c_int, C.c_uint64, f32p, C.c_int]
        lib.orc_sgd_epoch.argtypes = [C.c_int64, i32p, i32p, f32p, f32p, C.c_int, C.c_float, C.c_float, C.c_int]
        lib.orc_sgd_rmse.restype = C.c_double
        lib.orc_sgd_rmse.argtypes = [C.c_int64, i32p, i32p, f32p, f32p, C.c_int, C.c_int]
        self.lib = lib

    # ------------------------------------------------------------- images
    def img_generate(self, n, w, h, channels=3, seed=1, first_index=0, nthreads=0):
        out = np.empty((n, h, w, channels), np.uint8)
        self.lib.orc_img_generate(out.reshape(-1), n, w, h, channels, seed, first_index, nthreads)
        return out

    def img_generate_watermark(self, w, h, seed=7, nthreads=0):
        out = np.empty((h, w, 4), np.uint8)
        self.lib.orc_img_generate_watermark(out.reshape(-1), w, h, seed, nthreads)
        return out

    def img_coeffs(self, src_n, dst_n):
        i0, i1, w1 = (np.empty(dst_n, np.int32) for _ in range(3))
        self.lib.orc_img_coeffs(src_n, dst_n, i0, i1, w1)
        return i0, i1, w1

    def img_resize_watermark(self, src, wm, dw, dh, nthreads=0):
        src = np.ascontiguousarray(src)
        n, sh, sw, ch = src.shape
        assert ch == 3 and wm.shape == (dh, dw, 4)
        out = np.empty((n, dh, dw, 3), np.uint8)
        self.lib.orc_img_resize_watermark(src.reshape(-1), out.reshape(-1), np.ascontiguousarray(wm).reshape(-1),
                                          n, sw, sh, dw, dh, nthreads)
        return out

    # ----------------------------------------------------------- PageRank
    def rmat_edges(self, scale, edge_factor=16, seed=1, nthreads=0):
        m = edge_factor << scale
        src, dst = np.empty(m, np.int32), np.empty(m, np.int32)
        self.lib.orc_rmat_edges(scale, m, seed, src, dst, nthreads)
        return src, dst

    @staticmethod
    def build_pull_csr(V, src, dst):
        """Drop self loops and duplicates; incoming CSR sorted by (dst, src)."""
        keep = src != dst
        key = np.unique((dst[keep].astype(np.int64) << 32) | src[keep].astype(np.int64))
        d = (key >> 32).astype(np.int32)
        s = (key & 0xFFFFFFFF).astype(np.int32)
        offsets = np.zeros(V + 1, np.int32)
        np.cumsum(np.bincount(d, minlength=V), out=offsets[1:])
        outdeg = np.bincount(s, minlength=V).astype(np.int32)
        return offsets, s, outdeg

    def pr_run(self, offsets, col_idx, outdeg, iters, damping=0.85, r0=None, nthreads=0):
        V = len(offsets) - 1
        r = np.full(V, 1.0 / V) if r0 is None else np.array(r0, np.float64)
        self.lib.orc_pr_run(V, offsets, col_idx, outdeg, damping, iters, r, nthreads)
        return r

    # ---------------------------------------------------------- Graph-SGD
    def sgd_edges(self, V, E, seed=2, nthreads=0):
        u, v, r = np.empty(E, np.int32), np.empty(E, np.int32), np.empty(E, np.float32)
        self.lib.orc_sgd_edges(V, E, seed, u, v, r, nthreads)
        return u, v, r

    def sgd_group_by_user(self, V, u, v, r, window=1 << 21, k=16):
        """fr_sgd_group_by_user's layout, in place: stable by u, then by item
        block (latent rows > 64 MiB), each (block, user) run cut into 64-edge
        pieces dealt over ceil(E / window) rounds inside its block"""
        self.lib.orc_sgd_group_by_user(V, len(u), window, k, u, v, r)
        return u, v, r

    def sgd_init(self, V, k=16, seed=3, nthreads=0):
        L = np.empty((V, k), np.float32)
        self.lib.orc_sgd_init(V, k, seed, L.reshape(-1), nthreads)
        return L

    def sgd_epoch(self, u, v, r, L, eta, lam, nthreads=1):
        self.lib.orc_sgd_epoch(len(u), u, v, r, L.reshape(-1), L.shape[1], eta, lam, nthreads)

    def sgd_rmse(self, u, v, r, L, nthreads=0):
        return self.lib.orc_sgd_rmse(len(u), u, v, r, L.reshape(-1), L.shape[1], nthreads)


def load(path=DEFAULT_LIB) -> SideTaskOracle:
    return SideTaskOracle(path)
