"""CPU-only: the packed-lane integer identities the TMA image kernel relies on
(csrc/kernels/img.cu), checked exhaustively over their whole input domain."""
import numpy as np


def test_div255_identity_exhaustive():
    t = np.arange(0, 65408, dtype=np.int64)
    assert np.array_equal((t + 1 + (t >> 8)) >> 8, t // 255)


def test_packed_rg_blend_exhaustive():
    # every (px, wm, alpha) triple, evaluated two lanes at a time in uint32
    px = np.arange(256, dtype=np.uint32)
    a = np.arange(256, dtype=np.uint32)
    for w in range(256):
        P, A_ = np.meshgrid(px, a, indexing="ij")
        P2 = P | (P[::-1] << 16)                   # two different pixels per word
        W2 = np.uint32(w) | (np.uint32(255 - w) << 16)
        t = P2 * (255 - A_) + (W2 * A_ + np.uint32(0x007F007F))
        q = ((t + np.uint32(0x00010001) + ((t >> 8) & np.uint32(0x00FF00FF))) >> 8) & np.uint32(0x00FF00FF)
        want_lo = (P * (255 - A_) + w * A_ + 127) // 255
        want_hi = (P[::-1] * (255 - A_) + (255 - w) * A_ + 127) // 255
        assert np.array_equal(q & 0xFFFF, want_lo)
        assert np.array_equal(q >> 16, want_hi)


def test_packed_round_quarter():
    s = np.arange(0, 1021, dtype=np.uint32)
    x = s | (s[::-1] << 16)
    r = ((x + np.uint32(0x00020002)) >> 2) & np.uint32(0x00FF00FF)
    assert np.array_equal(r & 0xFFFF, (s + 2) >> 2)
    assert np.array_equal(r >> 16, (s[::-1] + 2) >> 2)
