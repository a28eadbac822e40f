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


# ---- round 2: the dp4a group (img_group8_dp), restated with numpy uint32 ops
def _byte_perm(x, y, s):
    """__byte_perm(x, y, s): byte i of the result = byte (s >> 4i) & 7 of y:x"""
    x = np.asarray(x, dtype=np.uint64)
    y = np.asarray(y, dtype=np.uint64)
    both = x | (y << np.uint64(32))
    out = np.zeros(np.broadcast(x, y).shape, dtype=np.uint64)
    for i in range(4):
        sel = (s >> (4 * i)) & 7
        out |= ((both >> np.uint64(8 * sel)) & np.uint64(0xFF)) << np.uint64(8 * i)
    return out.astype(np.uint32)


def _dp4a(a, w, c):
    a = np.asarray(a, dtype=np.uint32)
    acc = np.asarray(c, dtype=np.uint32).astype(np.uint64)
    for i in range(4):
        acc = acc + ((a >> np.uint32(8 * i)) & np.uint32(0xFF)).astype(np.uint64) * ((w >> (8 * i)) & 0xFF)
    return (acc & np.uint64(0xFFFFFFFF)).astype(np.uint32)


def _group8_dp(ra, rb, wm_rgba):
    """one thread's 8 output pixels (csrc/kernels/img.cu img_group8_dp): ra / rb
    = 48 source bytes of each row, wm_rgba = the 8 pixels' RGBA watermark"""
    va = ra.view("<u4")
    vb = rb.view("<u4")
    w = wm_rgba.astype(np.uint32)
    wc = lambda ch, p: np.uint32(w[p, ch] * w[p, 3] + 127)   # noqa: E731
    u32 = np.uint32
    uX, uY, uZ = [], [], []
    for q in range(4):
        a0, a1, a2 = va[3 * q:3 * q + 3]
        b0, b1, b2 = vb[3 * q:3 * q + 3]
        ga, gb = _byte_perm(a0, a1, 0x5421), _byte_perm(b0, b1, 0x5421)
        ha, hb = _byte_perm(a1, a2, 0x6532), _byte_perm(b1, b2, 0x6532)
        W03, W02, W13 = 0x40000040, 0x00400040, 0x40004000
        sR0 = _dp4a(a0, W03, _dp4a(b0, W03, 128))
        sG0 = _dp4a(ga, W02, _dp4a(gb, W02, 128))
        sB0 = _dp4a(ga, W13, _dp4a(gb, W13, 128))
        sR1 = _dp4a(ha, W02, _dp4a(hb, W02, 128))
        sG1 = _dp4a(ha, W13, _dp4a(hb, W13, 128))
        sB1 = _dp4a(a2, W03, _dp4a(b2, W03, 128))
        p0, p1 = 2 * q, 2 * q + 1
        wX = wc(0, p0) | (wc(2, p0) << u32(16))
        wY = wc(1, p0) | (wc(0, p1) << u32(16))
        wZ = wc(2, p1) | (wc(1, p1) << u32(16))
        na0, na1 = u32(255 - w[p0, 3]), u32(255 - w[p1, 3])
        X = _byte_perm(sR0, sB0, 0x6521)
        Z = _byte_perm(sB1, sG1, 0x6521)
        Ylo = _byte_perm(sG0, 0, 0x4441)
        Yhi = _byte_perm(sR1, 0, 0x4144)
        div = lambda t: u32(t + _byte_perm(t, 0, 0x4341) + u32(0x00010001))  # noqa: E731
        with np.errstate(over="ignore"):
            uX.append(div(u32(X * na0 + wX)))
            uZ.append(div(u32(Z * na1 + wZ)))
            uY.append(div(u32(Yhi * na1 + u32(Ylo * na0 + wY))))
    o = []
    for h in range(2):
        q = 2 * h
        A0 = _byte_perm(uX[q], uY[q], 0x7351)
        A1 = _byte_perm(uX[q + 1], uY[q + 1], 0x7351)
        o += [A0, _byte_perm(uZ[q], A1, 0x5413), _byte_perm(A1, uZ[q + 1], 0x5732)]
    return np.array(o, dtype="<u4").view(np.uint8)


def test_dp4a_group_matches_the_blend_rule():
    """the dp4a kernel's arithmetic, restated on the CPU, reproduces the
    oracle's rule (2x2 mean with (s+2)>>2, blend (px(255-a) + wa + 127)/255)
    for random pixels and every alpha extreme"""
    rng = np.random.default_rng(7)
    for trial in range(300):
        ra = rng.integers(0, 256, 48, dtype=np.uint8)
        rb = rng.integers(0, 256, 48, dtype=np.uint8)
        wm = rng.integers(0, 256, (8, 4), dtype=np.uint8)
        if trial % 3 == 1:
            wm[:, 3] = 0
        elif trial % 3 == 2:
            wm[:, 3] = 255
        if trial == 4:
            ra[:] = rb[:] = 255
        got = _group8_dp(ra, rb, wm)
        A = ra.reshape(16, 3).astype(np.int64)
        B = rb.reshape(16, 3).astype(np.int64)
        s = A[0::2] + A[1::2] + B[0::2] + B[1::2]
        px = (s + 2) >> 2
        a = wm[:, 3:4].astype(np.int64)
        want = (px * (255 - a) + wm[:, :3].astype(np.int64) * a + 127) // 255
        assert np.array_equal(got, want.astype(np.uint8).reshape(-1)), trial
