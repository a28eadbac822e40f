"""K5 image resize + watermark on the B200 vs the CPU oracle (bit-exact)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    from paper_2409_06941_b200 import gpu
    gpu.glib()
    return gpu


def test_generators_match_oracle(g, sidetask_oracle):
    o = sidetask_oracle
    for (n, w, h, ch, seed, first) in [(2, 37, 11, 3, 5, 0), (1, 3840, 2160, 3, 1, 7), (3, 16, 16, 4, 9, 2)]:
        got = g.img_generate(n, w, h, ch, seed, first).cpu().numpy()
        want = o.img_generate(n, w, h, ch, seed, first)
        assert np.array_equal(got, want)
    assert np.array_equal(g.img_generate_watermark(1920, 1080, 7).cpu().numpy(),
                          o.img_generate_watermark(1920, 1080, 7))


@pytest.mark.parametrize("n", [1, 2, 5])
def test_tma_2x_4k_bit_exact(g, sidetask_oracle, n):
    plan = g.ImagePlan(3840, 2160, 1920, 1080)
    assert plan.path == g.ImagePlan.TMA_2X
    src = g.img_generate(n, 3840, 2160, seed=11 + n)
    wm = g.img_generate_watermark(1920, 1080, seed=3)
    dst = torch.full((n, 1080, 1920, 3), 0xAB, dtype=torch.uint8, device="cuda")
    plan.run(src, dst, wm)
    torch.cuda.synchronize()
    want = sidetask_oracle.img_resize_watermark(src.cpu().numpy(), wm.cpu().numpy(), 1920, 1080)
    assert np.array_equal(dst.cpu().numpy(), want)


@pytest.mark.parametrize("math", ["1", "0"])
def test_prepared_watermark_path_bit_exact(g, sidetask_oracle, monkeypatch, math):
    """The task's path: watermark prepared once, per-step kernel on the prepared form.
    Both exact-2x math variants (FR_IMG_MATH: 1 = dp4a sums, the default; 0 =
    16-bit lane sums), each with its own prepared layout (10 / 8 B per pixel)."""
    monkeypatch.setenv("FR_IMG_MATH", math)
    plan = g.ImagePlan(3840, 2160, 1920, 1080)
    src = g.img_generate(3, 3840, 2160, seed=21)
    wm = g.img_generate_watermark(1920, 1080, seed=22)
    prepared = plan.prepare(wm)
    assert prepared.numel() == 1920 * 1080 * (10 if math == "1" else 8)
    dst = torch.empty((3, 1080, 1920, 3), dtype=torch.uint8, device="cuda")
    plan.run_prepared(src, dst, prepared)
    want = sidetask_oracle.img_resize_watermark(src.cpu().numpy(), wm.cpu().numpy(), 1920, 1080)
    assert np.array_equal(dst.cpu().numpy(), want)
    # extreme alphas: fully opaque / fully transparent watermark
    for a in (0, 255):
        wm2 = wm.clone()
        wm2[..., 3] = a
        plan.run_prepared(src[:1], dst[:1], plan.prepare(wm2))
        want = sidetask_oracle.img_resize_watermark(src[:1].cpu().numpy(), wm2.cpu().numpy(), 1920, 1080)
        assert np.array_equal(dst[:1].cpu().numpy(), want)


# exact-2x kernel variants: the warp-specialised kernel with one-pipeline CTAs
# (default) or 3-pipeline CTAs, the round-1 per-row-barrier kernel with the
# dp4a math or the 16-bit lane math
VARIANTS = {"ws": {}, "ws_pipes3": {"FR_IMG_PIPES": "3"}, "bar_dp4a": {"FR_IMG_CFG": "bar"},
            "bar_lanes": {"FR_IMG_MATH": "0"}}


@pytest.mark.parametrize("variant", sorted(VARIANTS))
@pytest.mark.parametrize("sw,sh,dw,dh", [(32, 2, 16, 1), (64, 30, 32, 15), (1024, 6, 512, 3), (4128, 10, 2064, 5)])
def test_tma_2x_small_shapes(g, sidetask_oracle, monkeypatch, variant, sw, sh, dw, dh):
    for k, v in VARIANTS[variant].items():
        monkeypatch.setenv(k, v)
    plan = g.ImagePlan(sw, sh, dw, dh)
    assert plan.path == g.ImagePlan.TMA_2X
    src = g.img_generate(3, sw, sh, seed=4)
    wm = g.img_generate_watermark(dw, dh, seed=8)
    dst = torch.empty((3, dh, dw, 3), dtype=torch.uint8, device="cuda")
    plan.run(src, dst, wm)
    want = sidetask_oracle.img_resize_watermark(src.cpu().numpy(), wm.cpu().numpy(), dw, dh)
    assert np.array_equal(dst.cpu().numpy(), want)


def test_general_path_random_shapes(g, sidetask_oracle):
    rng = np.random.default_rng(5)
    for _ in range(40):
        sh, sw, dh, dw = (int(x) for x in rng.integers(1, 300, 4))
        plan = g.ImagePlan(sw, sh, dw, dh)
        n = int(rng.integers(1, 3))
        src = g.img_generate(n, sw, sh, seed=int(rng.integers(1 << 30)))
        wm = g.img_generate_watermark(dw, dh, seed=int(rng.integers(1 << 30)))
        dst = torch.empty((n, dh, dw, 3), dtype=torch.uint8, device="cuda")
        plan.run(src, dst, wm)
        want = sidetask_oracle.img_resize_watermark(src.cpu().numpy(), wm.cpu().numpy(), dw, dh)
        assert np.array_equal(dst.cpu().numpy(), want), (sw, sh, dw, dh)


def test_general_path_matches_cv2(g):
    cv2 = pytest.importorskip("cv2")
    plan = g.ImagePlan(641, 479, 320, 240)
    assert plan.path == g.ImagePlan.GENERAL
    src = g.img_generate(1, 641, 479, seed=2)
    wm = torch.zeros((240, 320, 4), dtype=torch.uint8, device="cuda")  # alpha 0: pure resize
    dst = torch.empty((1, 240, 320, 3), dtype=torch.uint8, device="cuda")
    plan.run(src, dst, wm)
    want = cv2.resize(src[0].cpu().numpy(), (320, 240), interpolation=cv2.INTER_LINEAR_EXACT)
    assert np.array_equal(dst[0].cpu().numpy(), want)


def test_edge_cases(g):
    from paper_2409_06941_b200._abi import FreeRideError, ValidationError
    plan = g.ImagePlan(64, 64, 32, 32)
    src = torch.zeros((0, 64, 64, 3), dtype=torch.uint8, device="cuda")
    dst = torch.zeros((0, 32, 32, 3), dtype=torch.uint8, device="cuda")
    wm = torch.zeros((32, 32, 4), dtype=torch.uint8, device="cuda")
    plan.run(src, dst, wm)  # n = 0: no launch, no error
    big = torch.zeros(64 * 64 * 3 + 1, dtype=torch.uint8, device="cuda")
    out1 = torch.zeros((1, 32, 32, 3), dtype=torch.uint8, device="cuda")
    lib = g.glib()
    rc = lib.fr_img_resize_watermark(plan._h, big.data_ptr() + 1, out1.data_ptr(), wm.data_ptr(), 1,
                                     torch.cuda.current_stream().cuda_stream)
    assert rc == 8  # FR_ERR_UNSUPPORTED: TMA path needs 16-byte alignment
    with pytest.raises(ValidationError):
        g.ImagePlan(0, 4, 2, 2)
    with pytest.raises(ValueError):
        plan.run(src.cpu(), dst, wm)


@pytest.mark.parametrize("variant", ["ws", "ws_pipes3"])
def test_full_batch_64_bit_exact(g, sidetask_oracle, monkeypatch, variant):
    """configs[1] at its full size: 64 4K images -> 1080p, every byte checked."""
    for k, v in VARIANTS[variant].items():
        monkeypatch.setenv(k, v)
    n = 64
    plan = g.ImagePlan(3840, 2160, 1920, 1080)
    src = g.img_generate(n, 3840, 2160, seed=1)
    wm = g.img_generate_watermark(1920, 1080, seed=7)
    dst = torch.empty((n, 1080, 1920, 3), dtype=torch.uint8, device="cuda")
    s = g.low_priority_stream()
    torch.cuda.synchronize()
    plan.run(src, dst, wm, stream=s)
    s.synchronize()
    got = dst.cpu().numpy()
    want = sidetask_oracle.img_resize_watermark(src.cpu().numpy(), wm.cpu().numpy(), 1920, 1080)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("budget", [0, 3])
def test_ws_kernel_under_chaos_is_bit_exact(g, sidetask_oracle, monkeypatch, budget):
    """The warp-specialised K5 hands rows and stages between its producer and
    consumer warps on mbarriers only (no CTA barrier; compute-sanitizer's
    racecheck does not model mbarrier ordering and reports those hand-offs).
    With FR_IMG_CHAOS=1 every hand-off sleeps a pseudo-random 0-4 us first, so
    an ordering the mbarriers did not enforce would corrupt output bytes.
    budget 3: 9 CTAs, so a 16-frame launch claims 16-frame units."""
    monkeypatch.setenv("FR_IMG_CHAOS", "1")
    plan = g.ImagePlan(3840, 2160, 1920, 1080)
    plan.set_max_sms(budget)
    src = g.img_generate(16, 3840, 2160, seed=31)
    wm = g.img_generate_watermark(1920, 1080, seed=32)
    prep = plan.prepare(wm)
    dst = torch.empty((16, 1080, 1920, 3), dtype=torch.uint8, device="cuda")
    want = sidetask_oracle.img_resize_watermark(src.cpu().numpy(), wm.cpu().numpy(), 1920, 1080)
    for _ in range(2):
        dst.zero_()
        plan.run_prepared(src, dst, prep)
        torch.cuda.synchronize()
        assert np.array_equal(dst.cpu().numpy(), want)
    # the preemptible path (one-row claims) under the same chaos
    ctr = torch.zeros(8, dtype=torch.int32, device="cuda")
    dst.zero_()
    plan.run_preemptible(src, dst, prep, ctr)
    torch.cuda.synchronize()
    assert np.array_equal(dst.cpu().numpy(), want)
