"""Imperative interface on the B200 (PAPER.md:484-499 RunGpuWorkload;
imperative_run task.hpp:93): one preemptible K5
workload that a device-side stop word pauses between output rows.  Checked:
a stopped launch keeps every row it took (bit-exact), a resumed launch
finishes the batch bit-exact, and inside a pipeline the workload's time
outside bubbles per pause is far below one kernel (SPEC.md:181 bound)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    from paper_2409_06941_b200 import gpu
    gpu.glib()
    return gpu


@pytest.fixture(scope="module")
def batch(g, sidetask_oracle):
    n = 24
    src = g.img_generate(n, 3840, 2160, seed=21)
    wm = g.img_generate_watermark(1920, 1080, seed=22)
    want = sidetask_oracle.img_resize_watermark(src.cpu().numpy(), wm.cpu().numpy(), 1920, 1080)
    return src, wm, want


def rows_done(ctr):
    return int(ctr[2:4].view(torch.int64).item())


def test_stop_before_start_takes_no_row(g, batch):
    src, wm, _ = batch
    plan = g.ImagePlan(3840, 2160, 1920, 1080)
    prep = plan.prepare(wm)
    dst = torch.zeros((src.shape[0], 1080, 1920, 3), dtype=torch.uint8, device="cuda")
    ctr = torch.zeros(8, dtype=torch.int32, device="cuda")
    stop = torch.full((1,), 5, dtype=torch.int32, device="cuda")
    plan.run_preemptible(src, dst, prep, ctr, stop_word=stop, token=5)
    torch.cuda.synchronize()
    assert rows_done(ctr) == 0 and int(ctr[0]) == 0 and int(dst.abs().sum()) == 0


def test_preempted_then_resumed_is_bit_exact(g, batch):
    """The stop word is raised from a high-priority stream while the workload
    runs; when it lands before the workload ends, the workload must exit
    within a few rows (not finish the batch), keep every row it took, and a
    resumed launch must complete the batch bit-exact."""
    src, wm, want = batch
    n = src.shape[0]
    plan = g.ImagePlan(3840, 2160, 1920, 1080)
    # leave SMs free for the stopper: the fill_ below is a new launch, and the
    # workload's CTAs fill every register file they sit on (in the runtime the
    # stop word is raised by the stage's resident gap kernel instead)
    plan.set_max_sms(100)
    prep = plan.prepare(wm)
    lo = g.low_priority_stream()
    hi = torch.cuda.Stream(priority=torch.cuda.Stream.priority_range()[1])
    partial = 0
    for sleep in (0, 20_000, 60_000, 120_000, 0, 40_000):
        dst = torch.zeros((n, 1080, 1920, 3), dtype=torch.uint8, device="cuda")
        ctr = torch.zeros(8, dtype=torch.int32, device="cuda")
        stop = torch.zeros(1, dtype=torch.int32, device="cuda")
        t0, t1, t2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        torch.cuda.synchronize()
        t0.record(lo)
        plan.run_preemptible(src, dst, prep, ctr, stop_word=stop, token=1, stream=lo)
        t1.record(lo)
        with torch.cuda.stream(hi):
            if sleep:
                torch.cuda._sleep(sleep)
            stop.fill_(1)
            t2.record(hi)
        torch.cuda.synchronize()
        first = rows_done(ctr)
        unit = plan.preemptible_unit_rows(n)
        assert first % unit == 0                    # whole units only
        assert int(ctr[0]) == (first // unit) % (n * 1080 // unit)   # base advanced by the units taken = completed
        end_us, stop_us = t0.elapsed_time(t1) * 1e3, t0.elapsed_time(t2) * 1e3
        if stop_us < end_us - 1.0:
            assert end_us - stop_us < 50.0          # exits within a few rows of the stop
            partial += first < n * 1080
        # resume, no preemption: exactly the rows not yet taken
        plan.run_preemptible(src, dst, prep, ctr, max_rows=n * 1080 - first, stream=lo)
        torch.cuda.synchronize()
        assert rows_done(ctr) == n * 1080
        assert int(ctr[0]) == 0                   # base + taken wrapped to the batch start
        assert np.array_equal(dst.cpu().numpy(), want)
    assert partial > 0


def test_budget_loops_over_the_batch(g, batch):
    src, wm, want = batch
    n = 4
    plan = g.ImagePlan(3840, 2160, 1920, 1080)
    prep = plan.prepare(wm)
    dst = torch.zeros((n, 1080, 1920, 3), dtype=torch.uint8, device="cuda")
    ctr = torch.zeros(8, dtype=torch.int32, device="cuda")
    unit = plan.preemptible_unit_rows(n)
    assert unit == 4                                  # the same row of 4 consecutive frames
    plan.run_preemptible(src[:n], dst, prep, ctr, max_rows=2 * n * 1080 + 500)
    torch.cuda.synchronize()
    assert rows_done(ctr) == 2 * n * 1080 + 500 and int(ctr[0]) == 500 // unit
    assert np.array_equal(dst.cpu().numpy(), want[:n])


def test_imperative_task_in_bubbles(g, batch, sidetask_oracle):
    h = g.Harness(num_stages=4, num_micro_batches=4, stage=1, layers=2, profile_reps=3,
                  profile_epochs=2)
    task = g.ImageTask(batch=8, images_per_step=8, seed=31, imperative=True)
    ok, prof = h.submit("img-imp", task)
    assert ok and not prof["has_est_per_step"]          # imperative: not step-profiled
    warm = h.run(2, True)                               # InitSideTask in the first bubble
    base = h.run(4, False)
    r = h.run(4, True)
    assert r["steps_completed"] == r["steps_launched"] > 0
    assert r["work_units"] > 0 and r["used_s"] / r["bubble_s"] > 0.6
    assert r["pauses"] > 0
    # busy time outside bubbles per pause <= one kernel; the
    # device-side stop makes it about one output row
    assert r["overrun_s"] / r["pauses"] < 200e-6
    dt = (r["makespan_s"] - base["makespan_s"]) / base["makespan_s"]
    assert dt < 0.01
    # every row of the resident batch has been produced at least once by now
    assert warm["work_units"] + r["work_units"] >= 8 * 1080 * 1920
    src = sidetask_oracle.img_generate(8, 3840, 2160, seed=31)
    wm = sidetask_oracle.img_generate_watermark(1920, 1080, seed=31 ^ 0x77)
    want = sidetask_oracle.img_resize_watermark(src, wm, 1920, 1080)
    assert np.array_equal(task.outputs().cpu().numpy(), want)
    h.close()
