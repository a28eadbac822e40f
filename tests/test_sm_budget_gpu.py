"""Power-aware harvesting: the side-task kernels under an SM
budget stay exact (K5 bit-exact, PageRank L1 <= 1e-6, Graph-SGD RMSE within
1e-3 of the sequential oracle), and the harness's ΔT controller shrinks the
budget when the stage's ops slow down beyond it."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ETA, LAM = 0.01, 0.05


@pytest.fixture(scope="module")
def g():
    from paper_2409_06941_b200 import gpu
    gpu.glib()
    return gpu


@pytest.mark.parametrize("sms", [1, 7, 16, 148])
def test_image_under_sm_budget_bit_exact(g, sidetask_oracle, sms):
    plan = g.ImagePlan(3840, 2160, 1920, 1080)
    plan.set_max_sms(sms)
    plan.set_overlap(True)
    src = g.img_generate(6, 3840, 2160, seed=11)
    wm = g.img_generate_watermark(1920, 1080, seed=12)
    dst = torch.empty((6, 1080, 1920, 3), dtype=torch.uint8, device="cuda")
    prepared = plan.prepare(wm)
    s = g.low_priority_stream()
    torch.cuda.synchronize()
    for i in range(0, 6, 2):   # consecutive (PDL-chained) steps under the budget
        plan.run_prepared(src[i:i + 2], dst[i:i + 2], prepared, stream=s)
    s.synchronize()
    want = sidetask_oracle.img_resize_watermark(src.cpu().numpy(), wm.cpu().numpy(), 1920, 1080)
    assert np.array_equal(dst.cpu().numpy(), want)


@pytest.mark.parametrize("sms", [3, 20])
def test_pagerank_under_sm_budget(g, sidetask_oracle, sms):
    """a grid of `sms` CTAs walks all of the build's split-row chunk lists"""
    graph = g.PageRankGraph(scale=20, edge_factor=16, seed=1)
    src, dst = sidetask_oracle.rmat_edges(20, 16, seed=1)
    off, col, outdeg = sidetask_oracle.build_pull_csr(1 << 20, src, dst)
    st = g.PageRankState(graph)
    st.set_max_sms(sms)
    st.reset()
    st.step(20, 0.85)
    got = st.ranks().double().cpu().numpy()
    want = sidetask_oracle.pr_run(off, col, outdeg, 20, 0.85)
    assert np.abs(got - want).sum() <= 1e-6


def test_sgd_under_sm_budget(g, sidetask_oracle):
    V, E = 200000, 8000000
    p = g.SgdProblem(V=V, E=E, k=16, edge_seed=2, init_seed=3, by_user=True, window=1 << 20)
    p.set_max_sms(16)
    u, v, r = sidetask_oracle.sgd_group_by_user(V, *sidetask_oracle.sgd_edges(V, E, seed=2), window=1 << 20)
    L = sidetask_oracle.sgd_init(V, 16, seed=3)
    for ep in range(3):
        for a in range(0, E, 1 << 20):
            p.step(a, min(E, a + (1 << 20)), ETA, LAM)
        sidetask_oracle.sgd_epoch(u, v, r, L, ETA, LAM, nthreads=1)
    got, want = p.rmse(), sidetask_oracle.sgd_rmse(u, v, r, L)
    assert abs(got - want) <= 1e-3, (got, want)


def test_dt_controller_shrinks_the_budget(g):
    """full-GPU image steps slow the stage's GEMMs by ~10 % (power); with a
    0.3 % budget the controller must leave far fewer SMs to the side task,
    report the op slowdown it saw, and keep harvesting"""
    h = g.Harness(num_stages=4, num_micro_batches=4, stage=1, layers=6, hidden=2048, tokens=8192,
                  profile_reps=3, profile_epochs=2, step_group=3, dt_budget=0.003)
    ok, _ = h.submit("image", g.ImageTask(batch=64, images_per_step=16), profile_steps=8)
    assert ok
    h.run(2, False)                        # the controller's op reference
    first = h.run(4, True)
    assert first["side_sms_final"] < 148 and first["side_sms_mean"] < 148
    last = None
    for _ in range(3):
        last = h.run(4, True)
    assert last["steps_completed"] > 0 and last["work_units"] > 0
    assert last["side_sms_mean"] < 0.5 * 148, last
    assert -0.05 < last["op_growth"] < 0.05
    h.close()


def test_fixed_budget_is_reported(g):
    h = g.Harness(num_stages=4, num_micro_batches=4, stage=2, layers=2, profile_reps=2, profile_epochs=1,
                  side_sms=12)
    ok, _ = h.submit("image", g.ImageTask(batch=16, images_per_step=2), profile_steps=4)
    assert ok
    r = h.run(2, True)
    assert r["side_sms_final"] == 12 and r["side_sms_mean"] == 12 and r["steps_completed"] > 0
    h.close()
