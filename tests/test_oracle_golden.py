"""CPU: pin the oracle (and the product host core) to golden vectors.

 * SURVEY.md Appendix A values, computed there by the compiled reference
   (asserted literally here);
 * tests/golden/host_reference.json -- oracle/_ref outputs (make_golden.py);
 * tests/golden/{image_cv2,pagerank_scipy,sgd_numpy}.npz -- independent
   libraries (cv2 INTER_LINEAR_EXACT, scipy.sparse, numpy float32).
"""
import json
import os

import numpy as np
import pytest

from paper_2409_06941_b200.bubblesim import (BubbleType, Gate, Enforce, PipelineConfig,
                                             ProfileOptions, SideTaskSpec, SideTaskRuntime,
                                             SideTaskState, TaskProfile)

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_oracle_image_matches_cv2(sidetask_oracle):
    z = np.load(os.path.join(GOLD, "image_cv2.npz"))
    for i in range(5):
        src, wm, want = z[f"src{i}"], z[f"wm{i}"], z[f"out{i}"]
        got = sidetask_oracle.img_resize_watermark(src[None], wm, wm.shape[1], wm.shape[0])
        assert np.array_equal(got[0], want), i


def test_oracle_pagerank_matches_scipy(sidetask_oracle):
    z = np.load(os.path.join(GOLD, "pagerank_scipy.npz"))
    V = int(z["V"])
    off, col, outdeg = sidetask_oracle.build_pull_csr(V, z["src"], z["dst"])
    r = sidetask_oracle.pr_run(off, col, outdeg, int(z["iters"]), float(z["damping"]))
    assert np.abs(r - z["ranks"]).sum() < 1e-12


def test_oracle_sgd_matches_numpy_bitwise(sidetask_oracle):
    z = np.load(os.path.join(GOLD, "sgd_numpy.npz"))
    L = z["L0"].copy()
    for _ in range(2):
        sidetask_oracle.sgd_epoch(z["u"], z["v"], z["r"], L, float(z["eta"]), float(z["lam"]), nthreads=1)
    assert np.array_equal(L, z["L2"])
    assert abs(sidetask_oracle.sgd_rmse(z["u"], z["v"], z["r"], L) - float(z["rmse"])) < 1e-12


def _splitmix64(x):
    x = (x + np.uint64(0x9E3779B97F4A7C15))
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def _by_user_numpy(u, v, V, R, P):
    """fr_sgd_group_by_user's layout restated with numpy (independent of the C oracle)"""
    o = np.argsort(u, kind="stable")
    if P > 1:
        o = o[np.argsort((v[o].astype(np.int64) * P) // V, kind="stable")]
    if R > 1:
        us = u[o].astype(np.int64)
        blk = (v[o].astype(np.int64) * P) // V
        key = blk * (int(us.max()) + 1) + us
        start = np.flatnonzero(np.concatenate([[True], key[1:] != key[:-1]]))
        length = np.diff(np.concatenate([start, [len(us)]]))
        rid = np.cumsum(np.concatenate([[True], key[1:] != key[:-1]])) - 1
        rank = np.arange(len(us)) - start[rid]
        deg = length[rid]
        npieces, q = (deg + 63) // 64, rank // 64
        with np.errstate(over="ignore"):
            h = (_splitmix64(np.uint64(0x5347445250) ^ us.astype(np.uint64)) % np.uint64(R)).astype(np.int64)
        rnd = blk * R + (q * R // npieces + h) % R
        o = o[np.argsort(rnd, kind="stable")]
    return o


@pytest.mark.parametrize("V,E,k,window", [(5000, 200000, 16, 1 << 30), (5000, 200000, 16, 20000),
                                          (5000, 200000, 16, 4096), (200000, 1000000, 128, 1 << 30),
                                          (200000, 1000000, 128, 65536)])
def test_oracle_sgd_group_by_user_layout(sidetask_oracle, V, E, k, window):
    """by-user layout: stable by u (Gardenia's CSR order); by item block once the
    latent rows pass 64 MiB (here k = 128: P = 2); 64-edge pieces of each
    (block, user) run dealt over ceil(E / window) rounds inside the block"""
    u, v, r = sidetask_oracle.sgd_edges(V, E, seed=9)
    R = max(1, -(-E // window))
    P = max(1, -(-(V * k * 4) // (64 << 20)))
    assert P == sidetask_oracle.lib.orc_sgd_item_blocks(V, k)
    o = _by_user_numpy(u, v, V, R, P)
    gu, gv, gr = sidetask_oracle.sgd_group_by_user(V, u.copy(), v.copy(), r.copy(), window=window, k=k)
    assert np.array_equal(gu, u[o]) and np.array_equal(gv, v[o]) and np.array_equal(gr, r[o])


def test_appendix_a1_issue_order(product, ref):
    want = {0: "F1 F2 F3 F4 B1 B2 B3 B4", 1: "F1 F2 F3 B1 F4 B2 B3 B4",
            2: "F1 F2 B1 F3 B2 F4 B3 B4", 3: "F1 B1 F2 B2 F3 B3 F4 B4"}
    for api in (product, ref):
        for s, w in want.items():
            got = " ".join(("F" if k == 0 else "B") + str(mb) for k, mb in api.stage_issue_order(s, 4, 4))
            assert got == w


def test_appendix_a1_schedule_and_bubbles(product):
    cfg = PipelineConfig(4, 4, [1], [2], 1, 48.0, product.default_stage_memory(4, 48.0, 4.0, 4.0))
    tr = product.build_schedule(cfg)
    assert tr.epoch_spans == [(0, 21)] and len(tr.ops) == 32
    s0 = [(o.kind.name[0], o.micro_batch, o.start, o.end) for o in tr.ops if o.stage == 0]
    assert s0 == [("F", 1, 0, 1), ("F", 2, 1, 2), ("F", 3, 2, 3), ("F", 4, 3, 4),
                  ("B", 1, 10, 12), ("B", 2, 13, 15), ("B", 3, 16, 18), ("B", 4, 19, 21)]
    got = [(b.stage, b.btype.name, b.start, b.duration) for b in product.extract_bubbles(tr)]
    assert got == [(1, "A", 0, 1), (2, "A", 0, 2), (3, "A", 0, 3), (0, "B", 4, 6), (1, "B", 4, 4),
                   (2, "B", 4, 2), (0, "C", 12, 1), (1, "C", 13, 1), (2, "C", 14, 1), (0, "C", 15, 1),
                   (3, "A", 15, 6), (1, "C", 16, 1), (2, "A", 17, 4), (0, "C", 18, 1), (1, "A", 19, 2)]
    assert [b.available_memory for b in product.extract_bubbles(tr)][:3] == [32.0, 36.0, 40.0]
    assert abs(product.bubble_rate(tr, product.extract_bubbles(tr)) - 3 / 7) < 1e-15


def test_appendix_a2_c1_trace(product):
    cfg = PipelineConfig(4, 4, [220], [347], 1, 48.0, product.default_stage_memory(4, 48.0, 20.0, 6.5))
    tr = product.build_schedule(cfg)
    assert tr.epoch_spans == [(0, 3969)]
    bs = product.extract_bubbles(tr)
    assert sum(b.duration for b in bs) == 6804
    prof = product.profile_bubbles(cfg)
    assert [s.durations for s in prof.stages] == [[220, 220, 220, 1041], [220, 220, 220, 347, 694],
                                                  [220, 347, 440, 694], [660, 1041]]
    assert [s.available_memory for s in prof.stages] == [2.0, 8.5, 15.0, 21.5]
    big = PipelineConfig(8, 8, [220], [347], 1, 48.0, [4.0] * 8)
    t8 = product.build_schedule(big)
    assert t8.epoch_spans == [(0, 8505)]
    assert len(product.extract_bubbles(t8)) == 49
    assert abs(product.bubble_rate(t8, product.extract_bubbles(t8)) - 0.466667) < 1e-6


def test_appendix_a3_to_a5(product):
    assert product.program_directed_gate(0.05, 0.0304) == Gate.Run
    assert product.program_directed_gate(0.0304, 0.0304) == Gate.Yield
    rt = SideTaskRuntime(SideTaskSpec("t"), state=SideTaskState.Running)
    now, steps = 0, 0
    while True:  # 1 s bubble at 0.1 ms ticks, 304-tick steps, no overhead -> 32 steps
        d = product.iterative_run(rt, 10000, now, 0.0304, 1e-4, 304)
        if not d.run:
            break
        now, steps = d.step_end, steps + 1
    assert steps == 32 and now == 9728
    p = product.profile_task(SideTaskSpec("t", per_step_duration=304, memory_demand=2.63),
                             ProfileOptions(10, 0.0, 1e-4), 0)
    assert (p.est_per_step_duration, p.max_per_step_duration, p.est_memory) == (0.0304, 0.0304, 2.63)
    p = product.profile_task(SideTaskSpec("t", per_step_duration=304, memory_demand=2.63),
                             ProfileOptions(32, 0.1, 1e-4), 42)
    # Appendix A3 prints 0.030528125; the reference's double is 0.030528125000000003
    assert p.est_per_step_duration == 0.030528125000000003 and p.max_per_step_duration == 0.0332
    assert product.stream_seed(0, "t", "profile") == 3847494928280905648
    ws = product.workers([28.0, 32.0, 36.0, 40.0])
    assert product.select_worker(38, ws) == 3
    assert product.select_worker(40, ws) is None
    assert product.framework_enforce(None, 1000, 1100, 100) == Enforce.Kill
    assert product.framework_enforce(1050, 1000, 1100, 100) == Enforce.Ok
    assert product.framework_enforce(None, 1000, 1099, 100) == Enforce.Ok


def test_appendix_a6_breakdown_and_metrics(product):
    from paper_2409_06941_b200.bubblesim import (ActivityKind, ActivityRecord, AssignRecord, Bubble,
                                                 TaskWork)
    bubbles = [Bubble(0, 0, 4, 6, 8.0, BubbleType.B), Bubble(1, 0, 0, 1, 8.0, BubbleType.A),
               Bubble(1, 0, 4, 4, 8.0, BubbleType.B)]
    acts = [ActivityRecord(4, 5, "pr", 0, ActivityKind.Check), ActivityRecord(5, 8, "pr", 0, ActivityKind.Step),
            ActivityRecord(8, 9, "pr", 0, ActivityKind.Check)]
    bd = product.bubble_breakdown(2, [TaskProfile("pr", 0.01, 0.01, 2.0, 32)], bubbles,
                                  [AssignRecord(0, "pr", 0)], [], acts)
    assert (bd[0].used_by_side_tasks, bd[0].runtime_overhead, bd[0].idle_insufficient_time, bd[0].idle_oom) == (3, 2, 1, 0)
    assert bd[1].idle_oom == 5 and bd[1].total() == 5
    assert abs(product.time_increase(100, 101.1) - 0.011) < 1e-12
    assert abs(product.time_increase(100, 99.3) + 0.007) < 1e-12
    cb = product.cost_savings(3600.0, 0.011, [TaskWork("x", 100.0, 1000.0)])
    assert abs(cb.c_no_side - 3.96) < 1e-12 and abs(cb.c_extra - 0.04356) < 1e-12
    assert abs(cb.c_side_tasks - 0.018) < 1e-12 and abs(cb.s + 0.006454545) < 1e-8


def test_host_reference_fixture(product):
    with open(os.path.join(GOLD, "host_reference.json")) as f:
        gold = json.load(f)
    for name, g in gold.items():
        if not isinstance(g, dict):
            continue
        p, m, fp, bp, epochs, w, a = g["config"]
        cfg = PipelineConfig(p, m, [fp], [bp], epochs, 48.0, product.default_stage_memory(p, 48.0, w, a))
        tr = product.build_schedule(cfg)
        assert [[o.stage, int(o.kind), o.micro_batch, o.epoch, o.start, o.end] for o in tr.ops] == g["ops"], name
        assert [list(s) for s in tr.epoch_spans] == g["spans"]
        lb = product.extract_bubbles_linked(tr)
        assert [[b.bubble.stage, b.bubble.epoch, b.bubble.start, b.bubble.duration, b.bubble.available_memory,
                 int(b.bubble.btype), -1 if b.prev_op is None else b.prev_op,
                 -1 if b.next_op is None else b.next_op] for b in lb] == g["bubbles"], name
        assert product.bubble_rate(tr, [b.bubble for b in lb]) == g["rate"]
    assert product.stream_seed(0, "t", "profile") == gold["stream_seed_0_t_profile"]
