"""K3/K4 Graph-SGD on the B200 vs the CPU oracle: identical inputs (bit-exact
edges and initial factors), RMSE within 1e-3 after a fixed epoch count
(north star), K4 RMSE reduction equal to the oracle's on the same factors."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ETA, LAM = 0.01, 0.05


@pytest.fixture(scope="module")
def g():
    from paper_2409_06941_b200 import gpu
    gpu.glib()
    return gpu


@pytest.mark.parametrize("V,E,k", [(7, 50, 4), (1000, 20000, 16), (50000, 400000, 32)])
def test_inputs_match_oracle(g, sidetask_oracle, V, E, k):
    p = g.SgdProblem(V=V, E=E, k=k, edge_seed=11, init_seed=12)
    u, v, r = (t.cpu().numpy() for t in p.edges())
    ou, ov, orr = sidetask_oracle.sgd_edges(V, E, seed=11)
    assert np.array_equal(u, ou) and np.array_equal(v, ov) and np.array_equal(r, orr)
    assert np.array_equal(p.latent().cpu().numpy(), sidetask_oracle.sgd_init(V, k, seed=12))


def test_rmse_parity_medium(g, sidetask_oracle):
    V, E = 200000, 8000000
    p = g.SgdProblem(V=V, E=E, k=16, edge_seed=2, init_seed=3)
    u, v, r = sidetask_oracle.sgd_edges(V, E, seed=2)
    L = sidetask_oracle.sgd_init(V, 16, seed=3)
    assert abs(p.rmse() - sidetask_oracle.sgd_rmse(u, v, r, L)) < 1e-9   # K4 on equal factors
    for ep in range(3):
        p.epoch(ETA, LAM)
        sidetask_oracle.sgd_epoch(u, v, r, L, ETA, LAM, nthreads=1)     # sequential reference
        got, want = p.rmse(), sidetask_oracle.sgd_rmse(u, v, r, L)
        assert abs(got - want) <= 1e-3, (ep, got, want)
    # K4 parity on the GPU's own factors
    Lg = p.latent().cpu().numpy()
    assert abs(p.rmse() - sidetask_oracle.sgd_rmse(u, v, r, Lg)) < 1e-9


def test_rmse_parity_orkut_shape(g, sidetask_oracle):
    """configs[2] at full size: 3,072,441 vertices, 117,185,083 edges, rank 16."""
    V, E = 3072441, 117185083
    p = g.SgdProblem(V=V, E=E, k=16, edge_seed=2, init_seed=3)
    u, v, r = sidetask_oracle.sgd_edges(V, E, seed=2)
    gu, gv, gr = (t.cpu().numpy() for t in p.edges())
    assert np.array_equal(gu, u) and np.array_equal(gv, v) and np.array_equal(gr, r)
    del gu, gv, gr
    L = sidetask_oracle.sgd_init(V, 16, seed=3)
    r0 = p.rmse()
    prev = r0
    for ep in range(2):
        p.epoch(ETA, LAM)
        sidetask_oracle.sgd_epoch(u, v, r, L, ETA, LAM, nthreads=0)  # Hogwild on all host cores
        got, want = p.rmse(), sidetask_oracle.sgd_rmse(u, v, r, L)
        assert abs(got - want) <= 1e-3, (ep, got, want)
        assert got < prev
        prev = got


@pytest.mark.parametrize("V,E,k,window", [(7, 50, 16, 1 << 21), (1000, 20000, 16, 1000), (50000, 400000, 32, 65536),
                                          (3000, 100000, 8, 7), (200000, 1000000, 128, 1 << 16),
                                          (3072441, 117185083, 16, 1 << 21)])
def test_by_user_layout_matches_oracle(g, sidetask_oracle, V, E, k, window):
    """fr_sgd_group_by_user == the oracle's layout (stable by u, pieces dealt over rounds), bit-exact."""
    p = g.SgdProblem(V=V, E=E, k=k, edge_seed=11, init_seed=12, by_user=True, window=window)
    u, v, r = (t.cpu().numpy() for t in p.edges())
    ou, ov, orr = sidetask_oracle.sgd_group_by_user(V, *sidetask_oracle.sgd_edges(V, E, seed=11), window=window, k=k)
    assert np.array_equal(u, ou) and np.array_equal(v, ov) and np.array_equal(r, orr)


@pytest.mark.parametrize("V,E,k", [(200000, 8000000, 16), (50000, 2000000, 32)])
def test_by_user_rmse_parity(g, sidetask_oracle, V, E, k):
    """user-grouped kernel vs the sequential oracle over the same layout:
    |dRMSE| <= 1e-3 after the fixed epoch count (3).  The first epoch is
    looser (measured 2.5e-3 at 200k x 8M): sequential by-user order is an
    outlier trajectory -- every user's whole run sees the item rows already
    updated by all lower users -- which no parallel schedule reproduces; the
    two converge from the second epoch (3.3e-4, 2.7e-4)."""
    p = g.SgdProblem(V=V, E=E, k=k, edge_seed=2, init_seed=3, by_user=True)
    u, v, r = sidetask_oracle.sgd_group_by_user(V, *sidetask_oracle.sgd_edges(V, E, seed=2), k=k)
    L = sidetask_oracle.sgd_init(V, k, seed=3)
    for ep in range(3):
        p.epoch(ETA, LAM)
        sidetask_oracle.sgd_epoch(u, v, r, L, ETA, LAM, nthreads=1)
        got, want = p.rmse(), sidetask_oracle.sgd_rmse(u, v, r, L)
        assert abs(got - want) <= (1e-3 if ep == 2 else 4e-3), (ep, got, want)


def test_by_user_ragged_steps(g, sidetask_oracle):
    """steps over ragged edge ranges (runs and segments cut at arbitrary
    edges, steps straddling the layout's rounds) track the sequential oracle
    like a whole-epoch launch does"""
    V, E = 50000, 2000003
    p = g.SgdProblem(V=V, E=E, k=16, edge_seed=5, init_seed=6, by_user=True, window=1 << 18)
    u, v, r = sidetask_oracle.sgd_group_by_user(V, *sidetask_oracle.sgd_edges(V, E, seed=5), window=1 << 18)
    L = sidetask_oracle.sgd_init(V, 16, seed=6)
    r0 = p.rmse()
    cuts = [0, 1, 7, 1000, 77777, 1 << 20, E - 3, E]
    for ep in range(3):
        for x, y in zip(cuts, cuts[1:]):
            p.step(x, y, ETA, LAM)
        sidetask_oracle.sgd_epoch(u, v, r, L, ETA, LAM, nthreads=1)
        got, want = p.rmse(), sidetask_oracle.sgd_rmse(u, v, r, L)
        assert got < r0 and abs(got - want) <= (1e-3 if ep == 2 else 4e-3), (ep, got, want)


def test_by_user_long_run_stays_finite(g):
    """task-like stepping (2^19-edge steps straddling epochs) for 40 epochs:
    the held-row refresh keeps hub rows from overshooting (whole-run holds
    diverged to NaN here)"""
    V, E, step = 300000, 6000000, 1 << 19
    p = g.SgdProblem(V=V, E=E, k=16, edge_seed=2, init_seed=3, by_user=True, window=step)
    cur = 0
    for _ in range(40 * E // step):
        left = step
        while left > 0:
            n = min(left, E - cur)
            p.step(cur, cur + n, ETA, LAM)
            cur, left = (cur + n) % E, left - n
    rm = p.rmse()
    assert np.isfinite(rm) and rm < 1.0, rm   # 0.78 measured (sequential oracle: 0.76)


def test_rmse_parity_orkut_shape_by_user(g, sidetask_oracle):
    """configs[2] at full size in the user-grouped layout (the task's default)."""
    V, E = 3072441, 117185083
    p = g.SgdProblem(V=V, E=E, k=16, edge_seed=2, init_seed=3, by_user=True)
    u, v, r = sidetask_oracle.sgd_group_by_user(V, *sidetask_oracle.sgd_edges(V, E, seed=2))
    L = sidetask_oracle.sgd_init(V, 16, seed=3)
    prev = p.rmse()
    for ep in range(2):
        p.epoch(ETA, LAM)
        sidetask_oracle.sgd_epoch(u, v, r, L, ETA, LAM, nthreads=0)
        got, want = p.rmse(), sidetask_oracle.sgd_rmse(u, v, r, L)
        print("orkut by_user", ep, got, want)
        assert abs(got - want) <= (1e-3 if ep == 1 else 4e-3), (ep, got, want)
        assert got < prev
        prev = got


def test_sgd_task_in_bubbles(g):
    h = g.Harness(num_stages=4, num_micro_batches=4, stage=3, layers=2, profile_reps=2,
                  profile_epochs=1)
    task = g.SgdTask(V=300000, E=6000000, k=16, edges_per_step=1 << 19)   # by-user layout (default)
    ok, prof = h.submit("sgd", task, profile_steps=8)
    assert ok and prof["est_per_step_duration"] > 0
    h.run(2, True)
    r = h.run(3, True)
    assert r["steps_completed"] > 0
    prob, epochs = task.problem()
    assert prob.rmse() < 3.0   # from ~3.1 at init
    h.close()


@pytest.mark.parametrize("by_user", [False, True])
def test_from_edges_matches_oracle(g, sidetask_oracle, by_user):
    """the caller's ratings (a bipartite users x items shape, items power-law
    with the top one in 1 % of all ratings): same inputs, RMSE within 1e-3 of
    the sequential oracle after 3 epochs"""
    rng = np.random.default_rng(3)
    U, I, E = 40000, 10000, 1500000
    u = rng.integers(0, U, E, dtype=np.int32)
    v = (U + np.floor(I * rng.random(E) ** 2)).astype(np.int32)
    r = rng.integers(1, 6, E).astype(np.float32)
    V = U + I
    p = g.SgdProblem.from_edges(V, u, v, r, k=16, init_seed=5, by_user=by_user)
    ou, ov, orr = u.copy(), v.copy(), r.copy()
    if by_user:
        sidetask_oracle.sgd_group_by_user(V, ou, ov, orr)
    gu, gv, gr = (t.cpu().numpy() for t in p.edges())
    assert np.array_equal(gu, ou) and np.array_equal(gv, ov) and np.array_equal(gr, orr)
    L = sidetask_oracle.sgd_init(V, 16, seed=5)
    assert np.array_equal(p.latent().cpu().numpy(), L)
    for ep in range(3):
        p.epoch(ETA, LAM)
        sidetask_oracle.sgd_epoch(ou, ov, orr, L, ETA, LAM, nthreads=1)
    got, want = p.rmse(), sidetask_oracle.sgd_rmse(ou, ov, orr, L)
    assert abs(got - want) <= 1e-3, (got, want)


@pytest.mark.parametrize("by_user", [False, True])
def test_extreme_hub_stays_finite(g, sidetask_oracle, by_user):
    """a Zipf(1.3) item holding a quarter of all ratings: the hub cap on edges
    in flight keeps Hogwild from diverging (without it: NaN after one epoch)"""
    rng = np.random.default_rng(4)
    U, I, E = 40000, 10000, 1500000
    u = rng.integers(0, U, E, dtype=np.int32)
    v = (U + rng.zipf(1.3, E) % I).astype(np.int32)
    r = rng.integers(1, 6, E).astype(np.float32)
    V = U + I
    p = g.SgdProblem.from_edges(V, u, v, r, k=16, init_seed=5, by_user=by_user)
    r0 = p.rmse()
    for _ in range(3):
        p.epoch(ETA, LAM)
    rm = p.rmse()
    ou, ov, orr = u.copy(), v.copy(), r.copy()
    if by_user:
        sidetask_oracle.sgd_group_by_user(V, ou, ov, orr)
    L = sidetask_oracle.sgd_init(V, 16, seed=5)
    for _ in range(3):
        sidetask_oracle.sgd_epoch(ou, ov, orr, L, ETA, LAM, nthreads=1)
    want = sidetask_oracle.sgd_rmse(ou, ov, orr, L)
    print("extreme hub", by_user, r0, rm, want)
    assert np.isfinite(rm) and rm < r0 and abs(rm - want) <= 1e-2, (r0, rm, want)


def test_from_edges_rejects_bad_ids(g):
    with pytest.raises(Exception):
        g.SgdProblem.from_edges(10, np.array([0, 10], np.int32), np.array([1, 2], np.int32),
                                np.array([1, 2], np.float32))


def test_task_over_caller_ratings_in_bubbles(g):
    """fr_sgd_task_create_from_problem: the harvested task over the caller's
    ratings (re-laid out by user) lowers the RMSE"""
    rng = np.random.default_rng(12)
    U, I, E = 30000, 8000, 2000000
    u = rng.integers(0, U, E, dtype=np.int32)
    v = (U + np.floor(I * rng.random(E) ** 2)).astype(np.int32)
    r = rng.integers(1, 6, E).astype(np.float32)
    prob = g.SgdProblem.from_edges(U + I, u, v, r, k=16, init_seed=5)
    r0 = prob.rmse()
    task = g.SgdTask(problem=prob, edges_per_step=1 << 18)
    assert task.units_per_step == 1 << 18
    h = g.Harness(num_stages=4, num_micro_batches=4, stage=2, layers=2, profile_reps=2, profile_epochs=1)
    ok, _ = h.submit("sgd-user", task, profile_steps=4)
    assert ok
    run = h.run(3, True)
    assert run["steps_completed"] > 0
    p2, epochs = task.problem()
    assert p2.rmse() < r0
    h.close()



# ---- the benchmarked Graph-SGD path (bench.py SGD: by-user layout, rounds of
# 2^22 edges, overlapping PDL steps, step groups of 3) at the Orkut shape for
# SURVEY §8(d) C3's 5 epochs, against the sequential oracle in the same layout
BENCH_STEP = 1 << 22
ORKUT = (3072441, 117185083)


@pytest.fixture(scope="module")
def orkut_oracle_rmse(sidetask_oracle):
    """RMSE of the sequential oracle after each of 5 epochs (by-user layout, rounds of 2^22 edges)"""
    V, E = ORKUT
    u, v, r = sidetask_oracle.sgd_group_by_user(V, *sidetask_oracle.sgd_edges(V, E, seed=2), window=BENCH_STEP)
    L = sidetask_oracle.sgd_init(V, 16, seed=3)
    out = []
    for _ in range(5):
        sidetask_oracle.sgd_epoch(u, v, r, L, ETA, LAM, nthreads=1)
        out.append(sidetask_oracle.sgd_rmse(u, v, r, L))
    return out


def test_overlapped_task_steps_match_oracle_orkut(g, orkut_oracle_rmse):
    """standalone: the task's stepping (2^22-edge steps straddling epochs,
    fr_sgd_problem_set_overlap(1), back to back on one low-priority stream)
    for exactly 5 epochs: |dRMSE| <= 1e-3 vs the sequential oracle after
    every epoch (measured <= 5e-5: with rounds of 2^22 edges a round holds
    about one 64-edge piece of any user, so the epoch-1 by-user outlier of
    small windows does not arise)"""
    import torch
    V, E = ORKUT
    p = g.SgdProblem(V=V, E=E, k=16, edge_seed=2, init_seed=3, by_user=True, window=BENCH_STEP)
    p.set_overlap(True)
    s = g.low_priority_stream()
    cur, ep, got = 0, 0, []
    while ep < 5:
        left = BENCH_STEP
        while left > 0 and ep < 5:
            n = min(left, E - cur)
            p.step(cur, cur + n, ETA, LAM, stream=s)
            cur, left = cur + n, left - n
            if cur == E:
                cur, ep = 0, ep + 1
                torch.cuda.current_stream().wait_stream(s)
                got.append(p.rmse())   # breaks the PDL chain: the next step waits for it
    print("overlapped orkut", got, orkut_oracle_rmse)
    for e in range(5):
        assert abs(got[e] - orkut_oracle_rmse[e]) <= 1e-3, (e, got[e], orkut_oracle_rmse[e])


def test_sgd_task_in_bubbles_bench_settings_orkut(g, orkut_oracle_rmse):
    """the in-bubble task exactly as bench.py runs it (stage of the
    nanoGPT-1.2B-shaped 4-stage pipeline, step groups of 3, 2^22-edge
    overlapping steps) until it completes 5 epochs: RMSE within 1e-3 of the
    sequential oracle after 5 epochs"""
    V, E = ORKUT
    h = g.Harness(num_stages=4, num_micro_batches=4, stage=0, layers=6, hidden=2048, tokens=8192,
                  ffn_mult=4, step_group=3, profile_epochs=1, profile_reps=2)
    task = g.SgdTask(V=V, E=E, k=16, edges_per_step=BENCH_STEP, total_epochs=5)
    ok, _ = h.submit("sgd", task, profile_steps=8)
    assert ok
    steps = 0
    for _ in range(30):
        r = h.run(2, True)
        steps += r["steps_completed"]
        if h.task_status("sgd")["disposition"] == "completed":
            break
    st = h.task_status("sgd")
    assert st["disposition"] == "completed", (st, steps)
    prob, epochs = task.problem()
    assert epochs == 5
    got = prob.rmse()
    print("in-bubble orkut", steps, got, orkut_oracle_rmse[4])
    assert abs(got - orkut_oracle_rmse[4]) <= 1e-3, (got, orkut_oracle_rmse[4])
    h.close()
