"""K1/K2 PageRank on the B200 vs the CPU oracle: identical graph (bit-exact
CSR), ranks within L1 <= 1e-6 after a fixed iteration count (north star)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    from paper_2409_06941_b200 import gpu
    gpu.glib()
    return gpu


@pytest.fixture(scope="module")
def rmat20(g, sidetask_oracle):
    graph = g.PageRankGraph(scale=20, edge_factor=16, seed=1)
    src, dst = sidetask_oracle.rmat_edges(20, 16, seed=1)
    csr = sidetask_oracle.build_pull_csr(1 << 20, src, dst)
    return graph, csr


@pytest.mark.parametrize("scale,ef,seed", [(1, 4, 3), (6, 8, 2), (12, 16, 5)])
def test_graph_build_matches_oracle_small(g, sidetask_oracle, scale, ef, seed):
    graph = g.PageRankGraph(scale=scale, edge_factor=ef, seed=seed)
    src, dst = sidetask_oracle.rmat_edges(scale, ef, seed=seed)
    off, col, outdeg = sidetask_oracle.build_pull_csr(1 << scale, src, dst)
    o2, c2, d2 = (t.cpu().numpy() for t in graph.csr())
    assert graph.E == len(col)
    assert np.array_equal(o2, off) and np.array_equal(c2, col) and np.array_equal(d2, outdeg)


def test_graph_build_matches_oracle_scale20(rmat20):
    graph, (off, col, outdeg) = rmat20
    o2, c2, d2 = (t.cpu().numpy() for t in graph.csr())
    assert graph.V == 1 << 20 and graph.E == len(col)
    assert np.array_equal(o2, off) and np.array_equal(c2, col) and np.array_equal(d2, outdeg)
    assert (outdeg == 0).mean() > 0.3  # RMAT: dangling-heavy, the dropped-mass rule matters


@pytest.mark.parametrize("iters", [1, 20])
def test_ranks_l1_scale20(g, sidetask_oracle, rmat20, iters):
    graph, (off, col, outdeg) = rmat20
    st = g.PageRankState(graph)
    st.reset()
    st.step(iters, 0.85)
    got = st.ranks().double().cpu().numpy()
    want = sidetask_oracle.pr_run(off, col, outdeg, iters, 0.85)
    l1 = np.abs(got - want).sum()
    assert l1 <= 1e-6, l1
    assert want.sum() < 1.0  # dangling mass dropped, not redistributed


def test_ranks_l1_small_and_stepwise(g, sidetask_oracle):
    graph = g.PageRankGraph(scale=14, edge_factor=8, seed=9)
    src, dst = sidetask_oracle.rmat_edges(14, 8, seed=9)
    off, col, outdeg = sidetask_oracle.build_pull_csr(1 << 14, src, dst)
    st = g.PageRankState(graph)
    st.reset()
    for _ in range(7):      # 7 steps of 3 iterations == 21 iterations
        st.step(3, 0.85)
    got = st.ranks().double().cpu().numpy()
    want = sidetask_oracle.pr_run(off, col, outdeg, 21, 0.85)
    assert np.abs(got - want).sum() <= 1e-6


def test_pagerank_task_in_bubbles(g, sidetask_oracle):
    h = g.Harness(num_stages=4, num_micro_batches=4, stage=2, layers=2, profile_reps=2,
                  profile_epochs=1)
    task = g.PageRankTask(scale=16, edge_factor=16, seed=4, iters_per_step=2)
    ok, prof = h.submit("pagerank", task, profile_steps=8)
    assert ok
    h.run(2, True)
    r = h.run(2, True)
    assert r["steps_completed"] > 0
    ranks, iters = task.ranks()
    assert iters > 0 and iters % 2 == 0
    src, dst = sidetask_oracle.rmat_edges(16, 16, seed=4)
    off, col, outdeg = sidetask_oracle.build_pull_csr(1 << 16, src, dst)
    want = sidetask_oracle.pr_run(off, col, outdeg, iters, 0.85)
    assert np.abs(ranks.double().cpu().numpy() - want).sum() <= 1e-6
    h.close()


def test_damping_change_rewrites_constant_rows(g, sidetask_oracle, rmat20):
    """The zero-in-degree rows' rank (1-d)/V is written only while it may
    change: after a reset and after a damping change (two launches each)."""
    graph, (off, col, outdeg) = rmat20
    st = g.PageRankState(graph)
    st.reset()
    st.step(3, 0.85)
    st.step(1, 0.6)
    st.step(3, 0.6)
    got = st.ranks().double().cpu().numpy()
    want = sidetask_oracle.pr_run(off, col, outdeg, 3, 0.85)
    want = sidetask_oracle.pr_run(off, col, outdeg, 4, 0.6, r0=want)
    assert np.abs(got - want).sum() <= 1e-6


def test_reset_restarts(g, sidetask_oracle):
    graph = g.PageRankGraph(scale=16, edge_factor=16, seed=11)
    src, dst = sidetask_oracle.rmat_edges(16, 16, seed=11)
    off, col, outdeg = sidetask_oracle.build_pull_csr(1 << 16, src, dst)
    st = g.PageRankState(graph)
    st.reset()
    st.step(5, 0.85)
    st.reset()
    st.step(2, 0.85)
    want = sidetask_oracle.pr_run(off, col, outdeg, 2, 0.85)
    assert np.abs(st.ranks().double().cpu().numpy() - want).sum() <= 1e-6


def _edge_cases():
    rng = np.random.default_rng(7)
    V = 5000
    src = rng.integers(0, V, 60000, dtype=np.int32)
    dst = ((src + rng.zipf(1.6, 60000).astype(np.int64)) % V).astype(np.int32)   # skewed, with dups
    src[:100] = dst[:100]                                                       # self loops
    return [
        ("random_skewed", V, src, dst),
        ("single_vertex", 1, np.zeros(0, np.int32), np.zeros(0, np.int32)),
        ("only_self_loops", 3, np.array([0, 1, 2], np.int32), np.array([0, 1, 2], np.int32)),
        ("star_in", 70000, np.arange(1, 70000, dtype=np.int32), np.zeros(69999, np.int32)),   # one split row
        ("chain_odd_V", 1001, np.arange(1000, dtype=np.int32), np.arange(1, 1001, dtype=np.int32)),
        ("duplicates", 4, np.array([0, 0, 0, 1, 3, 3], np.int32), np.array([1, 1, 1, 2, 0, 0], np.int32)),
    ]


@pytest.mark.parametrize("case", _edge_cases(), ids=lambda c: c[0])
def test_from_edges_matches_oracle(g, sidetask_oracle, case):
    """fr_pr_graph_from_edges: the caller's graph (duplicates, self loops, an
    isolated-only graph, a hub row split across CTAs, odd V) builds the
    oracle's CSR and ranks within L1 <= 1e-6 after 20 iterations"""
    _, V, src, dst = case
    gr = g.PageRankGraph.from_edges(V, src, dst)
    off, col, outdeg = sidetask_oracle.build_pull_csr(V, src, dst)
    o, c, d = (t.cpu().numpy() for t in gr.csr())
    assert np.array_equal(o, off) and np.array_equal(c, col) and np.array_equal(d, outdeg)
    st = g.PageRankState(gr)
    st.reset()
    st.step(20, 0.85)
    got = st.ranks().double().cpu().numpy()
    want = sidetask_oracle.pr_run(off, col, outdeg, 20, 0.85)
    assert np.abs(got - want).sum() <= 1e-6


def test_from_edges_rejects_bad_ids(g):
    with pytest.raises(Exception):
        g.PageRankGraph.from_edges(10, np.array([0, 10], np.int32), np.array([1, 2], np.int32))
    with pytest.raises(Exception):
        g.PageRankGraph.from_edges(10, np.array([0, -1], np.int32), np.array([1, 2], np.int32))


def test_task_over_caller_graph_in_bubbles(g, sidetask_oracle):
    """fr_pagerank_task_create_from_graph: the harvested task over a
    caller-built graph reaches the oracle's ranks for its iteration count"""
    rng = np.random.default_rng(11)
    V = 20000
    src = rng.integers(0, V, 200000, dtype=np.int32)
    dst = ((src.astype(np.int64) * 7 + rng.zipf(1.5, 200000)) % V).astype(np.int32)
    graph = g.PageRankGraph.from_edges(V, src, dst)
    task = g.PageRankTask(graph=graph, iters_per_step=1)
    del graph   # the task keeps its own copy of the step arrays
    assert task.V == V and task.units_per_step == task.E
    h = g.Harness(num_stages=4, num_micro_batches=4, stage=1, layers=2, profile_reps=2, profile_epochs=1)
    ok, _ = h.submit("pr", task, profile_steps=4)
    assert ok
    h.run(2, True)
    ranks, iters = task.ranks()
    assert iters > 0
    off, col, outdeg = sidetask_oracle.build_pull_csr(V, src, dst)
    want = sidetask_oracle.pr_run(off, col, outdeg, iters, 0.85)
    assert np.abs(ranks.double().cpu().numpy() - want).sum() <= 1e-6
    h.close()

