"""Margin of the Graph-SGD RMSE parity (|GPU - sequential oracle| per epoch)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import sidetasks_oracle  # noqa: E402  (checker)
from paper_2409_06941_b200 import gpu  # noqa: E402

o = sidetasks_oracle.load()
V, E = 200000, 8000000
u, v, r = o.sgd_edges(V, E, seed=2)
want = []
L = o.sgd_init(V, 16, seed=3)
for ep in range(3):
    o.sgd_epoch(u, v, r, L, 0.01, 0.05, nthreads=1)
    want.append(o.sgd_rmse(u, v, r, L))
for rep in range(4):
    p = gpu.SgdProblem(V=V, E=E, k=16, edge_seed=2, init_seed=3)
    got = []
    for ep in range(3):
        p.epoch(0.01, 0.05)
        got.append(p.rmse())
    print([f"{g - w:+.2e}" for g, w in zip(got, want)], [f"{w:.4f}" for w in want])
