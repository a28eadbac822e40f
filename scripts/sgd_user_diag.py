"""Diagnostics for the user-grouped SGD step: RMSE per epoch vs the sequential
oracle (same order) for small/medium shapes, and a single-group case that must
track the sequential order closely."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2409_06941_b200 import gpu  # noqa: E402
from oracle import sidetasks_oracle  # noqa: E402

ETA, LAM = 0.01, 0.05


def run(orc, V, E, k, epochs, by_user, window=1 << 21):
    p = gpu.SgdProblem(V=V, E=E, k=k, edge_seed=2, init_seed=3, by_user=by_user, window=window)
    u, v, r = orc.sgd_edges(V, E, seed=2)
    if by_user:
        u, v, r = orc.sgd_group_by_user(V, u, v, r, window=window)
    L = orc.sgd_init(V, k, seed=3)
    out = []
    for _ in range(epochs):
        p.epoch(ETA, LAM)
        orc.sgd_epoch(u, v, r, L, ETA, LAM, nthreads=1)
        Lg = p.latent().cpu().numpy()
        out.append((round(p.rmse(), 6), round(orc.sgd_rmse(u, v, r, L), 6),
                    float(np.abs(Lg - L).max()), bool(np.isfinite(Lg).all())))
    print(dict(V=V, E=E, k=k, by_user=by_user, window=window, epochs=out), flush=True)


def main():
    orc = sidetasks_oracle.load()
    for V, E in [(2000, 100000), (200000, 8000000)]:
        run(orc, V, E, 16, 3, False)
        for w in (1 << 30, 1 << 21, 1 << 18):
            run(orc, V, E, 16, 3, True, w)


if __name__ == "__main__":
    main()
