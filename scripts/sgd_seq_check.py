"""With FR_SGD_CONFLICT_DIV huge the step runs as ONE lane group, i.e. in the
layout's sequential order: compare with the sequential oracle edge-for-edge
(task-like wrapping steps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import sidetasks_oracle  # noqa: E402
from paper_2409_06941_b200 import gpu  # noqa: E402


def main():
    orc = sidetasks_oracle.load()
    V, E, step = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    by_user = sys.argv[4] == "user"
    p = gpu.SgdProblem(V=V, E=E, k=16, edge_seed=2, init_seed=3, by_user=by_user, window=step)
    u, v, r = orc.sgd_edges(V, E, seed=2)
    if by_user:
        u, v, r = orc.sgd_group_by_user(V, u, v, r, window=step)
    L = orc.sgd_init(V, 16, seed=3)
    cur = 0
    for k in range(int(sys.argv[5])):
        left = step
        while left > 0:
            n = min(left, E - cur)
            p.step(cur, cur + n, 0.01, 0.05)
            orc.lib.orc_sgd_epoch(n, u[cur:], v[cur:], r[cur:], L.reshape(-1), 16, 0.01, 0.05, 1)
            cur, left = (cur + n) % E, left - n
        Lg = p.latent().cpu().numpy()
        d = np.abs(Lg - L)
        print(k, "cur", cur, "maxdiff", float(d.max()), "row", int(d.max(1).argmax()), "nan", int(np.isnan(Lg).sum()),
              flush=True)


if __name__ == "__main__":
    main()
