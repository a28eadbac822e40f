"""Probe: does an item-blocked order (edges sorted by (v block, u), each
block's L_v rows L2-sized) make the user-grouped SGD step faster at the Orkut
shape?  Times 2^21-edge steps of the user kernel over several orders."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import sidetasks_oracle  # noqa: E402
from paper_2409_06941_b200 import gpu  # noqa: E402
from paper_2409_06941_b200.gpu import check  # noqa: E402


def time_steps(p, chunk=1 << 21, reps=20):
    s = gpu.low_priority_stream()
    n = p.E // chunk
    for i in range(3):
        p.step(i * chunk, (i + 1) * chunk, stream=s)
    s.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for i, (a, b) in enumerate(ev):
        j = (i * 7 + 3) % n
        a.record(s)
        p.step(j * chunk, (j + 1) * chunk, stream=s)
        b.record(s)
    s.synchronize()
    return statistics.median(a.elapsed_time(b) * 1e3 for a, b in ev)


def main():
    orc = sidetasks_oracle.load()
    V, E = 3072441, 117185083
    u, v, r = orc.sgd_edges(V, E, seed=2)
    base = gpu.SgdProblem(V=V, E=E, k=16, edge_seed=2, init_seed=3, by_user=True)
    print("by_user rounds:", time_steps(base), "us", flush=True)
    del base
    for P in [int(x) for x in sys.argv[1:]] or [2, 4, 8]:
        blk = (v.astype(np.int64) * P) // V
        o = np.lexsort((u, blk))            # by block, then by u (stable)
        p = gpu.SgdProblem.from_edges(V, u[o], v[o], r[o], k=16, init_seed=3)
        check(gpu.glib().fr_sgd_problem_set_kernel(p._h, 1))
        t = time_steps(p)
        uu = u[o]
        runs = 1 + int(np.count_nonzero(uu[1:] != uu[:-1]))
        print(f"P={P}: {t:.1f} us per 2^21-edge step, mean run {E / runs:.1f} edges, "
              f"L_v block {V // P * 64 / 2**20:.0f} MiB", flush=True)
        del p


if __name__ == "__main__":
    main()
