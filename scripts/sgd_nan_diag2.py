"""Standalone long SGD runs (no harness): RMSE every 5 epochs, steps of `step` edges."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_06941_b200 import gpu  # noqa: E402


def main():
    for spec in sys.argv[1:]:
        mode, step, *w = spec.split(":")
        step, wrap = int(step), bool(w)
        p = gpu.SgdProblem(V=300000, E=6000000, k=16, edge_seed=2, init_seed=3, by_user=mode != "coo",
                           window=step)
        out = []
        cur = 0
        for ep in range(60):
            if wrap:   # the task's cursor: steps straddle epochs
                for _ in range(-(-p.E // step)):
                    left = step
                    while left > 0:
                        n = min(left, p.E - cur)
                        p.step(cur, cur + n, 0.01, 0.05)
                        cur, left = (cur + n) % p.E, left - n
            else:
                c = 0
                while c < p.E:
                    n = min(step, p.E - c)
                    p.step(c, c + n, 0.01, 0.05)
                    c += n
            if ep % 5 == 4:
                out.append(round(p.rmse(), 4))
        print(spec, out, flush=True)


if __name__ == "__main__":
    main()
