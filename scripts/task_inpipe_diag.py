"""Per-step device durations of a side task inside the bubbles of one stage
(bench shapes) vs the same steps run alone; also split by position in the
bubble (first step after BubbleStarted vs the rest).
Usage: python scripts/task_inpipe_diag.py {sgd|pagerank|image}"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2409_06941_b200 import gpu  # noqa: E402


def make(name):
    if name == "sgd":
        return gpu.SgdTask(edges_per_step=1 << 21)
    if name == "pagerank":
        return gpu.PageRankTask(scale=20, iters_per_step=1)
    return gpu.ImageTask(batch=64, images_per_step=16)


def pct(xs):
    xs = sorted(xs)
    return {"p10_us": xs[len(xs) // 10] * 1e6, "p50_us": xs[len(xs) // 2] * 1e6,
            "p90_us": xs[9 * len(xs) // 10] * 1e6, "n": len(xs)} if xs else None


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "sgd"
    h = gpu.Harness(num_stages=4, num_micro_batches=4, stage=1, layers=6, hidden=2048, tokens=8192)
    task = make(name)
    ok, prof = h.submit(name, task, profile_steps=16)
    h.run(3, True)
    h.run(4, True)
    bubbles, steps = h.timeline(1), h.timeline(2)
    first, rest = [], []
    for a, b in bubbles:
        inb = [(x, y) for x, y in steps if x < b and y > a]
        if inb:
            first.append(inb[0][1] - inb[0][0])
            rest += [y - x for x, y in inb[1:]]
    out = {"task": name, "standalone_profile_us": prof["est_per_step_duration"] * 1e6,
           "first_in_bubble": pct(first), "rest_in_bubble": pct(rest)}
    h.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
