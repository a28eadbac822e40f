"""Gap kernel at the driver-default carveout: does a smem-hungry task (PageRank,
192 KB per CTA) still run at speed in bubbles after a max-L1 task (SGD) left
the SMs in the L1-heavy split?  One harness, SGD then PageRank."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_06941_b200 import gpu  # noqa: E402


def main():
    h = gpu.Harness(num_stages=4, num_micro_batches=4, stage=1, layers=6, hidden=2048, tokens=8192)
    out = {}
    for name, task in (("sgd", gpu.SgdTask(edges_per_step=1 << 21)), ("pagerank", gpu.PageRankTask(iters_per_step=1)),
                       ("sgd2", gpu.SgdTask(edges_per_step=1 << 21))):
        ok, prof = h.submit(name, task, profile_steps=8)
        h.run(2, True)
        r = h.run(3, True)
        steps = [b - a for a, b in h.timeline(2)]
        out[name] = {"standalone_us": prof["est_per_step_duration"] * 1e6,
                     "in_bubble_p50_us": statistics.median(steps) * 1e6, "max_us": max(steps) * 1e6,
                     "fill": r["used_s"] / r["bubble_s"], "overrun_s": r["overrun_s"]}
        h.stop_task(name)
    h.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
