"""Is the in-bubble slowdown of a side-task step caused by the pipeline's GEMM
load (power state, caches) or by the harness itself?  Same bubble schedule
(fp/bp overridden to the bench stage's 3.3 / 6.5 ms) with tiny stand-in ops,
so the GPU is otherwise idle.  Usage: harness_idle_diag.py {sgd|image|pagerank}"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_06941_b200 import gpu  # noqa: E402
from task_inpipe_diag import make  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "sgd"
    inflight = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    h = gpu.Harness(num_stages=4, num_micro_batches=4, stage=1, layers=1, hidden=512, tokens=1024,
                    fp_ticks=3_300_000, bp_ticks=6_500_000, profile_epochs=1, max_inflight_steps=inflight)
    task = make(name)
    ok, prof = h.submit(name, task, profile_steps=16)
    h.run(2, True)
    h.run(3, True)
    steps = [b - a for a, b in h.timeline(2)]
    print(json.dumps({"task": name, "inflight": inflight, "standalone_us": prof["est_per_step_duration"] * 1e6,
                      "in_bubble_idle_gpu_p50_us": statistics.median(steps) * 1e6, "n": len(steps)}))
    h.close()


if __name__ == "__main__":
    main()
