"""Where does the iterative interface lose bubble time?  Per bubble of one
harvest run: lead gap (bubble start -> first step start), inter-step gaps,
tail gap (last step end -> bubble end), overrun past the end."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_06941_b200 import gpu  # noqa: E402


def main():
    stage = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    h = gpu.Harness(num_stages=4, num_micro_batches=4, stage=stage, layers=6, hidden=2048, tokens=8192)
    ips = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    h.submit("image", gpu.ImageTask(batch=64, images_per_step=ips), profile_steps=16)
    h.run(3, True)
    h.reprofile("image")
    r = h.run(6, True)
    bubbles = h.timeline(1)
    steps = h.timeline(2)
    lead, tail, gaps, over, nsteps = [], [], [], [], []
    for a, b in bubbles:
        inb = [(x, y) for x, y in steps if x < b and y > a]
        if not inb:
            continue
        nsteps.append(len(inb))
        lead.append(inb[0][0] - a)
        tail.append(b - inb[-1][1])
        over.append(max(0.0, inb[-1][1] - b))
        gaps += [inb[i + 1][0] - inb[i][1] for i in range(len(inb) - 1)]
    us = lambda xs: {"mean_us": statistics.fmean(xs) * 1e6, "p50_us": statistics.median(xs) * 1e6} if xs else None
    print(json.dumps({"fill": r["used_s"] / r["bubble_s"], "bubbles": len(bubbles), "mean_bubble_ms":
                      statistics.fmean(b - a for a, b in bubbles) * 1e3, "steps_per_bubble": statistics.fmean(nsteps),
                      "step_us": statistics.median(y - x for x, y in steps) * 1e6, "lead": us(lead),
                      "tail": us(tail), "inter_step_gap": us(gaps), "overrun": us(over),
                      "dispatch_host_us": r["dispatch_host_us"], "profile": h.profile()["stage_bubble_ticks"] / 1e6}))
    h.close()


if __name__ == "__main__":
    main()
