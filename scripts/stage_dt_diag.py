"""Where does a stage's ΔT come from?  Per op of one harness run with the image
side task vs the same run without: start lateness relative to the epoch's
first op, and duration growth (GEMMs slower after busy bubbles).

Usage: python scripts/stage_dt_diag.py [stage] [epochs] [images_per_step] [group]
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2409_06941_b200 import gpu  # noqa: E402


def per_op(ops, nops):
    """[(epoch, op) -> (start offset from the epoch's first op, duration)]"""
    out = []
    for e in range(len(ops) // nops):
        t0 = ops[e * nops][0]
        out.append([(a - t0, b - a) for a, b in ops[e * nops:(e + 1) * nops]])
    return out


def main():
    stage = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    ips = int(sys.argv[3]) if len(sys.argv) > 3 else 16
    G = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    torch.cuda.set_device(0)
    h = gpu.Harness(num_stages=4, num_micro_batches=4, stage=stage, layers=6, hidden=2048, tokens=8192,
                    ffn_mult=4, step_group=G)
    ok, _ = h.submit("image", gpu.ImageTask(batch=64, images_per_step=ips), profile_steps=32)
    assert ok
    h.run(3, True)
    h.reprofile("image")
    base = h.run(K, False)
    ops_b = h.timeline(0)
    bub_b = h.timeline(1)
    r = h.run(K, True)
    ops_w = h.timeline(0)
    bub_w = h.timeline(1)
    steps = h.timeline(2)
    nops = 8
    pb, pw = per_op(ops_b, nops), per_op(ops_w, nops)
    print(f"stage {stage}: makespan base {base['makespan_s']*1e3:.3f} ms, with {r['makespan_s']*1e3:.3f} ms, "
          f"dT {(r['makespan_s']-base['makespan_s'])/base['makespan_s']*100:+.3f} %  fill "
          f"{r['used_s']/r['bubble_s']:.3f} overrun {r['overrun_s']*1e3:.3f} ms")
    print("op  start_lateness_us(with-base, median over epochs)  dur_growth_us")
    for i in range(nops):
        late = statistics.median(pw[e][i][0] - pb[e][i][0] for e in range(1, K))
        grow = statistics.median(pw[e][i][1] - pb[e][i][1] for e in range(1, K))
        print(f"{i:2d}  {late*1e6:9.1f}  {grow*1e6:9.1f}")
    # epoch lengths
    eb = [ops_b[(e + 1) * nops][0] - ops_b[e * nops][0] for e in range(K - 1)]
    ew = [ops_w[(e + 1) * nops][0] - ops_w[e * nops][0] for e in range(K - 1)]
    print("epoch length base (ms):", [round(x * 1e3, 3) for x in eb])
    print("epoch length with (ms):", [round(x * 1e3, 3) for x in ew])
    # per-bubble: last step end past the bubble end (overrun) per bubble position
    nb = len(bub_w) // K
    over = [[] for _ in range(nb)]
    for j, (a, b) in enumerate(bub_w):
        ends = [s1 for s0, s1 in steps if s0 < b and s1 > a]
        if ends:
            over[j % nb].append(max(0.0, max(ends) - b))
    print("per bubble position: median overrun past bubble end (us):",
          [round(statistics.median(o) * 1e6, 1) if o else None for o in over])
    print("per bubble position: median duration base/with (us):",
          [(round(statistics.median(bub_b[j + e * nb][1] - bub_b[j + e * nb][0] for e in range(K)) * 1e6),
            round(statistics.median(bub_w[j + e * nb][1] - bub_w[j + e * nb][0] for e in range(K)) * 1e6))
           for j in range(nb)])
    h.close()


if __name__ == "__main__":
    main()
