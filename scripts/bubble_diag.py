"""Per-bubble diagnostics of one harness run: where does idle bubble time go?"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_06941_b200 import gpu  # noqa: E402


def main():
    s = int(os.environ.get("STAGE", "1"))
    ips = int(os.environ.get("IPS", "8"))
    h = gpu.Harness(num_stages=4, num_micro_batches=4, stage=s)
    prof = h.profile()
    pb = h.stage_bubbles()
    _, p0 = h.submit("image", gpu.ImageTask(images_per_step=ips))
    h.run(2, True)
    p1 = h.reprofile("image")
    print(json.dumps({"standalone_est_us": p0["est_per_step_duration"] * 1e6,
                      "in_pipeline_est_us": p1["est_per_step_duration"] * 1e6,
                      "in_pipeline_max_us": p1["max_per_step_duration"] * 1e6}))
    base = h.run(4, False)
    ops_no = h.timeline(0)
    bub_no = h.timeline(1)
    r = h.run(4, True)
    ops = h.timeline(0)
    bub = h.timeline(1)
    steps = h.timeline(2)
    print(json.dumps({"profile": prof, "profile_bubbles_ms": [b["duration"] / 1e6 for b in pb]}))
    nb = len(pb)
    for i, (a, b) in enumerate(bub):
        inside = [(x, y) for x, y in steps if y > a and x < b]
        used = sum(min(y, b) - max(x, a) for x, y in inside)
        first = (inside[0][0] - a) * 1e6 if inside else None
        last_gap = (b - max(y for _, y in inside)) * 1e6 if inside else None
        over = max((y - b) * 1e6 for _, y in inside) if inside else 0
        durs = [(y - x) * 1e6 for x, y in inside]
        print(json.dumps({
            "i": i, "type_idx": i % nb, "dur_ms": round((b - a) * 1e3, 4),
            "prof_ms": pb[i % nb]["duration"] / 1e6,
            "base_dur_ms": round((bub_no[i][1] - bub_no[i][0]) * 1e3, 4) if i < len(bub_no) else None,
            "fill": round(used / (b - a), 4) if b > a else 0, "n_steps": len(inside),
            "first_step_us": None if first is None else round(first, 1),
            "tail_idle_us": None if last_gap is None else round(last_gap, 1),
            "overrun_us": round(over, 1),
            "step_us_mean": round(sum(durs) / len(durs), 1) if durs else None,
            "step_us_max": round(max(durs), 1) if durs else None,
        }))
    # op duration inflation (interference)
    d_no = [b - a for a, b in ops_no]
    d_w = [b - a for a, b in ops]
    st_no = [a for a, _ in ops_no]
    st_w = [a for a, _ in ops]
    print(json.dumps({
        "op_dur_mean_no_ms": sum(d_no) / len(d_no) * 1e3, "op_dur_mean_with_ms": sum(d_w) / len(d_w) * 1e3,
        "op_start_shift_mean_us": sum(w - n for w, n in zip(st_w, st_no)) / len(st_w) * 1e6,
        "op_start_shift_max_us": max(w - n for w, n in zip(st_w, st_no)) * 1e6,
        "makespan_no": base["makespan_s"], "makespan_with": r["makespan_s"],
        "fill": r["used_s"] / r["bubble_s"], "overrun_s": r["overrun_s"],
    }))


if __name__ == "__main__":
    main()
