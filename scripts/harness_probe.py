"""Probe the bubble-harvesting runtime on one GPU: every stage of a 4-stage
1F1B pipeline replayed in turn, image side task harvesting its bubbles."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_06941_b200 import gpu  # noqa: E402


def main():
    epochs = int(os.environ.get("EPOCHS", "8"))
    ips = int(os.environ.get("IPS", "8"))
    host_io = os.environ.get("HOST_IO", "0") == "1"
    stages = [int(s) for s in os.environ.get("STAGES", "0,1,2,3").split(",")]
    for s in stages:
        t0 = time.time()
        h = gpu.Harness(num_stages=4, num_micro_batches=4, stage=s)
        prof = h.profile()
        task = gpu.ImageTask(images_per_step=ips, host_io=host_io)
        ok, tp = h.submit("image", task)
        warm = h.run(2, True)
        base = h.run(epochs, False)
        withr = h.run(epochs, True)
        base2 = h.run(epochs, False)
        dt = (withr["makespan_s"] - base["makespan_s"]) / base["makespan_s"]
        dt2 = (base2["makespan_s"] - base["makespan_s"]) / base["makespan_s"]
        print(json.dumps({
            "stage": s, "setup_s": round(time.time() - t0, 2), "assigned": ok,
            "fp_ms": prof["fp_ticks"] / 1e6, "bp_ms": prof["bp_ticks"] / 1e6,
            "span_ms": prof["epoch_span"] / 1e6, "fp_tflops": round(prof["fp_tflops"], 1),
            "bp_tflops": round(prof["bp_tflops"], 1), "stage_bubble_ms": prof["stage_bubble_ticks"] / 1e6,
            "clock_err_ns": prof["clock_offset_err_ns"],
            "est_step_us": tp["est_per_step_duration"] * 1e6, "max_step_us": tp["max_per_step_duration"] * 1e6,
            "makespan_no": base["makespan_s"], "makespan_with": withr["makespan_s"],
            "makespan_no2": base2["makespan_s"], "dT": dt, "noise_dT": dt2,
            "bubble_s": withr["bubble_s"], "used_s": withr["used_s"], "fill": withr["used_s"] / withr["bubble_s"] if withr["bubble_s"] else 0,
            "overrun_s": withr["overrun_s"], "max_overrun_us": withr["max_step_overrun_s"] * 1e6,
            "steps": withr["steps_completed"], "px": withr["work_units"],
            "px_per_bubble_s": withr["work_units"] / base["bubble_s"] if base["bubble_s"] else 0,
            "dispatch_us": withr["dispatch_host_us"], "pauses": withr["pauses"], "kills": withr["kills"],
            "breakdown": withr["breakdown"], "warm_steps": warm["steps_completed"],
        }), flush=True)
        h.close()


if __name__ == "__main__":
    main()
