"""Repeat the Fig. 9 OOM scenario of tests/test_limits_gpu.py and print every
run's report (hunting a flake where no OOM kill happened in 12 runs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_06941_b200 import gpu  # noqa: E402


def main():
    for trial in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
        h = gpu.Harness(num_stages=4, num_micro_batches=4, stage=1, layers=2, profile_reps=2,
                        profile_epochs=1, memory_headroom_gib=0.1, grace_ns=10_000_000_000)
        task = gpu.SyntheticTask(step_ns=200_000, memory_demand_gib=0.25, leak_gib_per_step=0.05)
        ok, prof = h.submit("leaky", task, profile_steps=4)
        launched = kills = 0
        log = []
        for _ in range(12):
            r = h.run(2, True)
            launched += r["steps_launched"]
            kills += r["kills_oom"]
            log.append((r["steps_launched"], r["steps_completed"], r["kills_oom"], r["kills_pause_timeout"],
                        round(r["used_s"] * 1e3, 2), round(r["bubble_s"] * 1e3, 2), h.task_status("leaky")["state"]))
            if kills:
                break
        print(trial, "kills", kills, "launched", launched, log[:4], "...", log[-1], flush=True)
        h.close()


if __name__ == "__main__":
    main()
