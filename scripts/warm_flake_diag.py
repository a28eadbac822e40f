"""Repeat the harness warm-up (submit + 2 epochs with the image task) and print
the run report whenever no step completed -- hunting the 'no step in the
warm-up' flake."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_06941_b200 import gpu  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
    bad = 0
    for i in range(n):
        h = gpu.Harness(num_stages=4, num_micro_batches=4, stage=1, layers=2, hidden=2048, tokens=8192,
                        profile_reps=3, profile_epochs=2)
        ok, prof = h.submit("image", gpu.ImageTask(batch=16, images_per_step=2), profile_steps=16)
        warm = h.run(2, True)
        st = h.task_status("image") if hasattr(h, "task_status") else None
        if warm["steps_completed"] == 0:
            bad += 1
            print("NO STEP", i, {k: v for k, v in warm.items() if k != "breakdown"}, warm["breakdown"], st,
                  "prof", prof, "bubbles", sorted(d for _, d in [(0, b) for b in h.stage_bubbles()])[:3] if False else None,
                  flush=True)
        else:
            print("ok", i, warm["steps_completed"], st, flush=True)
        h.close()
    print("bad", bad, "of", n)


if __name__ == "__main__":
    main()
