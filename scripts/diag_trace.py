"""The GPU RunTrace of a short harvest (stage 2, image task, step groups 1 and
3) with its gate / signal logs written to gpurun_out/, for checking
replay_check verdicts by hand (the pause-stamp flake of round 2).
Usage: python scripts/diag_trace.py"""
import json, sys
sys.path.insert(0, '.')
from paper_2409_06941_b200 import gpu
import torch
torch.cuda.set_device(0)
gpu.glib()
for sg in (1, 3):
    h = gpu.Harness(num_stages=4, num_micro_batches=4, stage=2, layers=2, hidden=2048, tokens=8192,
                    profile_reps=3, profile_epochs=2, step_group=sg)
    ok, _ = h.submit("image", gpu.ImageTask(batch=16, images_per_step=2), profile_steps=8)
    h.run(2, True)
    tr = h.run_trace(trace_path=f"gpurun_out/diag_trace_sg{sg}.jsonl")
    print("sg", sg, "violations", tr["violations"][:5])
    json.dump({"gate": h.gate_log(), "sig": h.signal_log()}, open(f"gpurun_out/diag_logs_sg{sg}.json", "w"), default=str)
    h.close()
