"""SGD task in bubbles: RMSE after profiling and after each harness run (NaN hunt)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2409_06941_b200 import gpu  # noqa: E402


def main():
    by_user = sys.argv[1] == "user" if len(sys.argv) > 1 else True
    h = gpu.Harness(num_stages=4, num_micro_batches=4, stage=3, layers=2, profile_reps=2, profile_epochs=1)
    eps = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 19
    task = gpu.SgdTask(V=300000, E=6000000, k=16, edges_per_step=eps, by_user=by_user)
    prob, _ = task.problem()
    print("created", prob.rmse(), flush=True)
    ok, prof = h.submit("sgd", task, profile_steps=8)
    prob, ep = task.problem()
    L = prob.latent()
    print("after submit", ok, prof["est_per_step_duration"], prob.rmse(), "nan", int(torch.isnan(L).sum()), flush=True)
    for i in range(3):
        r = h.run(2, True)
        prob, ep = task.problem()
        L = prob.latent()
        print("run", i, r["steps_completed"], "epochs", ep, prob.rmse(), "nan", int(torch.isnan(L).sum()),
              "absmax", float(L.abs().max()), flush=True)
    h.close()


if __name__ == "__main__":
    main()
