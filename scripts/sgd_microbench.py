"""Device-timed Graph-SGD step at the Orkut shape (CUDA events)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2409_06941_b200 import gpu  # noqa: E402


def main():
    chunk = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 21
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    by_user = len(sys.argv) > 3 and sys.argv[3] == "user"
    p = gpu.SgdProblem(by_user=by_user)
    s = gpu.low_priority_stream()
    torch.cuda.synchronize()
    n = p.E // chunk
    for i in range(3):
        p.step(i * chunk, (i + 1) * chunk, stream=s)
    s.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for i, (a, b) in enumerate(ev):
        j = (i + 3) % n
        a.record(s)
        p.step(j * chunk, (j + 1) * chunk, stream=s)
        b.record(s)
    s.synchronize()
    t = statistics.median(a.elapsed_time(b) * 1e-3 for a, b in ev)
    # algorithmic bytes per edge: 268 (COO); by user 12 + 128 per edge + 128 per run of equal u
    bpe = 268
    if by_user:   # L_u loads: one per run of equal u and every 16 edges within it
        u = p.edges()[0]
        start = torch.ones(u.numel(), dtype=torch.bool, device=u.device)
        start[1:] = u[1:] != u[:-1]
        idx = torch.arange(u.numel(), device=u.device)
        rs = torch.cummax(torch.where(start, idx, torch.zeros_like(idx)), 0).values
        bpe = 12 + 128 + 128 * (((idx - rs) % 16) == 0).double().mean().item()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    p.epoch(stream=s)
    e1.record(s)
    s.synchronize()
    te = e0.elapsed_time(e1) * 1e-3
    print(json.dumps({"by_user": by_user, "chunk": chunk, "step_us": t * 1e6, "edges_per_s": chunk / t,
                      "bytes_per_edge": bpe, "alg_GBps": chunk * bpe / t / 1e9, "epoch_ms": te * 1e3,
                      "epoch_alg_GBps": p.E * bpe / te / 1e9, "rmse_after": p.rmse()}))


if __name__ == "__main__":
    main()
