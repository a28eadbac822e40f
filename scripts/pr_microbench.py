"""Device-timed PageRank pull iteration at RMAT scale 20 (CUDA events)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2409_06941_b200 import gpu  # noqa: E402


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    g = gpu.PageRankGraph(scale=scale, edge_factor=16, seed=1)
    st = gpu.PageRankState(g)
    s = gpu.low_priority_stream()
    st.reset(stream=s)
    for _ in range(5):
        st.step(1, 0.85, stream=s)
    s.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(s)
        st.step(1, 0.85, stream=s)
        b.record(s)
    s.synchronize()
    t = statistics.median(a.elapsed_time(b) * 1e-3 for a, b in ev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    st.step(reps, 0.85, stream=s)      # back-to-back iterations, no events between
    b.record(s)
    s.synchronize()
    t_chain = a.elapsed_time(b) * 1e-3 / reps
    alg = 4 * (g.V + 1) + 4 * g.E + 16 * g.V
    print(json.dumps({"scale": scale, "V": g.V, "E": g.E, "blocks": g.n_blocks, "iter_us": t * 1e6, "chain_iter_us": t_chain * 1e6,
                      "edges_per_s": g.E / t, "alg_GBps": alg / t / 1e9,
                      "gather_GBps_l2_sectors": g.E * 32 / t / 1e9}))


if __name__ == "__main__":
    main()
