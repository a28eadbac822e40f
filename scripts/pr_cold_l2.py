"""PageRank iteration time with a warm L2 vs after an L2 flush (a 256 MB
write between iterations, like the GEMM op between two bubbles)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2409_06941_b200 import gpu  # noqa: E402


def main():
    g = gpu.PageRankGraph(scale=20, edge_factor=16, seed=1)
    st = gpu.PageRankState(g)
    s = gpu.low_priority_stream()
    st.reset(stream=s)
    junk = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = {}
    for flush in (False, True):
        ts = []
        for i in range(30):
            if flush:
                with torch.cuda.stream(torch.cuda.Stream(stream_ptr=s.cuda_stream) if hasattr(s, "cuda_stream") else torch.cuda.current_stream()):
                    pass
                junk.fill_(i & 0xFF)
                torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            st.step(1, 0.85, stream=s)
            b.record(s)
            s.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        out["cold_us" if flush else "warm_us"] = statistics.median(ts[5:])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
