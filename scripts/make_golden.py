"""Generates tests/golden/* -- fixtures that pin the oracle (oracle/) to
independent implementations available in this container:

  image_cv2.npz     cv2.resize(INTER_LINEAR_EXACT) on random frames + the
                    integer watermark blend (numpy), several shapes
  pagerank_scipy.npz  scipy.sparse power iteration (dangling mass dropped)
  sgd_numpy.npz     float32 numpy restatement of the sequential SGD epoch
  host_reference.json  outputs of the reference's own compiled sources
                    (oracle/_ref) for SURVEY.md Appendix A configurations

Run from the repo root: python scripts/make_golden.py
"""
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)


def image_fixture(rng):
    import cv2
    cases = {}
    for i, (sh, sw, dh, dw) in enumerate([(64, 96, 32, 48), (37, 53, 20, 29), (16, 16, 31, 33),
                                          (120, 200, 60, 100), (9, 250, 4, 125)]):
        src = rng.integers(0, 256, (sh, sw, 3), dtype=np.uint8)
        wm = rng.integers(0, 256, (dh, dw, 4), dtype=np.uint8)
        rs = cv2.resize(src, (dw, dh), interpolation=cv2.INTER_LINEAR_EXACT).astype(np.int64)
        a = wm[..., 3:4].astype(np.int64)
        out = ((rs * (255 - a) + wm[..., :3].astype(np.int64) * a + 127) // 255).astype(np.uint8)
        cases[f"src{i}"], cases[f"wm{i}"], cases[f"out{i}"] = src, wm, out
    np.savez_compressed(os.path.join(OUT, "image_cv2.npz"), **cases)


def pagerank_fixture(rng):
    import scipy.sparse as sp
    V, m = 1024, 12000
    src = rng.integers(0, V, m).astype(np.int32) ** 2 % V   # skewed
    dst = rng.integers(0, V, m).astype(np.int32)
    keep = src != dst
    pairs = np.unique(np.stack([dst[keep], src[keep]], 1), axis=0)
    d, s = pairs[:, 0], pairs[:, 1]
    A = sp.csr_matrix((np.ones(len(d)), (d, s)), shape=(V, V))   # A[v, u] = 1 for u -> v
    outdeg = np.bincount(s, minlength=V).astype(np.float64)
    inv = np.where(outdeg > 0, 1.0 / np.maximum(outdeg, 1), 0.0)
    r = np.full(V, 1.0 / V)
    d_ = 0.85
    for _ in range(20):
        r = (1 - d_) / V + d_ * (A @ (r * inv))
    np.savez_compressed(os.path.join(OUT, "pagerank_scipy.npz"), src=s.astype(np.int32),
                        dst=d.astype(np.int32), V=V, iters=20, damping=d_, ranks=r)


def sgd_fixture(rng):
    V, E, k = 300, 2000, 16
    u = rng.integers(0, V, E).astype(np.int32)
    v = rng.integers(0, V, E).astype(np.int32)
    r = rng.integers(1, 6, E).astype(np.float32)
    L0 = (rng.random((V, k)) * 0.25).astype(np.float32)
    L = L0.copy()
    eta, lam = np.float32(0.01), np.float32(0.05)
    for _ in range(2):
        for e in range(E):
            lu, lv = L[u[e]], L[v[e]]
            dot = np.float32(0.0)
            for j in range(k):
                dot = np.float32(dot + np.float32(lu[j] * lv[j]))
            err = np.float32(r[e] - dot)
            for j in range(k):
                a, b = lu[j], lv[j]
                lu[j] = np.float32(a + np.float32(eta * np.float32(np.float32(err * b) - np.float32(lam * a))))
                lv[j] = np.float32(b + np.float32(eta * np.float32(np.float32(err * a) - np.float32(lam * b))))
    pred = np.einsum("ij,ij->i", L[u].astype(np.float64), L[v].astype(np.float64))
    rmse = float(np.sqrt(np.mean((r.astype(np.float64) - pred) ** 2)))
    np.savez_compressed(os.path.join(OUT, "sgd_numpy.npz"), u=u, v=v, r=r, L0=L0, L2=L, eta=eta,
                        lam=lam, rmse=rmse)


def host_fixture():
    from paper_2409_06941_b200.bubblesim import BubbleSim, PipelineConfig, ProfileOptions, SideTaskSpec
    ref = BubbleSim(ctypes.CDLL(os.path.join(ROOT, "oracle", "_ref", "libbubblesim_ref.so")))
    out = {}
    for name, (p, m, fp, bp, epochs, w, a) in {
        "A1_p4m4_fp1bp2": (4, 4, 1, 2, 1, 4.0, 4.0),
        "A1_p4m4_fp1bp2_2ep": (4, 4, 1, 2, 2, 4.0, 4.0),
        "A2_C1": (4, 4, 220, 347, 1, 20.0, 6.5),
        "A2_p8m8": (8, 8, 220, 347, 1, 4.0, 4.0),
        "p4m8_fp1bp1": (4, 8, 1, 1, 1, 4.0, 4.0),
        "p1m3": (1, 3, 1, 2, 1, 4.0, 4.0),
    }.items():
        cfg = PipelineConfig(p, m, [fp], [bp], epochs, 48.0, ref.default_stage_memory(p, 48.0, w, a))
        tr = ref.build_schedule(cfg)
        lb = ref.extract_bubbles_linked(tr)
        out[name] = {
            "config": [p, m, fp, bp, epochs, w, a],
            "ops": [[o.stage, int(o.kind), o.micro_batch, o.epoch, o.start, o.end] for o in tr.ops],
            "spans": tr.epoch_spans,
            "bubbles": [[b.bubble.stage, b.bubble.epoch, b.bubble.start, b.bubble.duration,
                         b.bubble.available_memory, int(b.bubble.btype),
                         -1 if b.prev_op is None else b.prev_op, -1 if b.next_op is None else b.next_op]
                        for b in lb],
            "rate": ref.bubble_rate(tr, [b.bubble for b in lb]),
            "profile": [[s.durations, s.available_memory] for s in ref.profile_bubbles(cfg).stages],
        }
    out["stream_seed_0_t_profile"] = ref.stream_seed(0, "t", "profile")
    p = ref.profile_task(SideTaskSpec("t", per_step_duration=304, memory_demand=2.63), ProfileOptions(32, 0.1, 1e-4), 42)
    out["profile_task_jitter"] = [p.est_per_step_duration, p.max_per_step_duration, p.est_memory]
    with open(os.path.join(OUT, "host_reference.json"), "w") as f:
        json.dump(out, f)


def main():
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(20240911)
    image_fixture(rng)
    pagerank_fixture(rng)
    sgd_fixture(rng)
    host_fixture()
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
