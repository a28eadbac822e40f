"""Small invocations of every side-task kernel for compute-sanitizer
(memcheck / racecheck / synccheck): K5 TMA + general + preemptible paths and
the host-I/O ring, PageRank build (RMAT and caller edges) + pull, SGD generate
+ per-edge / by-user (rounds, item blocks) steps + RMSE, the synthetic step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2409_06941_b200 import gpu  # noqa: E402

gpu.glib()
s = gpu.low_priority_stream()
# K5: exact-2x TMA path, general path, preemptible path
plan = gpu.ImagePlan(640, 360, 320, 180)
src = gpu.img_generate(3, 640, 360, seed=1)
wm = gpu.img_generate_watermark(320, 180, seed=2)
dst = torch.empty((3, 180, 320, 3), dtype=torch.uint8, device="cuda")
plan.run(src, dst, wm, stream=s)
prep = plan.prepare(wm, stream=s)
# overlapping consecutive launches (programmatic dependent launch, rotating counters)
plan.set_overlap(True)
for i in range(3):
    plan.run_prepared(src[i:i + 1], dst[i:i + 1], prep, stream=s)
plan.set_overlap(False)
ctr = torch.zeros(8, dtype=torch.int32, device="cuda")
plan.run_preemptible(src, dst, prep, ctr, max_rows=700, stream=s)
# round 2: every exact-2x variant (plan-creation knobs), frame units (a small
# SM budget so a 4-frame launch claims 4-frame units), the preemptible path
for env in ({}, {"FR_IMG_PIPES": "3"}, {"FR_IMG_CFG": "bar"}, {"FR_IMG_MATH": "0"}):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    pv = gpu.ImagePlan(640, 360, 320, 180)
    for k, v in old.items():
        if v is None:
            os.environ.pop(k)
        else:
            os.environ[k] = v
    pp = pv.prepare(wm, stream=s)
    src4 = gpu.img_generate(4, 640, 360, seed=9)
    dst4 = torch.empty((4, 180, 320, 3), dtype=torch.uint8, device="cuda")
    pv.run_prepared(src4, dst4, pp, stream=s)
    pv.set_max_sms(2)
    pv.run_prepared(src4, dst4, pp, stream=s)
    c4 = torch.zeros(8, dtype=torch.int32, device="cuda")
    pv.run_preemptible(src4, dst4, pp, c4, max_rows=500, stream=s)
    s.synchronize()
gen = gpu.ImagePlan(300, 200, 170, 90)
src2 = gpu.img_generate(2, 300, 200, seed=3)
wm2 = gpu.img_generate_watermark(170, 90, seed=4)
dst2 = torch.empty((2, 90, 170, 3), dtype=torch.uint8, device="cuda")
gen.run(src2, dst2, wm2, stream=s)
# PageRank: all-hot (scale 12) and partial hot prefix + split rows (scale 16)
for scale in (12, 16):
    g = gpu.PageRankGraph(scale=scale, edge_factor=16, seed=5)
    st = gpu.PageRankState(g)
    st.reset(stream=s)
    st.step(3, 0.85, stream=s)
    s.synchronize()
# PageRank on a caller-supplied edge list (self loops, duplicates, a hub row)
srcs = torch.cat([torch.arange(1, 3000), torch.tensor([5, 5, 7, 7])]).to(torch.int32)
dsts = torch.cat([torch.zeros(2999, dtype=torch.int64), torch.tensor([5, 6, 8, 8])]).to(torch.int32)
ge = gpu.PageRankGraph.from_edges(3001, srcs, dsts)
ste = gpu.PageRankState(ge)
ste.reset(stream=s)
ste.step(2, 0.85, stream=s)
s.synchronize()
# SGD: per-edge kernel (COO), by-user kernel on the rounds layout (k = 16) and
# on the item-blocked layout (k = 128: latent rows > 64 MiB -> 2 blocks)
p = gpu.SgdProblem(V=5000, E=40000, k=16, edge_seed=6, init_seed=7)
p.step(0, 40000, stream=s)
p.rmse()
pu = gpu.SgdProblem(V=5000, E=40000, k=16, edge_seed=6, init_seed=7, by_user=True, window=4096)
gpu.check(gpu.glib().fr_sgd_problem_set_overlap(pu._h, 1))   # overlapping consecutive steps
pu.step(0, 17, stream=s)
pu.step(17, 20000, stream=s)
pu.step(20000, 40000, stream=s)
pu.rmse()
pb = gpu.SgdProblem(V=140000, E=300000, k=128, edge_seed=6, init_seed=7, by_user=True, window=65536)
pb.step(0, 65536, stream=s)
pb.rmse()
s.synchronize()
# host-I/O image task (ring of device slots fed by the copy engines)
ht = gpu.ImageTask(sw=640, sh=360, dw=320, dh=180, batch=4, images_per_step=1, host_io=True, host_ring=3, seed=9)
assert ht.vt.create(ht.user) == 0 and ht.vt.init(ht.user, s.cuda_stream) == 0
for _ in range(6):
    assert ht.vt.run_next_step(ht.user, s.cuda_stream) == 0
assert ht.vt.stop(ht.user) == 0
s.synchronize()
# the runtime: gap / stamp kernels, a short harvest with the synthetic task
h = gpu.Harness(num_stages=2, num_micro_batches=2, stage=1, layers=1, hidden=512, tokens=1024,
                profile_reps=1, profile_epochs=1)
h.submit("syn", gpu.SyntheticTask(step_ns=50_000, memory_demand_gib=0.01), profile_steps=2)
h.run(2, True)
h.close()
torch.cuda.synchronize()
print("sanitize workload done")
