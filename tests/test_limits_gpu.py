"""Framework-enforced limits on the GPU (reference
limits.cpp:13-26 check_memory / framework_enforce; Fig. 9 scenarios,
SPEC.md:573): every task allocates from its own CUDA memory pool whose usage
is checked against est_memory + headroom, and a pause that is not observed
within the grace period kills the task (cooperative kernels are cancelled on
the device)."""
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    from paper_2409_06941_b200 import gpu
    gpu.glib()
    return gpu


def harness(g, **kw):
    return g.Harness(num_stages=4, num_micro_batches=4, stage=1, layers=2, profile_reps=2,
                     profile_epochs=1, **kw)


def test_profiled_memory_is_the_pool_high_water_mark(g):
    h = harness(g)
    task = g.SyntheticTask(step_ns=100_000, memory_demand_gib=0.5, leak_gib_per_step=0.0)
    ok, prof = h.submit("syn", task, profile_steps=4)
    assert ok and abs(prof["est_memory"] - 0.5) < 1e-3
    h.run(2, True)
    st = h.task_status("syn")
    assert st["disposition"] == "active" and abs(st["memory_used_gib"] - 0.5) < 1e-3
    h.close()


def test_memory_leak_is_oom_killed(g):
    """Fig. 9 OOM scenario: 0.25 GiB demand + 0.05 GiB leaked per step;
    profiled over 6 standalone steps (est 0.55 GiB) + 0.1 GiB headroom."""
    # a generous grace: a step that grows the pool may hold the worker in
    # cudaMallocAsync for a while; this scenario is about the memory limit only
    h = harness(g, memory_headroom_gib=0.1, grace_ns=10_000_000_000)
    task = g.SyntheticTask(step_ns=200_000, memory_demand_gib=0.25, leak_gib_per_step=0.05)
    ok, prof = h.submit("leaky", task, profile_steps=4)
    assert ok and abs(prof["est_memory"] - 0.55) < 1e-3
    launched = kills_oom = 0
    for _ in range(12):                          # until the leak crosses the limit
        r = h.run(2, True)
        launched += r["steps_launched"]
        kills_oom += r["kills_oom"]
        assert r["kills_pause_timeout"] == 0
        if kills_oom:
            break
    assert kills_oom == 1
    st = h.task_status("leaky")
    assert st["state"] == "stopped" and st["disposition"] == "killed_oom"
    assert st["memory_used_gib"] < 1e-6          # every allocation released
    # init 0.25 + 8 leaked steps = 0.65 GiB (not killed: strict >), the 9th kills
    assert launched == 9
    again = h.run(2, True)                       # the worker is free again
    assert again["steps_launched"] == 0 and again["kills"] == 0
    h.close()


@pytest.mark.parametrize("cooperative", [True, False])
def test_pause_timeout_kill(g, cooperative):
    """Fig. 9 timeout scenario: profiled at 0.1 ms per step, the task's real
    steps run 0.4 s -- far past the bubble end; the pause is not observed
    within the 0.1 s grace -> killed.  A cooperative step kernel is cancelled
    on the device (its step ends ~grace after the bubble end); a
    non-cooperative one can only be waited for."""
    h = harness(g, grace_ns=100_000_000)
    task = g.SyntheticTask(step_ns=400_000_000, profile_step_ns=100_000, memory_demand_gib=0.1,
                           cooperative=cooperative)
    ok, _ = h.submit("overrun", task, profile_steps=4)
    assert ok
    kills, longest = 0, 0.0
    for _ in range(4):           # the overrunning step needs a bubble after InitSideTask's
        r = h.run(2, True)
        assert r["kills_oom"] == 0
        kills += r["kills_pause_timeout"]
        if r["kills_pause_timeout"]:
            longest = max(b - a for a, b in h.timeline(2))
            break
    assert kills == 1
    st = h.task_status("overrun")
    assert st["state"] == "stopped" and st["disposition"] == "killed_pause_timeout"
    assert st["memory_used_gib"] < 1e-6
    if cooperative:
        assert longest < 0.3                     # cancelled, not run to 0.4 s
    else:
        assert longest >= 0.39
    h.close()
