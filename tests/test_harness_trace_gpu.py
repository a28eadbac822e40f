"""The GPU dispatcher's parity object: the harness run as
a RunTrace (engine.hpp:75-92) that replay_check (engine.hpp:100-104) accepts,
every program-directed gate decision replayed through the REFERENCE's
iterative_run (task.cpp:89-100, oracle/_ref), and every bubble signal replayed
through the reference's Alg. 2 (manager.cpp:37-70) -- identical admit / yield
sequences and manager actions.  Plus the init guard (ArmInitGuard,
manager.hpp:58 -> KilledInitTimeout, engine.hpp:16 / task.hpp:102) and the
reclamation delay (limits.hpp:12) on the real runtime."""
import time

import pytest

pytestmark = pytest.mark.gpu

GRACE_NS = 5_000_000


@pytest.fixture(scope="module")
def g():
    from paper_2409_06941_b200 import gpu
    gpu.glib()
    return gpu


def small_harness(g, stage, **kw):
    return g.Harness(num_stages=4, num_micro_batches=4, stage=stage, layers=2, hidden=2048,
                     tokens=8192, profile_reps=3, profile_epochs=2, **kw)


def replay_signals(ref, prof, avail, sigs, bubbles, ws=None):
    """Alg. 2 through the reference, with the task views the harness saw"""
    from paper_2409_06941_b200.bubblesim import Bubble, BubbleType, SideTaskState, TaskView
    if ws is None:
        ws = ref.workers([avail])
        assert ref.submit_task(prof, ws).assigned
    for k, s in enumerate(sigs):
        view = TaskView(SideTaskState(s["view_state"]), bool(s["view_initializing"]))
        seen = []

        def lookup(tid, view=view, want=s["task"], seen=seen):
            seen.append(tid)
            assert tid == want, (k, tid, want)
            return view
        if s["kind"] == 0:
            pb = bubbles[s["bubble"]]
            b = Bubble(0, s["epoch"], s["t"], s["duration"], avail, BubbleType(pb["btype"]))
            acts = ref.on_bubble_started(ws, 0, b, lookup)
        else:
            acts = ref.on_bubble_ended(ws, 0, s["t"], lookup)
        assert [int(a.kind) for a in acts] == s["actions"], (k, s, acts)
        assert all(a.task_id == s["task"] for a in acts)
        assert bool(seen) == bool(s["looked_up"]), (k, s)
    return ws


@pytest.mark.parametrize("stage", [0, 1, 2, 3])
def test_gpu_dispatch_replays_through_reference(g, ref, stage):
    from paper_2409_06941_b200.bubblesim import SideTaskRuntime, SideTaskSpec, SideTaskState, TaskProfile
    h = small_harness(g, stage, step_group=3)
    ok, p = h.submit("image", g.ImageTask(batch=16, images_per_step=2), profile_steps=8)
    assert ok
    avail = h.profile()["available_memory"]
    prof = TaskProfile("image", p["est_per_step_duration"], p["max_per_step_duration"], p["est_memory"],
                       p["profiled_steps"])
    bubbles = h.stage_bubbles()
    ws = None
    admitted = yielded = 0
    for run in range(3):
        r = h.run(2, True)
        sigs = h.signal_log()
        assert sum(s["kind"] == 1 for s in sigs) == 2 * len(bubbles)   # every bubble ended, 2 epochs
        ws = replay_signals(ref, prof, avail, sigs, bubbles, ws)
        # every gate decision, through the reference's iterative_run
        running = SideTaskRuntime(SideTaskSpec("image"), SideTaskState.Running)
        for d in h.gate_log():
            want = ref.iterative_run(running, d["bubble_end"], d["now"], d["est_seconds"], 1e-9, d["step_ticks"])
            assert want.run == bool(d["run"]), d
            if want.run:
                assert want.step_end == d["step_end"], d
            s = sigs[d["signal"]]
            assert s["kind"] == 0 and 1 in s["actions"]          # started by an IssueStart
            assert d["bubble_end"] == s["t"] + s["duration"]     # StartSideTask's bubble end
            admitted += want.run
            yielded += not want.run
        # the measured RunTrace passes the reference's replay_check
        tr = h.run_trace()
        assert tr["violations"] == [], tr["violations"][:5]
        steps = [a for a in tr["activities"] if a[4] == 1]
        assert len(steps) == r["steps_completed"]
        assert len(tr["ops"]) == 2 * 8 and len(tr["bubbles"]) == 2 * len(bubbles)
    assert admitted > 10 and yielded > 0
    h.close()


def test_tampered_trace_is_caught(g, product, tmp_path):
    """replay_check on a GPU trace is not vacuous: a step moved before its
    StartSideTask and an op moved into its predecessor are reported"""
    import json
    h = small_harness(g, 2)
    ok, _ = h.submit("image", g.ImageTask(batch=16, images_per_step=2), profile_steps=8)
    assert ok
    h.run(2, True)
    path = tmp_path / "gpu_trace.jsonl"
    tr = h.run_trace(trace_path=str(path))
    assert tr["violations"] == []
    assert product.replay_check_file(str(path)) == []
    lines = [json.loads(x) for x in path.read_text().splitlines()]
    assert lines[0]["measured"] is True
    first_start = min(x["t"] for x in lines if x.get("type") == "transition" and x["kind"] == "start")
    for x in lines:
        if x.get("type") == "activity" and x["kind"] == "step":
            x["start"], x["end"] = first_start - 1_000_000, first_start - 900_000
            break
    ops = [x for x in lines if x.get("type") == "op"]
    ops[3]["start"] = ops[2]["start"]
    bad = tmp_path / "bad.jsonl"
    bad.write_text("\n".join(json.dumps(x) for x in lines) + "\n")
    v = product.replay_check_file(str(bad))
    assert any("activity" in x for x in v) and any("stage predecessor" in x for x in v), v
    h.close()


def test_init_guard_kills_init_timeout(g, ref):
    """an InitSideTask that outlasts its bubble: ArmInitGuard at the bubble
    end, KilledInitTimeout one grace period later; the pool pages go back
    only after the reclamation delay"""
    h = small_harness(g, 1, grace_ns=GRACE_NS, reclamation_delay_ns=400_000_000)
    task = g.SyntheticTask(step_ns=100_000, memory_demand_gib=0.25, init_ns=2_000_000_000)
    ok, _ = h.submit("slow-init", task, profile_steps=2)
    assert ok
    r = h.run(1, True)
    assert r["kills"] == 1 and r["kills_init_timeout"] == 1, r
    assert h.task_status("slow-init")["disposition"] == "killed_init_timeout"
    sigs = h.signal_log()
    arm = [s for s in sigs if s["kind"] == 1 and 3 in s["actions"]]
    assert len(arm) == 1 and arm[0]["view_initializing"] == 1
    tr = h.run_trace()
    assert tr["violations"] == [], tr["violations"]
    (kill,) = tr["kills"]
    assert kill[3] == 2                                   # KillReason::InitTimeout
    late = kill[0] - arm[0]["t"]
    assert GRACE_NS <= late < GRACE_NS + 1_000_000, late  # exactly one grace period after the bubble end
    assert ("slow-init", 4, 0, 1) in [(d[0], d[1], d[2], d[3]) for d in tr["dispositions"]]
    # the run ended well inside the 0.4 s reclamation delay: pages still held
    assert h.task_memory("slow-init")["reserved_gib"] >= 0.25
    time.sleep(0.5)
    h.run(1, False)
    assert h.task_memory("slow-init")["reserved_gib"] == 0.0
    h.close()


def test_init_inside_bubble_is_not_killed(g):
    """the guard is disarmed when the init lands before bubble end + grace"""
    h = small_harness(g, 1, grace_ns=GRACE_NS)
    task = g.SyntheticTask(step_ns=100_000, memory_demand_gib=0.1, init_ns=200_000)
    ok, _ = h.submit("quick-init", task, profile_steps=2)
    assert ok
    r = h.run(2, True)
    assert r["kills"] == 0 and r["steps_completed"] > 0
    assert h.task_status("quick-init")["disposition"] == "active"
    assert h.run_trace()["violations"] == []
    h.close()
