"""a13: the simulated dispatch engine (run_experiment, engine.hpp:97-98).

The product engine (csrc/host/engine.cpp, event agenda) against the
tick-stepped oracle (oracle/engine_oracle.py) whose decision functions are
the reference's own compiled sources (oracle/_ref): the whole RunTrace --
op timings, signalled bubbles, submissions, RPCs, transitions, activities
(the step-dispatch order), kills, dispositions, makespan -- must be
identical.  Plus SPEC.md acceptance scenarios 5, 6, 7 and 9.
"""
import os
import random
import sys

import pytest

from paper_2409_06941_b200.bubblesim import (ActivityRecord, ActivityKind, AssignRecord, Bubble,
                                             BubbleType, LimitConfig, MisbehaviorKind, PipelineConfig,
                                             SideTaskSpec, TaskInterface, TaskProfile, TransitionKind,
                                             TransitionRecord)

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import engine_oracle as eo  # noqa: E402


def canon(tr):
    out = {k: sorted(v, key=repr) if isinstance(v, list) else v for k, v in tr.items()}
    out["ops"] = tr["ops"]  # already in the reference's (start, stage, end, mb) order
    return out


def rand_case(rng):
    p = rng.randint(1, 4)
    m = rng.randint(1, 4)
    per = rng.random() < 0.4
    fp = [rng.randint(1, 12) for _ in range(p)] if per else [rng.randint(1, 12)]
    bp = [rng.randint(1, 20) for _ in range(p)] if per else [rng.randint(1, 20)]
    mem = [round(rng.uniform(0, 30), 2) for _ in range(p)]
    cfg = PipelineConfig(p, m, fp, bp, rng.randint(1, 3), 48.0, mem, rng.choice([1e-3, 1e-2]))
    tasks = []
    for i in range(rng.randint(0, 4)):
        sp = SideTaskSpec(f"t{i}")
        sp.interface_kind = rng.choice([TaskInterface.Iterative] * 3 + [TaskInterface.Imperative])
        sp.per_step_duration = rng.randint(1, 8)
        sp.init_duration = rng.choice([0, 0, 1, 3, 7])
        sp.memory_demand = round(rng.uniform(0, 40), 2)
        sp.submit_time = rng.choice([0, 0, rng.randint(0, 60)])
        if rng.random() < 0.3:
            sp.total_steps = rng.randint(1, 15)
        r = rng.random()
        if r < 0.1:
            sp.misbehavior = MisbehaviorKind.IgnoresPause
        elif r < 0.2:
            sp.misbehavior = MisbehaviorKind.MemoryLeak
            sp.leak_rate_gib_per_s = rng.uniform(0.5, 50)
        if rng.random() < 0.2:
            sp.memory_limit = round(rng.uniform(0, 40), 2)
        tasks.append(sp)
    kw = dict(check_overhead=rng.choice([0, 1, 1, 2]), rpc_latency=rng.choice([0, 0, 1, 3]),
              step_jitter=rng.choice([0.0, 0.0, 0.2]), profile_steps=rng.choice([1, 4, 32]),
              gate_max=rng.random() < 0.2)
    limits = LimitConfig(grace_period=rng.choice([5, 10, 30, 100]),
                         memory_headroom=rng.choice([0.0, 0.5]))
    return cfg, tasks, kw, limits


def oracle_run(ref, cfg, tasks, kw, limits, seed, with_tasks=True):
    opts = eo.Opts(check_overhead=kw["check_overhead"], rpc_latency=kw["rpc_latency"],
                   step_jitter=kw["step_jitter"], profile_steps=kw["profile_steps"],
                   gate_max=kw["gate_max"], grace=limits.grace_period, headroom=limits.memory_headroom)
    return eo.run(ref, cfg, tasks, opts, seed, with_tasks)


def test_engine_matches_oracle_random(product, ref):
    rng = random.Random(97)
    n_tasks_seen = n_kills = n_steps = 0
    for case in range(250):
        cfg, tasks, kw, limits = rand_case(rng)
        seed = rng.getrandbits(64)
        want = oracle_run(ref, cfg, tasks, kw, limits, seed)
        got = product.run_experiment(cfg, tasks, seed, True, limits=limits, **kw)
        a, b = canon(got), canon(want)
        for k in b:
            assert a[k] == b[k], (case, k)
        n_tasks_seen += len(tasks)
        n_kills += len(got["kills"])
        n_steps += sum(1 for x in got["activities"] if x[4] == int(ActivityKind.Step))
    assert n_tasks_seen > 200 and n_kills > 5 and n_steps > 500   # the cases exercise the rules


def test_no_tasks_equals_build_schedule(product):
    cfg = PipelineConfig(4, 4, [220], [347], 3, 48.0, [20.0, 16.0, 12.0, 8.0])
    tr = product.build_schedule(cfg)
    got = product.run_experiment(cfg, [], 1, with_tasks=False)
    assert got["ops"] == [(o.stage, int(o.kind), o.micro_batch, o.epoch, o.start, o.end) for o in tr.ops]
    assert got["makespan"] == tr.epoch_spans[-1][1]
    # the signalled bubbles of an undelayed run are exactly extract_bubbles'
    want = sorted((b.stage, b.epoch, b.start, b.duration) for b in product.extract_bubbles(tr))
    assert sorted(x[:4] for x in got["bubbles"]) == want


def fig_cfg(epochs=4):
    return PipelineConfig(4, 4, [100], [200], epochs, 48.0, [20.0, 16.0, 12.0, 8.0])


def test_iterative_noise_free_zero_overhead_dT_is_zero(product):
    cfg = fig_cfg()
    tasks = [SideTaskSpec("pr", per_step_duration=7, memory_demand=4.0),
             SideTaskSpec("img", per_step_duration=13, memory_demand=4.0)]
    base = product.run_experiment(cfg, tasks, 5, with_tasks=False)
    run = product.run_experiment(cfg, tasks, 5, check_overhead=0)
    assert run["makespan"] == base["makespan"]                      # SPEC acceptance 5
    steps = [a for a in run["activities"] if a[4] == int(ActivityKind.Step)]
    assert len(steps) > 50
    bub = {}
    for s, e, st, d, *_ in run["bubbles"]:
        bub.setdefault(s, []).append((st, st + d))
    for a in steps:  # every step wholly inside a signalled bubble of its stage
        assert any(lo <= a[0] and a[1] <= hi for lo, hi in bub[a[3]]), a


def test_imperative_dT_positive_and_bounded(product):
    cfg = fig_cfg()
    it = [SideTaskSpec("a", per_step_duration=9, memory_demand=4.0)]
    im = [SideTaskSpec("a", TaskInterface.Imperative, per_step_duration=9, memory_demand=4.0)]
    base = product.run_experiment(cfg, it, 3, with_tasks=False)["makespan"]
    r_it = product.run_experiment(cfg, it, 3, check_overhead=0)
    r_im = product.run_experiment(cfg, im, 3, check_overhead=0)
    pauses = sum(1 for t in r_im["transitions"] if t[2] == int(TransitionKind.PauseSideTask))
    assert r_it["makespan"] == base
    assert 0 < r_im["makespan"] - base <= pauses * 9                 # SPEC acceptance 5
    assert r_it["makespan"] < r_im["makespan"]


def test_fig9_timeout_kill(product):
    cfg = fig_cfg()
    t = SideTaskSpec("rogue", TaskInterface.Imperative, per_step_duration=5, memory_demand=4.0,
                     misbehavior=MisbehaviorKind.IgnoresPause)
    run = product.run_experiment(cfg, [t], 1, check_overhead=0, limits=LimitConfig(grace_period=40))
    first_pause = min(r[0] for r in run["rpcs"] if r[2] == int(TransitionKind.PauseSideTask))
    assert run["kills"] == [(first_pause + 40, "rogue", run["kills"][0][2], 1)]   # SPEC acceptance 6
    assert run["dispositions"][0][1] == 3                                       # killed-pause-timeout


def test_fig9_oom_kill(product):
    cfg = fig_cfg(6)
    t = SideTaskSpec("leak", per_step_duration=4, memory_demand=6.0, memory_limit=8.0,
                     misbehavior=MisbehaviorKind.MemoryLeak, leak_rate_gib_per_s=20.0)
    base = product.run_experiment(cfg, [t], 1, with_tasks=False)["makespan"]
    run = product.run_experiment(cfg, [t], 1, check_overhead=0)
    assert len(run["kills"]) == 1 and run["kills"][0][3] == 0                   # OOM
    k = run["kills"][0][0]
    busy = sum(min(a[1], k) - a[0] for a in run["activities"] if a[4] == int(ActivityKind.Step) and a[0] < k)
    assert 6.0 + 20.0 * busy * 1e-3 > 8.0                       # exceeded at the kill tick ...
    assert 6.0 + 20.0 * (busy - 1) * 1e-3 <= 8.0                # ... and not one tick earlier
    assert run["makespan"] == base                              # training unaffected


def test_determinism_and_breakdown_conservation(product):
    rng = random.Random(5)
    for _ in range(60):
        cfg, tasks, kw, limits = rand_case(rng)
        a = product.run_experiment(cfg, tasks, 11, True, limits=limits, **kw)
        b = product.run_experiment(cfg, tasks, 11, True, limits=limits, **kw)
        assert a == b                                                # SPEC acceptance 9
        profiles = [TaskProfile(t.id, 0.0, 0.0, t.memory_demand, 1) for t in tasks]
        bubbles = [Bubble(s, e, st, d, av, BubbleType(bt)) for s, e, st, d, av, bt in a["bubbles"]]
        bd = product.bubble_breakdown(
            cfg.num_stages, profiles, bubbles, [AssignRecord(t, k, w) for t, k, w in a["assigns"]],
            [TransitionRecord(t, k, TransitionKind(kind), w) for t, k, kind, w in a["transitions"]],
            [ActivityRecord(s, e, k, w, ActivityKind(kind), c) for s, e, k, w, kind, c in a["activities"]])
        for s, sb in enumerate(bd):                                  # SPEC acceptance 7
            assert sb.total() == sum(d for st, e, x, d, *_ in a["bubbles"] if st == s)
