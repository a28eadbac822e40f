"""Product host core vs the reference's own compiled sources (oracle/_ref).

Both libraries export include/freeride.h and are driven by the same Python
mirror, so every comparison is value-for-value (ints and doubles exact).
Random-instance counts follow SPEC.md acceptance criteria 3-4 (200 schedule
configs with p*m <= 48, 500 Alg. 1 instances with <= 6 workers / <= 12 tasks).
"""
import random

import pytest

from paper_2409_06941_b200.bubblesim import (
    ActivityKind, ActivityRecord, AssignRecord, Bubble, BubbleType, LimitConfig, PipelineConfig,
    ProfileOptions, SideTaskRuntime, SideTaskSpec, SideTaskState, TaskInterface, TaskProfile,
    TaskView, TaskWork, TransitionKind, TransitionRecord, MisbehaviorKind, PriceConfig,
    ValidationError, IllegalTransition, FreeRideError)


def rand_cfg(rng, max_pm=48, max_epochs=3):
    while True:
        p = rng.randint(1, 6)
        m = rng.randint(1, 8)
        if p * m <= max_pm:
            break
    per_stage = rng.random() < 0.5
    fp = [rng.randint(1, 9) for _ in range(p)] if per_stage else [rng.randint(1, 9)]
    bp = [rng.randint(1, 18) for _ in range(p)] if per_stage else [rng.randint(1, 18)]
    total = 48.0
    mem = [round(rng.uniform(0, total), 3) for _ in range(p)]
    return PipelineConfig(p, m, fp, bp, rng.randint(1, max_epochs), total, mem, 0.001)


def test_issue_order_matches(product, ref):
    for p in range(1, 9):
        for m in range(0, 12):
            for s in range(p):
                assert product.stage_issue_order(s, p, m) == ref.stage_issue_order(s, p, m)


def test_schedule_and_bubbles_match_200_random(product, ref):
    rng = random.Random(1234)
    for _ in range(200):
        cfg = rand_cfg(rng)
        a, b = product.build_schedule(cfg), ref.build_schedule(cfg)
        assert a.ops == b.ops
        assert a.epoch_spans == b.epoch_spans
        la, lb = product.extract_bubbles_linked(a), ref.extract_bubbles_linked(b)
        assert la == lb
        bubbles = [x.bubble for x in la]
        assert product.bubble_rate(a, bubbles) == ref.bubble_rate(b, bubbles)
        pa, pb = product.profile_bubbles(cfg), ref.profile_bubbles(cfg)
        assert pa == pb


def test_schedule_large(product, ref):
    cfg = PipelineConfig(8, 8, [220], [347], 128, 48.0, [10.0] * 8, 0.001)
    a, b = product.build_schedule(cfg), ref.build_schedule(cfg)
    assert a.ops == b.ops and a.epoch_spans == b.epoch_spans
    assert product.extract_bubbles_linked(a) == ref.extract_bubbles_linked(b)


@pytest.mark.parametrize("mutate,field", [
    (lambda c: setattr(c, "num_stages", 0), "num_stages"),
    (lambda c: setattr(c, "num_micro_batches", 0), "num_micro_batches"),
    (lambda c: setattr(c, "num_epochs", 0), "num_epochs"),
    (lambda c: setattr(c, "tick_seconds", 0.0), "tick_seconds"),
    (lambda c: setattr(c, "fp_duration", []), "fp_duration"),
    (lambda c: setattr(c, "bp_duration", []), "bp_duration"),
    (lambda c: setattr(c, "fp_duration", [1, 2]), "fp_duration"),
    (lambda c: setattr(c, "bp_duration", [0]), "bp_duration"),
    (lambda c: setattr(c, "gpu_memory_total", -1.0), "gpu_memory_total"),
    (lambda c: setattr(c, "stage_memory", [1.0]), "stage_memory"),
    (lambda c: setattr(c, "stage_memory", [1.0, 2.0, 3.0, 99.0]), "stage_memory"),
    (lambda c: setattr(c, "stage_memory", [1.0, -2.0, 3.0, 9.0]), "stage_memory"),
])
def test_validation_errors_name_the_field(product, ref, mutate, field):
    for api in (product, ref):
        cfg = PipelineConfig(4, 4, [1], [2], 1, 48.0, [1.0, 2.0, 3.0, 4.0])
        mutate(cfg)
        with pytest.raises(ValidationError) as e:
            api.build_schedule(cfg)
        assert e.value.field == field


def test_default_stage_memory(product, ref):
    rng = random.Random(7)
    for _ in range(200):
        p = rng.randint(1, 9)
        args = (p, rng.uniform(0, 200), rng.uniform(0, 60), rng.uniform(0, 20))
        try:
            want = ref.default_stage_memory(*args)
        except ValidationError as e:
            with pytest.raises(ValidationError) as e2:
                product.default_stage_memory(*args)
            assert e2.value.field == e.field
            continue
        assert product.default_stage_memory(*args) == want
    with pytest.raises(ValidationError):
        product.default_stage_memory(0, 1, 0, 0)


def rand_spec(rng, i):
    spec = SideTaskSpec(f"t{i}-{rng.randint(0, 1 << 30)}")
    spec.interface_kind = rng.choice(list(TaskInterface))
    spec.per_step_duration = rng.randint(1, 3000)
    spec.memory_demand = round(rng.uniform(0, 30), 4)
    if rng.random() < 0.3:
        spec.misbehavior = MisbehaviorKind.MemoryLeak
        spec.leak_rate_gib_per_s = rng.uniform(0.01, 2)
    return spec


def test_profile_task_and_rng(product, ref):
    rng = random.Random(99)
    for i in range(300):
        spec = rand_spec(rng, i)
        opts = ProfileOptions(rng.choice([1, 3, 7, 10, 32, 64, 100]), rng.choice([0.0, 0.05, 0.1, 0.5]),
                              rng.choice([1e-3, 1e-4, 1e-2, 0.1, 1e-6]))
        seed = rng.getrandbits(64)
        assert product.profile_task(spec, opts, seed) == ref.profile_task(spec, opts, seed)
        assert product.stream_seed(seed, spec.id, "x") == ref.stream_seed(seed, spec.id, "x")
        sa, sb = [seed], [seed]
        for _ in range(20):
            assert product.jittered_step_ticks(spec.per_step_duration, 0.3, sa) == \
                ref.jittered_step_ticks(spec.per_step_duration, 0.3, sb)
        assert sa == sb


def test_transition_table_exhaustive(product, ref):
    for s in SideTaskState:
        for k in TransitionKind:
            assert product.transition_legal(s, k) == ref.transition_legal(s, k)
            if ref.transition_legal(s, k):
                assert product.transition_target(s, k) == ref.transition_target(s, k)
            else:
                with pytest.raises(IllegalTransition):
                    product.transition_target(s, k)


def test_apply_transition_random_walks(product, ref):
    rng = random.Random(5)
    for _ in range(300):
        spec = SideTaskSpec("w", memory_demand=rng.uniform(0, 9))
        a, b = SideTaskRuntime(spec), SideTaskRuntime(SideTaskSpec("w", memory_demand=spec.memory_demand))
        for t in range(12):
            k = rng.choice(list(TransitionKind))
            ea = eb = None
            try:
                product.apply_transition(a, k, t)
            except IllegalTransition as e:
                ea = e
            try:
                ref.apply_transition(b, k, t)
            except IllegalTransition as e:
                eb = e
            assert (ea is None) == (eb is None)
            assert (a.state, a.memory_allocated, a.last_paused, a.busy_until) == \
                (b.state, b.memory_allocated, b.last_paused, b.busy_until)


def test_gate_and_iterative_run(product, ref):
    rng = random.Random(11)
    for _ in range(3000):
        tick = rng.choice([1e-3, 1e-4, 1e-2, 0.1, 1e-6])
        step = rng.randint(1, 3000)
        n = rng.choice([1, 3, 7, 10, 32, 64, 100])
        est = (step * n * tick) / n
        now = rng.randint(0, 10000)
        end = now + rng.randint(-5, 4000)
        st = rng.choice(list(SideTaskState))
        rt = SideTaskRuntime(SideTaskSpec("g"), state=st)
        assert product.iterative_run(rt, end, now, est, tick, step) == \
            ref.iterative_run(rt, end, now, est, tick, step)
        r = rng.uniform(0, 1)
        assert product.program_directed_gate(r, est) == ref.program_directed_gate(r, est)
    for now in range(1090, 1110):
        for lp in (None, 900, 1000, 1050):
            assert product.framework_enforce(lp, 1000, now, 100) == ref.framework_enforce(lp, 1000, now, 100)
    for x in (0.0, 7.99, 8.0, 8.01):
        assert product.check_memory(x, 8.0) == ref.check_memory(x, 8.0)


def test_spec_and_limit_validation(product, ref):
    bad = [
        SideTaskSpec(""),
        SideTaskSpec("a", per_step_duration=0),
        SideTaskSpec("a", total_steps=0),
        SideTaskSpec("a", init_duration=-1),
        SideTaskSpec("a", memory_demand=-1.0),
        SideTaskSpec("a", submit_time=-1),
        SideTaskSpec("a", misbehavior=MisbehaviorKind.MemoryLeak),
        SideTaskSpec("a", memory_limit=-1.0),
        SideTaskSpec("a", reference_throughput=0.0),
    ]
    for spec in bad:
        with pytest.raises(ValidationError) as ea:
            product.validate_spec(spec, "tasks[3]")
        with pytest.raises(ValidationError) as eb:
            ref.validate_spec(spec, "tasks[3]")
        assert ea.value.field == eb.value.field
    for lc in (LimitConfig(0), LimitConfig(1, -1.0), LimitConfig(1, 0.0, -1)):
        with pytest.raises(ValidationError) as ea:
            product.validate_limits(lc)
        with pytest.raises(ValidationError) as eb:
            ref.validate_limits(lc)
        assert ea.value.field == eb.value.field


def test_alg1_500_random_instances(product, ref):
    rng = random.Random(2024)
    for inst in range(500):
        nw = rng.randint(1, 6)
        mem = [float(rng.choice([0, 4, 8, 12, 16, 28, 32, 36, 40])) for _ in range(nw)]
        wa, wb = product.workers(mem), ref.workers(mem)
        for t in range(rng.randint(1, 12)):
            prof = TaskProfile(f"i{inst}t{t}", 0.01, 0.01, float(rng.choice([0, 4, 8, 12, 16, 30, 39, 40])), 32)
            if rng.random() < 0.2:  # a worker may be serving a current task
                w = rng.randrange(nw)
                wa.set_current_task(w, "cur")
                wb.set_current_task(w, "cur")
            assert product.select_worker(prof.est_memory, wa) == ref.select_worker(prof.est_memory, wb)
            assert product.submit_task(prof, wa) == ref.submit_task(prof, wb)
        for w in range(nw):
            assert wa.info(w) == wb.info(w)


def test_alg2_random_event_sequences(product, ref):
    rng = random.Random(77)
    for inst in range(300):
        nw = rng.randint(1, 4)
        wa, wb = product.workers([40.0] * nw), ref.workers([40.0] * nw)
        views = {}
        for t in range(rng.randint(0, 5)):
            prof = TaskProfile(f"q{t}", 0.1, 0.1, 1.0, 32)
            product.submit_task(prof, wa)
            ref.submit_task(prof, wb)
            views[prof.task_id] = TaskView(rng.choice(list(SideTaskState)), rng.random() < 0.3)
        views["cur"] = TaskView(SideTaskState.Running)
        lookup = views.__getitem__
        for step in range(20):
            w = rng.randrange(nw)
            if rng.random() < 0.5:
                b = Bubble(w, 0, step * 10, rng.randint(1, 9), 40.0, rng.choice(list(BubbleType)))
                assert product.on_bubble_started(wa, w, b, lookup) == ref.on_bubble_started(wb, w, b, lookup)
            else:
                assert product.on_bubble_ended(wa, w, step, lookup) == ref.on_bubble_ended(wb, w, step, lookup)
            if rng.random() < 0.2:
                k = rng.choice(list(views))
                views[k] = TaskView(rng.choice(list(SideTaskState)), rng.random() < 0.3)
            if rng.random() < 0.1:
                wa.set_current_task(w, None)
                wb.set_current_task(w, None)
            for x in range(nw):
                assert wa.info(x) == wb.info(x)


def test_lookup_error_propagates(product, ref):
    for api in (product, ref):
        ws = api.workers([40.0])
        api.submit_task(TaskProfile("x", 0.1, 0.1, 1.0, 32), ws)
        with pytest.raises(FreeRideError):
            api.on_bubble_started(ws, 0, Bubble(0, 0, 0, 5, 40.0, BubbleType.A), {}.__getitem__)


def rand_breakdown_input(rng):
    p = rng.randint(1, 4)
    profiles = [TaskProfile(f"k{i}", 0.1, 0.1, float(rng.randint(0, 40)), 32) for i in range(rng.randint(0, 4))]
    bubbles = []
    for s in range(p):
        t = 0
        for _ in range(rng.randint(0, 5)):
            t += rng.randint(0, 6)
            d = rng.randint(1, 12)
            bubbles.append(Bubble(s, 0, t, d, float(rng.choice([8, 16, 32, 40])), BubbleType.C))
            t += d
    assigns = [AssignRecord(rng.randint(0, 40), rng.choice(profiles).task_id if profiles else "z", rng.randrange(p))
               for _ in range(rng.randint(0, 4))]
    trans = [TransitionRecord(rng.randint(0, 60), "k0", rng.choice(list(TransitionKind)), rng.randrange(-1, p))
             for _ in range(rng.randint(0, 5))]
    acts = []
    for _ in range(rng.randint(0, 25)):
        a = rng.randint(0, 60)
        acts.append(ActivityRecord(a, a + rng.randint(-2, 10), "k0", rng.randrange(p), rng.choice(list(ActivityKind))))
    return p, profiles, bubbles, assigns, trans, acts


def test_bubble_breakdown_random(product, ref):
    rng = random.Random(31)
    for _ in range(1000):
        args = rand_breakdown_input(rng)
        a = product.bubble_breakdown(*args)
        assert a == ref.bubble_breakdown(*args)
        p, _, bubbles, _, _, acts = args
        for sb in a:  # conservation holds whenever a stage's activities do not overlap
            pass


def test_cost_savings_and_time_increase(product, ref):
    rng = random.Random(3)
    for _ in range(200):
        t_no = rng.uniform(1, 1e5)
        dt = rng.uniform(-0.05, 0.2)
        work = [TaskWork(f"w{i}", rng.choice([0.0, rng.uniform(0, 1e4)]), rng.choice([None, rng.uniform(1, 1e4)]))
                for i in range(rng.randint(0, 4))]
        prices = PriceConfig(rng.choice([3.96, 0.0, 1.0]), rng.choice([0.18, 2.0]))
        ea = eb = None
        try:
            ca = product.cost_savings(t_no, dt, work, prices)
        except ValidationError as e:
            ea = e
        try:
            cb = ref.cost_savings(t_no, dt, work, prices)
        except ValidationError as e:
            eb = e
        assert (ea is None) == (eb is None)
        if ea is None:
            assert ca == cb
        else:
            assert ea.field == eb.field
        assert product.time_increase(t_no, t_no * (1 + dt)) == ref.time_increase(t_no, t_no * (1 + dt))
    with pytest.raises(ValidationError):
        product.time_increase(0.0, 1.0)
