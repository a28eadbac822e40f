"""CPU-only: the measured-trace mode of replay_check (a RunTrace recorded on
the GPU by fr_harness_run_trace) and the pipeline ΔT of the
bench (paper_2409_06941_b200/pipeline_dt.py)."""
import json

import pytest

from paper_2409_06941_b200 import pipeline_dt as PD
from paper_2409_06941_b200.bubblesim import PipelineConfig, SideTaskSpec


def _trace(product, tmp_path):
    cfg = PipelineConfig(4, 4, [3], [5], 2, 48.0, [10, 20, 30, 40], 1e-3)
    t = SideTaskSpec("pr")
    t.per_step_duration = 2
    t.memory_demand = 1.0
    p = str(tmp_path / "sim.jsonl")
    product.run_experiment(cfg, [t], 5, True, trace_path=p)
    return [json.loads(x) for x in open(p).read().splitlines()]


def _check(product, tmp_path, lines, name):
    p = str(tmp_path / name)
    with open(p, "w") as f:
        f.write("\n".join(json.dumps(x) for x in lines) + "\n")
    return product.replay_check_file(p)


def _no_checks(lines):
    """the GPU runtime records no Check activities (its gate runs on the host)"""
    return [x for x in lines if not (x.get("type") == "activity" and x["kind"] == "check")]


def _measured(lines, tol=0):
    out = [dict(x) for x in lines]
    out[0]["measured"] = True
    out[0]["tolerance"] = tol
    return out


def test_measured_flag_round_trips_and_sim_traces_stay_unchanged(product, tmp_path):
    lines = _trace(product, tmp_path)
    assert "measured" not in lines[0]          # simulated traces are byte-identical to round 1
    assert _check(product, tmp_path, _measured(lines), "m.jsonl") == []


def test_measured_op_durations_and_partial_stages(product, tmp_path):
    lines = _trace(product, tmp_path)
    # a measured op took one tick less than configured
    op = next(x for x in lines if x.get("type") == "op" and x["end"] - x["start"] > 1)
    op["end"] -= 1
    assert any("lasts" in v for v in _check(product, tmp_path, lines, "sim.jsonl"))
    assert _check(product, tmp_path, _measured(lines), "meas.jsonl") == []
    # a replica trace holds one stage only (and its worker's records)
    one = [x for x in _measured(lines) if x.get("type") not in ("op", "bubble", "activity") or
           x.get("stage", x.get("worker")) == 2]
    keep = {x["task"] for x in one if x.get("type") == "activity"}
    one = [x for x in one if x.get("type") not in ("transition", "rpc", "kill", "disposition", "submit", "assign")
           or x.get("task") in keep or x.get("type") in ("submit",)]
    v = _check(product, tmp_path, one, "one.jsonl")
    assert not any("distinct ops" in x for x in v), v


def test_measured_allows_a_step_tail_over_the_next_op(product, tmp_path):
    lines = _no_checks(_trace(product, tmp_path))
    ops = {(x["stage"], x["start"]): x for x in lines if x.get("type") == "op"}
    allacts = [x for x in lines if x.get("type") == "activity"]
    acts = [x for x in allacts if x["kind"] == "step"]
    assert acts

    def next_op(a):
        return min((o for (s, st), o in ops.items() if s == a["worker"] and st >= a["end"]),
                   key=lambda o: o["start"], default=None)
    # a step that is the last side activity before its stage's next op
    a = next(a for a in acts if next_op(a) and not any(
        b is not a and b["worker"] == a["worker"] and a["end"] <= b["start"] < next_op(a)["start"] for b in allacts))
    a["end"] = next_op(a)["start"] + 1          # the step's tail co-runs with the next op
    assert any("overlaps" in v for v in _check(product, tmp_path, lines, "sim.jsonl"))
    assert _check(product, tmp_path, _measured(lines), "meas.jsonl") == []


def test_measured_still_catches_logic_violations(product, tmp_path):
    lines = _measured(_trace(product, tmp_path))
    start = min(x["t"] for x in lines if x.get("type") == "transition" and x["kind"] == "start")
    step = next(x for x in lines if x.get("type") == "activity" and x["kind"] == "step")
    step["start"], step["end"] = start - 3, start - 2    # a step before StartSideTask
    v = _check(product, tmp_path, lines, "bad.jsonl")
    assert any("activity" in x for x in v), v


def test_tolerance_absorbs_clock_domain_skew(product, tmp_path):
    lines = _measured(_no_checks(_trace(product, tmp_path)), tol=2)
    start = min(x["t"] for x in lines if x.get("type") == "transition" and x["kind"] == "start")
    step = min((x for x in lines if x.get("type") == "activity" and x["kind"] == "step"), key=lambda x: x["start"])
    shift = step["start"] - (start - 1)
    step["start"] -= shift                     # 1 tick before the stamp of its StartSideTask
    assert _check(product, tmp_path, lines, "tol.jsonl") == []
    lines[0]["tolerance"] = 0
    assert _check(product, tmp_path, lines, "tol0.jsonl") != []


# ------------------------------------------------------------ pipeline ΔT
def test_pipeline_dt_no_change_is_zero(product):
    base = {s: (3e-3, 6e-3) for s in range(4)}
    r = PD.critical_path_dt(product, 4, 4, 4, base, base)
    assert r["dT"] == 0.0 and r["makespan_no_s"] == r["makespan_with_s"]


def test_pipeline_dt_uniform_slowdown_scales_makespan(product):
    base = {s: (3e-3, 6e-3) for s in range(4)}
    slow = {s: (3.3e-3, 6.6e-3) for s in range(4)}
    assert PD.critical_path_dt(product, 4, 4, 4, base, slow)["dT"] == pytest.approx(0.1, abs=1e-6)


def test_pipeline_dt_charges_a_slower_stage_through_the_dag(product):
    """one stage's ops 10 % slower: the linked pipeline pays it on the
    critical path (every micro-batch crosses every stage), far more than the
    replica of a stage with slack shows"""
    base = {s: (3e-3, 6e-3) for s in range(4)}
    r = PD.critical_path_dt(product, 4, 4, 4, base, {2: (3.3e-3, 6.6e-3)})
    assert 0.02 < r["dT"] < 0.1, r
    assert r["op_growth"][2] == pytest.approx((0.1, 0.1)) and r["op_growth"][0] == (0.0, 0.0)


def test_issue_kinds_follow_the_reference_order(product, ref):
    for s in range(4):
        assert PD.issue_kinds(product, s, 4, 4) == [int(k) for k, _ in ref.stage_issue_order(s, 4, 4)]


def test_op_means_by_kind():
    kinds = [0, 0, 1, 1]
    ops = [(0.0, 1.0), (1.0, 2.0), (2.0, 4.0), (4.0, 6.0)] * 2
    assert PD.op_means(ops, kinds) == (1.0, 2.0)
