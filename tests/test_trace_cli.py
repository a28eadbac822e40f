"""§8(f) row 3: the run-trace stream, replay_check and the command-line
front end (reference trace.hpp:16-22, engine.hpp:100-104, config.hpp:52-56,
cli.hpp:10-31, whose bodies the reference never shipped; SPEC.md:490-497,
519-557, acceptance 7 and 9)."""
import json
import os
import random
import subprocess

import pytest

from paper_2409_06941_b200.bubblesim import PipelineConfig, SideTaskSpec

from test_engine import rand_case

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SIM = os.path.join(ROOT, "paper_2409_06941_b200", "_lib", "freeride-sim")
CONFIGS = os.path.join(ROOT, "configs")


def sim(*args):
    return subprocess.run([SIM, *args], capture_output=True, text=True)


def test_replay_check_fuzz(product):
    """SPEC.md:574 acceptance 7: every seeded run is sound (1000 runs)."""
    rng = random.Random(2024)
    for case in range(500):
        cfg, tasks, kw, limits = rand_case(rng)
        seed = rng.getrandbits(64)
        for with_tasks in (True, False):
            tr = product.run_experiment(cfg, tasks, seed, with_tasks, limits=limits, check=True, **kw)
            assert tr["violations"] == [], (case, with_tasks, tr["violations"][:3])


def test_trace_round_trip_and_corruption(product, tmp_path):
    cfg = PipelineConfig(4, 4, [3], [5], 2, 48.0, [10, 20, 30, 40], 1e-3)
    t = SideTaskSpec("pr")
    t.per_step_duration = 2
    t.memory_demand = 1.0
    p1 = str(tmp_path / "a.jsonl")
    product.run_experiment(cfg, [t], 5, True, trace_path=p1)
    assert product.replay_check_file(p1) == []
    # byte-stable: read + write reproduces the file (via the CLI's check path)
    text = open(p1).read()
    lines = text.splitlines()
    assert json.loads(lines[0])["type"] == "meta" and json.loads(lines[-1])["type"] == "end"
    # corrupt: move one op onto its predecessor
    ops = [i for i, l in enumerate(lines) if json.loads(l)["type"] == "op"]
    rec = json.loads(lines[ops[5]])
    rec["start"] -= 1
    rec["end"] -= 1
    lines[ops[5]] = json.dumps(rec, separators=(",", ":"))
    p2 = str(tmp_path / "bad.jsonl")
    open(p2, "w").write("\n".join(lines) + "\n")
    v = product.replay_check_file(p2)
    assert v and any("before its" in x or "overlaps" in x for x in v), v
    r = sim("check", p2)
    assert r.returncode == 3 and "op" in r.stderr


@pytest.fixture(scope="module")
def built(product):
    assert os.path.exists(SIM)
    return SIM


def test_cli_run_is_deterministic_and_sound(built, tmp_path):
    """SPEC.md:576 acceptance 9: byte-identical traces for equal inputs."""
    a, b = str(tmp_path / "a"), str(tmp_path / "b")
    for out in (a, b):
        r = sim("run", os.path.join(CONFIGS, "mixed_workload.json"), "--out", out)
        assert r.returncode == 0, r.stderr
    for f in ("baseline.trace.jsonl", "treatment.trace.jsonl", "report.json", "breakdown.csv"):
        assert open(os.path.join(a, f), "rb").read() == open(os.path.join(b, f), "rb").read()
    rep = json.load(open(os.path.join(a, "report.json")))
    assert rep["delta_t"] == 0.0 and abs(rep["bubble_rate"] - 3 / 7) < 1e-12   # noise-free iterative: ΔT = 0
    assert sim("check", os.path.join(a, "treatment.trace.jsonl")).returncode == 0
    r = sim("run", os.path.join(CONFIGS, "mixed_workload.json"), "--out", str(tmp_path / "c"), "--seed", "99")
    assert r.returncode == 0


@pytest.mark.parametrize("name,disposition", [("fig9_oom", "killed-oom"),
                                              ("fig9_timeout", "killed-pause-timeout")])
def test_cli_fig9_scenarios(built, tmp_path, name, disposition):
    out = str(tmp_path / name)
    r = sim("run", os.path.join(CONFIGS, name + ".json"), "--out", out, "--format", "json-lines")
    assert r.returncode == 0, r.stderr
    rep = json.load(open(os.path.join(out, "report.json")))
    assert [d["disposition"] for d in rep["dispositions"]] == [disposition]
    assert os.path.exists(os.path.join(out, "breakdown.jsonl"))


def test_cli_sweep_bubble_rates(built, tmp_path):
    """micro-batch sweep {4, 8} with fp = bp = 1 -> 3/7, 3/11."""
    out = str(tmp_path / "sweep")
    r = sim("sweep", os.path.join(CONFIGS, "sweep_micro_batches.json"), "--out", out, "--jobs", "2")
    assert r.returncode == 0, r.stderr
    rows = open(os.path.join(out, "sweep.csv")).read().splitlines()
    assert rows[0].startswith("point,micro_batches")
    rates = [float(x.split(",")[4]) for x in rows[1:]]
    assert abs(rates[0] - 3 / 7) < 1e-12 and abs(rates[1] - 3 / 11) < 1e-12


def test_cli_profile_matches_appendix_a2(built):
    r = sim("profile", os.path.join(CONFIGS, "c1_pagerank.json"))
    assert r.returncode == 0
    d = json.loads(r.stdout)
    assert abs(d["bubble_rate"] - 3 / 7) < 1e-12
    assert [round(x * 1000) for x in d["stages"][0]["bubble_durations_s"]] == [220, 220, 220, 1041]
    assert [s["available_memory"] for s in d["stages"]] == [2.0, 8.5, 15.0, 21.5]


def test_cli_exit_codes(built, tmp_path):
    bad = tmp_path / "bad.json"
    bad.write_text("{ not json")
    r = sim("run", str(bad), "--out", str(tmp_path / "x"))
    assert r.returncode == 2                                 # schema / parse
    doc = json.load(open(os.path.join(CONFIGS, "mixed_workload.json")))
    doc["tasks"][1]["id"] = doc["tasks"][0]["id"]
    dup = tmp_path / "dup.json"
    dup.write_text(json.dumps(doc))
    r = sim("run", str(dup), "--out", str(tmp_path / "y"))
    assert r.returncode == 1 and "tasks[1].id" in r.stderr   # validation names the field
    doc = json.load(open(os.path.join(CONFIGS, "mixed_workload.json")))
    del doc["pipeline"]["num_stages"]
    miss = tmp_path / "miss.json"
    miss.write_text(json.dumps(doc))
    r = sim("profile", str(miss))
    assert r.returncode == 2 and "$.pipeline.num_stages" in r.stderr
    doc = json.load(open(os.path.join(CONFIGS, "mixed_workload.json")))
    doc["tasks"][0]["per_step_duration"] = 0.0305       # not a whole number of 1 ms ticks
    frac = tmp_path / "frac.json"
    frac.write_text(json.dumps(doc))
    assert sim("profile", str(frac)).returncode == 1
    assert sim("bogus", "x").returncode == 2
