"""Pipeline ΔT from per-stage replica measurements.

In replica mode each GPU replays one stage against the *undelayed* dependency
times of the other stages, so a stage's slower ops are charged to its own
makespan only when it has no slack (stage 0: its last BP ends the epoch);
the stages with trailing bubbles absorb them.  A real pipeline charges them
along the critical path (ΔT = makespan growth of pipeline
training; reference metrics.cpp:18-22).

critical_path_dt() feeds the measured per-stage FP / BP op durations of the
runs with and without side tasks into the product's own build_schedule (the
reference's 1F1B DAG, pipeline.cpp:111-132: same-stage chain across epochs,
FP(s-1)->FP(s), BP(s+1)->BP(s), FP(s)->BP(s)) and returns the makespan
growth through time_increase (metrics.cpp:18-22).  Any start delay an op
suffers from a side step still holding the SMs when it becomes ready lands in
the op's measured duration (its start event is recorded when its dependency
wait ends), so the durations carry both effects.
"""
from __future__ import annotations

import statistics
from typing import Dict, List, Sequence, Tuple


def op_means(ops: Sequence[Tuple[float, float]], kinds: Sequence[int]) -> Tuple[float, float]:
    """(mean FP, mean BP) duration in seconds; kinds = the stage's issue-order
    op kinds (0 = FP, 1 = BP) of one epoch, repeated over the run's epochs"""
    n = len(kinds)
    fp = [b - a for i, (a, b) in enumerate(ops) if kinds[i % n] == 0]
    bp = [b - a for i, (a, b) in enumerate(ops) if kinds[i % n] == 1]
    return statistics.fmean(fp), statistics.fmean(bp)


def issue_kinds(api, stage: int, p: int, m: int) -> List[int]:
    """op kinds (0 = FP, 1 = BP) of stage_issue_order(stage, p, m)"""
    return [int(k) for k, _mb in api.stage_issue_order(stage, p, m)]


def makespan(api, p: int, m: int, epochs: int, fp_s: Sequence[float], bp_s: Sequence[float]) -> int:
    """build_schedule makespan (ns ticks) of a p-stage 1F1B pipeline with the
    given per-stage op durations (seconds)"""
    from .bubblesim import PipelineConfig
    cfg = PipelineConfig(p, m, [max(1, round(x * 1e9)) for x in fp_s], [max(1, round(x * 1e9)) for x in bp_s],
                         epochs, 1.0, [1.0] * p, 1e-9)
    tr = api.build_schedule(cfg)
    return tr.epoch_spans[-1][1] - tr.epoch_spans[0][0]


def critical_path_dt(api, p: int, m: int, epochs: int, base: Dict[int, Tuple[float, float]],
                     with_: Dict[int, Tuple[float, float]]) -> dict:
    """base / with_: stage -> (mean FP s, mean BP s).  Stages missing from
    with_ run no side task (their base durations are used)."""
    fb = [base[s][0] for s in range(p)]
    bb = [base[s][1] for s in range(p)]
    fw = [with_.get(s, base[s])[0] for s in range(p)]
    bw = [with_.get(s, base[s])[1] for s in range(p)]
    t0 = makespan(api, p, m, epochs, fb, bb)
    t1 = makespan(api, p, m, epochs, fw, bw)
    return {"dT": api.time_increase(t0 * 1e-9, t1 * 1e-9), "makespan_no_s": t0 * 1e-9, "makespan_with_s": t1 * 1e-9,
            "op_growth": {s: (fw[s] / fb[s] - 1.0, bw[s] / bb[s] - 1.0) for s in range(p)}}
