"""Measured per-op traces in the reference's trace document schema.

The planner simulates every unit of a plan (proj/src/pipeline.cpp:96-297)
and emits a trace document v1 (proj/src/plan_io.cpp:169-209): per unit the
events {stage, chunk, pos, op F/B/R, start, end}, makespan, bubble ratio,
per-stage peak memory and memory series.  The CUDA stages record the same
events on the device (include/epp_gpu.h epp_stage_trace*), so a training step
yields a *measured* document of the same shape, which the planner's own tools
read (trace_from_json, render) and which is diffed event by event against the
simulated one (`residuals`): the closed-loop cost fit's per-op error.
"""
from __future__ import annotations

import json
from typing import Dict, List, Optional, Sequence

from .schedule import Plan

OPS = {0: "F", 1: "B", 2: "R"}


def _unit_of(plan: Plan) -> Dict[int, tuple]:
    out = {}
    for u, unit in enumerate(plan.units):
        for pos, cid in enumerate(unit.chunks):
            out[cid] = (u, pos)
    return out


def measured_trace(plan: Plan, stage_events: Dict[int, Sequence[dict]],
                   state_bytes: Optional[Sequence[float]] = None, mem_capacity: float = 0.0) -> dict:
    """Trace document v1 of one executed step.

    stage_events[p] (p 1-based): the events CudaStage.trace_read() returned
    on stage p, in issue order, times in seconds from that stage's trace
    origin (all stages' origins are taken after a barrier, so they agree to
    within the barrier's skew).  Each unit's times are made relative to the
    unit's first event (the simulator starts every unit at 0).  Memory:
    state_bytes[p-1] (the stage's resident weights / optimizer state, as the
    planner's stage_state_bytes) + the activation bytes the stage held after
    each op (`live`)."""
    where = _unit_of(plan)
    dp = plan.pp_degree
    n_units = len(plan.units)
    per_unit: List[List[dict]] = [[] for _ in range(n_units)]
    mem: List[List[List[tuple]]] = [[[] for _ in range(dp)] for _ in range(n_units)]
    for p, evs in stage_events.items():
        for e in evs:
            u, pos = where[int(e["chunk"])]
            per_unit[u].append({"stage": int(p), "chunk": int(e["chunk"]), "pos": pos, "op": e["op"],
                                "start": float(e["start"]), "end": float(e["end"])})
            if e["op"] != "R":
                mem[u][p - 1].append((float(e["end"]), float(e.get("live", 0))))
    units = []
    total = busy = weighted = 0.0
    for u in range(n_units):
        evs = per_unit[u]
        if not evs:
            continue
        t0 = min(e["start"] for e in evs)
        for e in evs:
            e["start"] -= t0
            e["end"] -= t0
        evs.sort(key=lambda e: (e["start"], e["stage"], e["pos"]))
        makespan = max(e["end"] for e in evs)
        stage_busy = [0.0] * dp
        for e in evs:
            stage_busy[e["stage"] - 1] += e["end"] - e["start"]
        base = [float(state_bytes[p]) if state_bytes else 0.0 for p in range(dp)]
        series, peak = [], []
        for p in range(dp):
            s = [[0.0, base[p]]] + [[t - t0, base[p] + b] for (t, b) in sorted(mem[u][p])]
            series.append(s)
            peak.append(max(x[1] for x in s))
        units.append({"makespan": makespan,
                      "bubble_ratio": 1.0 - sum(stage_busy) / (dp * makespan) if makespan > 0 else 0.0,
                      "peak_memory": peak,
                      "capacity_violation": [bool(mem_capacity and x > mem_capacity) for x in peak],
                      "events": evs, "memory": series})
        total += makespan
        busy += sum(stage_busy)
        weighted += makespan * dp
    return {"version": 1, "kind": "trace", "units": units, "total_seconds": total,
            "bubble_ratio": 1.0 - busy / weighted if weighted > 0 else 0.0}


def residuals(measured: dict, simulated) -> dict:
    """Per-event comparison of a measured trace with the planner's simulated
    trace of the same plan: relative duration error per op kind (mean of
    |measured - simulated| / simulated, and the duration-weighted signed
    error), per-unit makespan ratio, bubble ratios."""
    sim = json.loads(simulated) if isinstance(simulated, (str, bytes)) else simulated
    if len(sim["units"]) != len(measured["units"]):
        raise ValueError("traces cover different numbers of units")
    per_op: Dict[str, dict] = {}
    ratios = []
    for mu, su in zip(measured["units"], sim["units"]):
        key = {(e["stage"], e["chunk"], e["op"]): e["end"] - e["start"] for e in su["events"]}
        for e in mu["events"]:
            d_sim = key.get((e["stage"], e["chunk"], e["op"]))
            if d_sim is None or d_sim <= 0:
                continue
            d = e["end"] - e["start"]
            r = per_op.setdefault(e["op"], {"events": 0, "abs_rel": 0.0, "measured_s": 0.0, "simulated_s": 0.0})
            r["events"] += 1
            r["abs_rel"] += abs(d - d_sim) / d_sim
            r["measured_s"] += d
            r["simulated_s"] += d_sim
        if su["makespan"] > 0:
            ratios.append(mu["makespan"] / su["makespan"])
    ops = {}
    for k, r in sorted(per_op.items()):
        ops[k] = {"events": r["events"], "mean_abs_rel_err": r["abs_rel"] / r["events"],
                  "weighted_rel_err": (r["measured_s"] - r["simulated_s"]) / r["simulated_s"]
                  if r["simulated_s"] > 0 else None}
    return {"per_op": ops,
            "makespan_measured_s": measured["total_seconds"], "makespan_simulated_s": sim["total_seconds"],
            "makespan_ratio": measured["total_seconds"] / sim["total_seconds"] if sim["total_seconds"] else None,
            "unit_makespan_ratio_min": min(ratios) if ratios else None,
            "unit_makespan_ratio_max": max(ratios) if ratios else None,
            "bubble_ratio_measured": measured["bubble_ratio"], "bubble_ratio_simulated": sim["bubble_ratio"]}
