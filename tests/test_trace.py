"""Measured trace documents (paper_2509_21275_b200/trace.py): built from
per-stage event lists in the shape the CUDA stages record them
(include/epp_gpu.h epp_stage_trace_read), they are trace documents v1 the
reference's own reader accepts (proj/src/plan_io.cpp:169-209 trace_to_json /
trace_from_json, read here through render), and a step whose measured events
equal the simulated ones has zero residuals."""
import json

import pytest

from paper_2509_21275_b200 import model as M
from paper_2509_21275_b200 import schedule as S
from paper_2509_21275_b200 import trace as T


def _plan(planner, dp, seed, tight=False):
    m = M.MODELS["gpt-1.3b"]
    cfg = M.planner_config(m, dp, mem_capacity=(28e9 if tight else 120e9))
    lengths = planner.generate_workload("github_like", 64, seed, 32768)
    doc = planner.make_plan_document(cfg, lengths, None, "main", 4)
    return doc, S.parse_plan(doc, lengths)


def _as_stage_events(sim, offset=0.0):
    """The simulated trace's events laid out the way a stage reports them:
    per stage, issue order, one clock per stage running across units."""
    per = {}
    t0 = 0.0
    for u in sim["units"]:
        for e in sorted(u["events"], key=lambda e: (e["start"], e["op"] != "R")):
            per.setdefault(e["stage"], []).append({"chunk": e["chunk"], "op": e["op"],
                                                   "start": e["start"] + t0 + offset,
                                                   "end": e["end"] + t0 + offset, "live": 1000})
        t0 += u["makespan"] + 0.5
    return per


@pytest.mark.parametrize("dp,tight", [(1, False), (2, False), (4, True), (8, True)])
def test_simulated_events_round_trip(planner, dp, tight):
    doc, plan = _plan(planner, dp, dp, tight)
    sim_text, total = planner.simulate_plan_document(doc)
    sim = json.loads(sim_text)
    meas = T.measured_trace(plan, _as_stage_events(sim, offset=3.0), state_bytes=[1e9] * dp,
                            mem_capacity=180e9)
    assert meas["kind"] == "trace" and meas["version"] == 1
    assert len(meas["units"]) == len(sim["units"])
    for mu, su in zip(meas["units"], sim["units"]):
        key = lambda e: (e["stage"], e["chunk"], e["op"])   # noqa: E731
        got = sorted((key(e), e["pos"], round(e["start"], 9), round(e["end"], 9)) for e in mu["events"])
        want = sorted((key(e), e["pos"], round(e["start"], 9), round(e["end"], 9)) for e in su["events"])
        assert got == want
        assert mu["makespan"] == pytest.approx(su["makespan"], rel=1e-12)
        assert mu["bubble_ratio"] == pytest.approx(su["bubble_ratio"], rel=1e-9, abs=1e-12)
        assert len(mu["memory"]) == dp and all(s[0] == [0.0, 1e9] for s in mu["memory"])
    assert meas["total_seconds"] == pytest.approx(total, rel=1e-12)
    r = T.residuals(meas, sim_text)
    assert r["makespan_ratio"] == pytest.approx(1.0)
    assert set(r["per_op"]) >= {"F", "B"}
    for v in r["per_op"].values():
        assert v["mean_abs_rel_err"] == pytest.approx(0.0, abs=1e-9)
    if tight:
        assert "R" in r["per_op"], "tight memory should produce recompute events"
    # the reference's trace reader (through render) accepts the document
    svg = planner.render_svg(json.dumps(meas))
    assert svg.startswith("<svg") or "<svg" in svg[:200]


def test_residuals_scale(planner):
    doc, plan = _plan(planner, 2, 5)
    sim_text, _ = planner.simulate_plan_document(doc)
    sim = json.loads(sim_text)
    per = _as_stage_events(sim)
    slow = {p: [dict(e, start=e["start"] * 1.1, end=e["end"] * 1.1) for e in evs] for p, evs in per.items()}
    r = T.residuals(T.measured_trace(plan, slow), sim_text)
    assert r["per_op"]["F"]["mean_abs_rel_err"] == pytest.approx(0.1, rel=1e-6)
    assert r["per_op"]["B"]["weighted_rel_err"] == pytest.approx(0.1, rel=1e-6)
