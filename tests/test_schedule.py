"""The executor's per-stage op lists (schedule.stage_ops, closed form) equal
the event order of the reference schedule as simulated by the planner
(trace documents of simulate_plan, proj/src/pipeline.cpp:96-297)."""
import json

import pytest

from paper_2509_21275_b200 import model as M
from paper_2509_21275_b200 import schedule as S


@pytest.mark.parametrize("dp", [1, 2, 4, 8])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_oplists_match_simulated_trace(planner, dp, seed):
    m = M.MODELS["gpt-1.3b"]
    cfg = M.planner_config(m, dp, mem_capacity=60e9 if dp > 1 else 120e9)
    lengths = planner.generate_workload("github_like", 96, seed, 65536)
    doc = planner.make_plan_document(cfg, lengths, None, "main", 4)
    plan = S.parse_plan(doc, lengths)
    trace, _ = planner.simulate_plan_document(doc)
    tr = json.loads(trace)
    assert len(tr["units"]) == len(plan.units)
    for u, tu in zip(plan.units, tr["units"]):
        n = len(u.chunks)
        for p in range(1, dp + 1):
            ev = sorted((e for e in tu["events"] if e["stage"] == p and e["op"] in ("F", "B")),
                        key=lambda e: (e["start"], 0 if e["op"] == "F" else 1))
            want = [(e["op"], e["pos"]) for e in ev]
            got = S.stage_ops(n, u.n_prefill, dp, p, u.backward_order)
            assert got == want, (p, got[:8], want[:8])
        # checkpoint counts per (stage, pos) equal the recompute events' layers
        for e in tu["events"]:
            if e["op"] == "R":
                assert u.ckpt[e["stage"] - 1][e["pos"]] > 0


def test_token_layout_covers_every_token_once(planner):
    cfg = M.planner_config(M.MODELS["gpt-1.3b"], 4, mem_capacity=180e9)
    lengths = planner.generate_workload("github_like", 128, 9, 32768)
    plan = S.parse_plan(planner.make_plan_document(cfg, lengths, None, "main", 4), lengths)
    seen = {}
    for lay in plan.chunks.values():
        assert sum(n for (_, _, n) in lay.members) == lay.tokens
        for (s, start, n) in lay.members:
            for t in range(start, start + n):
                assert (s, t) not in seen
                seen[(s, t)] = lay.id
    assert len(seen) == sum(lengths)
    tokens = S.synthetic_tokens(lengths, 50304, 0)
    n_targets = 0
    for lay in plan.chunks.values():
        ids, tgt = S.chunk_token_arrays(lay, tokens)
        assert len(ids) == lay.tokens
        n_targets += int((tgt >= 0).sum())
    assert n_targets == plan.total_targets
