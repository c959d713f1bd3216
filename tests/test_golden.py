"""The product planner reproduces the reference planner's committed output
bytes (tests/golden/planner_fixtures.json, generated from oracle/_ref by
tests/golden/make_golden.py) — plan documents, trace documents, errors and
synthetic workloads.  Runs anywhere (no /root/reference needed)."""
import json
from pathlib import Path

import pytest

FIX = json.loads((Path(__file__).parent / "golden" / "planner_fixtures.json").read_text())


@pytest.mark.parametrize("fx", FIX["fixtures"], ids=[f["name"] for f in FIX["fixtures"]])
def test_plan_bytes(planner, fx):
    if fx["error"]:
        with pytest.raises(getattr(planner, fx["error"][0])) as e:
            planner.make_plan_document(fx["config"], fx["lengths"], fx["slices"], fx["mode"], 2)
        assert str(e.value) == fx["error"][1]
        return
    for jobs in (1, 3):
        doc = planner.make_plan_document(fx["config"], fx["lengths"], fx["slices"], fx["mode"], jobs)
        assert doc == fx["plan"], f"{fx['name']} jobs={jobs}"
    if fx["trace"]:
        trace, _ = planner.simulate_plan_document(fx["plan"])
        assert trace == fx["trace"]


@pytest.mark.parametrize("name", sorted(FIX["workloads"]))
def test_workload_vectors(planner, name):
    want = FIX["workloads"][name]
    preset, seed = name.rsplit("_", 1)
    seed = int(seed)
    if preset == "github_like":
        got = planner.generate_workload(preset, 512, seed, 196608)
    elif preset == "commoncrawl_like":
        got = planner.generate_workload(preset, 300, seed, 131072)
    else:
        got = planner.generate_workload(preset, 100, seed, 8192, 100, 0)
    assert got == want


def test_worked_example_layout(planner):
    """SURVEY §8b worked example: chunk 2 = tail of seq 0 + packed shorts."""
    from paper_2509_21275_b200 import schedule
    fx = next(f for f in FIX["fixtures"] if f["name"] == "worked_example")
    plan = schedule.parse_plan(fx["plan"], fx["lengths"])
    kinds = {c.id: c.kind for c in plan.chunks.values()}
    assert kinds[0] == 1 and kinds[2] == 2
    # members in packer order: tail first, then shorts by (tokens desc, seq asc)
    assert [m[0] for m in plan.chunks[2].members] == [0, 3]
    assert [m[0] for m in plan.chunks[3].members] == [4, 1, 2]
