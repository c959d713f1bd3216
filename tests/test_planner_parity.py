"""Byte-for-byte parity of the product planner with the compiled reference
(oracle/_ref) over seeds x configs x modes x slice counts, including error
classes/messages, traces and the cost fit."""
import json
import random

import pytest

from golden.make_golden import DESK8, TIGHT8, WORKED
from paper_2509_21275_b200 import model as M

MODES = ["main", "no_wbc", "no_ckpt", "full_ckpt"]


def both(planner, ref_api, cfg, lengths, slices, mode, jobs):
    out = []
    for lib in (None, ref_api):
        try:
            out.append(("ok", planner.make_plan_document(cfg, lengths, slices, mode, jobs, _lib=lib)))
        except planner.Error as e:
            out.append((type(e).__name__, str(e)))
    return out


@pytest.mark.parametrize("cfg_name", ["desk8", "tight8"])
@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("mode", MODES)
def test_reference_configs(planner, ref_api, cfg_name, seed, mode):
    cfg = DESK8 if cfg_name == "desk8" else TIGHT8
    lengths = planner.generate_workload("github_like", 256, seed, 196608)
    a, b = both(planner, ref_api, cfg, lengths, None, mode, 4)
    assert a == b


@pytest.mark.parametrize("model", ["tiny", "gpt-1.3b", "gpt-7b", "llama-7b"])
@pytest.mark.parametrize("dp", [1, 2, 4, 8])
def test_b200_configs(planner, ref_api, model, dp):
    m = M.MODELS[model]
    if m.layers % dp:
        pytest.skip("layers not divisible by pp_degree")
    cap = {"tiny": 4096, "gpt-1.3b": 32768, "gpt-7b": 16384, "llama-7b": 65536}[model]
    cfg = M.planner_config(m, dp, mem_capacity=180e9)
    lengths = planner.generate_workload("github_like", 64 * dp, 7 + dp, cap)
    a, b = both(planner, ref_api, cfg, lengths, None, "main", 4)
    assert a == b


@pytest.mark.parametrize("slices", [1, 2, 3, 5, 8, 16])
def test_explicit_slices_and_extremes(planner, ref_api, slices):
    cfg = M.planner_config(M.MODELS["gpt-7b"], 8, mem_capacity=80e9)
    for lengths in ([2048] * 128, [131072] * 8, [131072, 3, 1, 77]):
        a, b = both(planner, ref_api, cfg, lengths, slices, "main", 2)
        assert a == b


def test_random_small_instances(planner, ref_api):
    rng = random.Random(5)
    for i in range(40):
        dp = rng.choice([1, 2, 4])
        cfg = json.loads(json.dumps(WORKED))
        cfg["cluster"]["pp_degree"] = cfg["cluster"]["num_gpus"] = dp
        cfg["model"]["layers"] = 4 * dp
        cfg["model"]["stage_state_bytes"] = [2e9] * dp
        cfg["cluster"]["mem_capacity"] = rng.choice([1e12, 2.02e9, 2.005e9, 2.001e9])
        lengths = [rng.randint(1, 20000) for _ in range(rng.randint(1, 40))]
        slices = rng.choice([None, 1, 2, 3, 4])
        mode = rng.choice(MODES)
        a, b = both(planner, ref_api, cfg, lengths, slices, mode, rng.choice([1, 3]))
        assert a == b, (i, dp, lengths, slices, mode)


def test_errors_match(planner, ref_api):
    bad = json.loads(json.dumps(WORKED))
    bad["cluster"]["num_gpus"] = 7
    assert both(planner, ref_api, bad, [10], None, "main", 1)[0][0] == "ConfigError"
    a, b = both(planner, ref_api, bad, [10], None, "main", 1)
    assert a == b
    a, b = both(planner, ref_api, WORKED, [], None, "main", 1)
    assert a == b and a[0] == "ContractError"
    a, b = both(planner, ref_api, WORKED, [5, 3], 9, "main", 1)
    assert a == b


def test_trace_and_fit_parity(planner, ref_api):
    lengths = planner.generate_workload("github_like", 128, 3, 65536)
    doc = planner.make_plan_document(DESK8, lengths, 3, "main", 2)
    assert planner.simulate_plan_document(doc) == planner.simulate_plan_document(doc, _lib=ref_api)
    samples = []
    rng = random.Random(1)
    for _ in range(12):
        ctx = rng.choice([0, 0, 1000, 5000])
        sl = [rng.randint(100, 8000)]
        for ph in ("forward", "backward"):
            samples.append({"context": ctx, "slices": sl, "phase": ph,
                            "seconds": 1e-3 + 1e-9 * (ctx + sl[0]) ** 2 + 2e-6 * sl[0] * (2 if ph == "backward" else 1)})
    assert planner.fit_cost_params(DESK8, samples) == planner.fit_cost_params(DESK8, samples, _lib=ref_api)


def test_render_contract(planner):
    doc = planner.make_plan_document(WORKED, [9000, 300, 200, 1500, 700], 3, "main", 1)
    trace, _ = planner.simulate_plan_document(doc)
    svg = planner.render_svg(trace)
    events = sum(len(u["events"]) for u in json.loads(trace)["units"])
    assert svg.count('class="bar"') == events
    assert svg.count(">stage ") == 2 * len(json.loads(trace)["units"])
