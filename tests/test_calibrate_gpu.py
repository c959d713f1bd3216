"""Closed-loop cost model on the GPU executor: per-op stage times of one
planned step fitted to Eq. 1 (fit_cost_params) predict the measured step
time, and the fitted configuration still plans the batch."""
import pytest
import torch

from paper_2509_21275_b200 import calibrate, model as M, planner, schedule
from paper_2509_21275_b200.executor import LocalPipeline

pytestmark = pytest.mark.gpu


def test_fit_predicts_step_time():
    from paper_2509_21275_b200.gpu import CudaStage
    m = M.ModelConfig("c", "gpt", layers=4, hidden=512, heads=4, kv_heads=4, ffn=2048, vocab=4096)
    lengths = planner.generate_workload("github_like", 48, 3, 8192)
    cfg = M.planner_config(m, 1, mem_capacity=1e12, reserve_bytes=0, cost=M.default_cost(m))
    plan = schedule.parse_plan(planner.make_plan_document(cfg, lengths, 4, "main", 1), lengths)
    tokens = schedule.synthetic_tokens(lengths, m.vocab, seed=1)
    st = CudaStage(m, 0, m.layers, True, True, dtype="bf16")
    st.init_weights(1)
    LocalPipeline([st], torch.device("cuda")).run_step(plan, tokens)        # warm
    timed = calibrate.TimedStage(st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    LocalPipeline([timed], torch.device("cuda")).run_step(plan, tokens)
    e1.record()
    torch.cuda.synchronize()
    measured = e0.elapsed_time(e1) / 1e3
    samples = timed.samples()
    assert len([s for s in samples if s["phase"] == "forward"]) >= 4
    fitted = calibrate.planner_config_only(calibrate.calibrated_config(cfg, samples))
    assert all(v >= 0 for k, v in fitted["cost"].items() if k != "layer_fwd_seconds")
    doc = planner.make_plan_document(fitted, lengths, 4, "main", 1)
    predicted = calibrate.predicted_seconds(doc)
    assert 0.7 < measured / predicted < 1.4, (measured, predicted)
