"""Pins the numerics oracle (oracle/numerics.py, parity otherwise unpinned):
chunked execution of planner-produced micro-batches through TorchStage, any
stage split, reproduces whole-sequence autograd loss and gradients."""
import numpy as np
import pytest
import torch

from oracle import numerics as O
from paper_2509_21275_b200 import model as M
from paper_2509_21275_b200 import schedule as S
from paper_2509_21275_b200.executor import LocalPipeline, stage_layers

torch.set_default_dtype(torch.float32)


def spec_of(m):
    return O.ModelSpec(m.arch, m.layers, m.hidden, m.heads, m.kv_heads, m.head_dim, m.ffn, m.vocab,
                       m.rope_theta, m.norm_eps)


def small(arch):
    if arch == "gpt":
        return M.ModelConfig("t", "gpt", layers=4, hidden=64, heads=4, kv_heads=4, ffn=128, vocab=256)
    return M.ModelConfig("t", "llama", layers=4, hidden=64, heads=4, kv_heads=2, ffn=96, vocab=256)


def plan_for(planner, m, lengths, dp, slices, mem=None, mode="main"):
    cfg = M.planner_config(m, dp, mem_capacity=mem or 1e12, reserve_bytes=0)
    doc = planner.make_plan_document(cfg, lengths, slices, mode, 1)
    return S.parse_plan(doc, lengths)


def run_chunked(m, params, plan, tokens):
    spec = spec_of(m)
    dp = plan.pp_degree
    stages = []
    for p in range(dp):
        first, num = stage_layers(m.layers, dp, p)
        stages.append(O.TorchStage(spec, params, first, num, p == 0, p == dp - 1))
    LocalPipeline(stages, torch.device("cpu")).run_step(plan, tokens)
    grads = {}
    for st in stages:
        grads.update(st.grads())
    return stages, grads


@pytest.mark.parametrize("arch", ["gpt", "llama"])
@pytest.mark.parametrize("dp,slices", [(1, 3), (2, 3), (2, 2), (4, 4)])
def test_chunked_equals_whole(planner, arch, dp, slices):
    m = small(arch)
    lengths = [300, 37, 21, 90, 5, 64, 180]
    plan = plan_for(planner, m, lengths, dp, slices)
    kinds = {c.kind for c in plan.chunks.values()}
    assert 1 in kinds or 2 in kinds, "expected split/hybrid chunks"
    params = O.init_params(spec_of(m), seed=3)
    tokens = S.synthetic_tokens(lengths, m.vocab, seed=11)
    stages, grads = run_chunked(m, params, plan, tokens)
    loss, ref_grads, per_seq = O.whole_batch_grads(spec_of(m), params,
                                                    [torch.from_numpy(t).long() for t in tokens])
    last = stages[-1]
    assert last.loss_count == plan.total_targets
    assert abs(last.loss_sum / last.loss_count - loss.item()) < 1e-5
    for name, g in ref_grads.items():
        err = (grads[name] - g).norm() / (g.norm() + 1e-30)
        assert err < 1e-4, (name, float(err))
    # per-micro-batch loss = sum of the whole-sequence token losses it holds
    for cid, (lsum, cnt) in last.chunk_losses.items():
        lay = plan.chunks[cid]
        want = 0.0
        for (s, start, n) in lay.members:
            want += float(per_seq[s][start:start + n].sum())
        assert abs(lsum - want) < 1e-3 * max(1.0, abs(want)), cid


def test_checkpointing_plan_is_numerically_transparent(planner):
    """A memory-tight plan (ladder active) computes the same gradients."""
    m = small("gpt")
    lengths = [400, 33, 60, 250, 12]
    cfg_loose = plan_for(planner, m, lengths, 2, 4)
    cfg = M.planner_config(m, 2, mem_capacity=1e12, reserve_bytes=0)
    # squeeze memory until the MILP must checkpoint (largest budget that does)
    act = cfg["model"]["token_act_bytes"]
    plan = None
    for tokens_fit in (600, 500, 450, 400, 350, 300, 250, 200):
        cfg["cluster"]["mem_capacity"] = cfg["model"]["stage_state_bytes"][0] + act * tokens_fit / 2
        try:
            p = S.parse_plan(planner.make_plan_document(cfg, lengths, 4, "main", 1), lengths)
        except planner.InfeasibleError:
            break
        if any(any(v for row in u.ckpt for v in row) for u in p.units):
            plan = p
            break
    assert plan is not None, "ladder inactive at every feasible budget"
    params = O.init_params(spec_of(m), seed=5)
    tokens = S.synthetic_tokens(lengths, m.vocab, seed=2)
    _, g1 = run_chunked(m, params, plan, tokens)
    _, g2 = run_chunked(m, params, cfg_loose, tokens)
    for k in g1:
        assert torch.allclose(g1[k], g2[k], rtol=1e-4, atol=1e-7), k
