"""Parity at the benchmark's shapes: the kernel variants bench.py runs,
checked against the fp32 oracle (oracle/numerics.py) evaluated on the GPU in
fp32 with TF32 off.

Two transformer layers at GPT-1.3B width (D 2048, 16 heads of 128, FFN 8192,
V 50304), at Llama-7B width (D 4096, GQA 32/8, SwiGLU 11008, V 32000) and at
GPT-7B width (D 4096, 32 heads, FFN 16384, V 50304; bf16 only),
on a planned batch with one 20K-token sequence split into 4 slices (the last
one, a Hybrid chunk, at 16.8-17.1K context followed by packed documents) and
a Batched chunk of short documents.  Chunks hold 3.9-8.2K tokens, so every
GEMM takes the CTA-pair kernel (QKV + RoPE scatter, GELU up-projection, GELU'
W2 dgrad, residual adds, fp32 weight-gradient accumulation), every norm runs
the CTA-per-row kernels (D >= 1024) and attention runs the tcgen05 kernels on
context up to 20K; tests assert from epp_gpu_kernel_stats that they did.

Tolerances:
  * fp32 mode (SIMT kernels): loss and every gradient rel <= 1e-3
    (north_star), per-chunk loss rel <= 1e-5;
  * bf16 mode (tcgen05, fp32 accumulate): each parameter's gradient error
    against the fp32 oracle is held to two yardsticks computed from the SAME
    oracle, so the tolerance is the model's bf16 floor, not a free constant:
      - <= 2x the error of the oracle run under torch.autocast(bfloat16)
        (+ 1e-3 absolute).  Measured (tools/bf16_error_table.py ->
        profiles/r02_bf16_error_table_*.json): GPT-1.3B width 1.05-1.70x,
        Llama-7B width 0.70-0.77x.  The GPT excess is the residual stream:
        the executor stores it (and its gradient) in bf16 between layers, as
        bf16 training frameworks do, while autocast keeps it in fp32;
      - <= the error of the oracle with all parameters and activations in
        bf16 (model.bfloat16()): measured 0.55-0.77x;
    loss rel <= 2e-3 and per-chunk loss rel <= 2e-3.
"""
import math

import pytest
import torch

from oracle import numerics as O
from paper_2509_21275_b200 import model as M
from paper_2509_21275_b200 import schedule as S
from paper_2509_21275_b200.executor import LocalPipeline, stage_layers

pytestmark = pytest.mark.gpu

WIDTHS = {
    "gpt-1.3b": M.ModelConfig("gpt-1.3b-w", "gpt", layers=2, hidden=2048, heads=16, kv_heads=16, ffn=8192,
                              vocab=50304),
    "llama-7b": M.ModelConfig("llama-7b-w", "llama", layers=2, hidden=4096, heads=32, kv_heads=8, ffn=11008,
                              vocab=32000),
    # the headline benchmark's model (bench.py default): LayerNorm / GELU at
    # D 4096, 32 MHA heads, FFN 16384
    "gpt-7b": M.ModelConfig("gpt-7b-w", "gpt", layers=2, hidden=4096, heads=32, kv_heads=32, ffn=16384,
                            vocab=50304),
}
LENGTHS = [20480, 2300, 1500, 900, 610, 300, 129, 77]
SLICES = 4


def spec_of(m):
    return O.ModelSpec(m.arch, m.layers, m.hidden, m.heads, m.kv_heads, m.head_dim, m.ffn, m.vocab,
                       m.rope_theta, m.norm_eps)


def make_plan(planner, m, dp, tight):
    cfg = M.planner_config(m, dp, mem_capacity=1e12, reserve_bytes=0)
    if not tight:
        return S.parse_plan(planner.make_plan_document(cfg, LENGTHS, SLICES, "main", 1), LENGTHS)
    act = cfg["model"]["token_act_bytes"]
    for tokens_fit in (24000, 20000, 16000, 14000, 12000, 10000, 9000):
        cfg["cluster"]["mem_capacity"] = max(cfg["model"]["stage_state_bytes"]) + act * tokens_fit / dp
        try:
            plan = S.parse_plan(planner.make_plan_document(cfg, LENGTHS, SLICES, "main", 1), LENGTHS)
        except planner.InfeasibleError:
            break
        if any(any(v for row in u.ckpt for v in row) for u in plan.units):
            return plan
    raise AssertionError("no memory budget activates the ladder")


_ORACLE = {}


def oracle(arch, autocast=False, pure_bf16=False):
    """(loss, grads, per-sequence token losses) of the whole batch, on the
    GPU: fp32 (TF32 off), under bf16 autocast, or with bf16 parameters and
    activations throughout; cached per arch."""
    key = (arch, autocast, pure_bf16)
    if key not in _ORACLE:
        m = WIDTHS[arch]
        torch.backends.cuda.matmul.allow_tf32 = False
        torch.backends.cudnn.allow_tf32 = False
        params = {k: v.cuda() for k, v in O.init_params(spec_of(m), seed=11).items()}
        if pure_bf16:
            params = {k: v.bfloat16() for k, v in params.items()}
        tokens = S.synthetic_tokens(LENGTHS, m.vocab, seed=5)
        loss, grads, per_seq = O.whole_batch_grads(spec_of(m), params,
                                                   [torch.from_numpy(t).long().cuda() for t in tokens],
                                                   autocast_bf16=autocast)
        _ORACLE[key] = (loss.item(), {k: g.float() for k, g in grads.items()}, [x.double() for x in per_seq])
        del params
        torch.cuda.empty_cache()
    return _ORACLE[key]


def run_cuda(m, plan, dtype):
    from paper_2509_21275_b200.gpu import CudaStage
    params = O.init_params(spec_of(m), seed=11)
    tokens = S.synthetic_tokens(LENGTHS, m.vocab, seed=5)
    dp = plan.pp_degree
    stages = []
    for p in range(dp):
        first, num = stage_layers(m.layers, dp, p)
        st = CudaStage(m, first, num, p == 0, p == dp - 1, dtype=dtype)
        st.load_weights(params)
        stages.append(st)
    LocalPipeline(stages, torch.device("cuda")).run_step(plan, tokens)
    torch.cuda.synchronize()
    grads = {}
    for st in stages:
        grads.update({k: v.view(params[k].shape) for k, v in st.grads().items()})
    loss_sum, cnt = stages[-1].loss()
    chunk = {cid: stages[-1].chunk_loss(cid) for cid in plan.chunks}
    for st in stages:
        assert st.memory()[0] == 0, "chunk / sequence buffers leaked"
        st.close()
    return loss_sum, cnt, grads, chunk


def oracle_chunk_losses(plan, per_seq):
    """Per-micro-batch (sum of token losses, #targets) from the whole-sequence
    per-token losses and the chunk's member layout (tail first, then shorts)."""
    out = {}
    for cid, lay in plan.chunks.items():
        s_sum, n_t = 0.0, 0
        for (seq, start, n) in lay.members:
            s_sum += float(per_seq[seq][start:start + n].sum())
            n_t += max(0, min(n, LENGTHS[seq] - start - 1))
        out[cid] = (s_sum, n_t)
    return out


def rel(a, b):
    return float((a.float() - b.float()).norm() / (b.float().norm() + 1e-30))


def assert_bench_variants(arch, dtype):
    """The benchmark's kernel variants really ran (demangled template args:
    gemm_tc2_kernel<BN, STAGES, A_MN, B_MN, EPI>, EPI 6 RopeScatter,
    4 StoreGelu, 5 GeluBwd, 7 SwiGlu, 8 SwiGluBwd, 2 AddRes, 1 AccumF32)."""
    from paper_2509_21275_b200.gpu import kernel_stats
    ks = kernel_stats()
    names = " ".join(k for k, v in ks.items() if v > 0)
    if dtype == "f32":
        assert "gemm_simt_kernel" in names and "attn_fwd_f32" in names
        return
    pair = [k for k in ks if "gemm_tc2_kernel<" in k and ks[k] > 0]
    epis = {k.split("gemm_tc2_kernel<")[1].split(">")[0].split(",")[-1].strip() for k in pair}
    want = {"6", "2", "1"} | ({"4", "5"} if WIDTHS[arch].arch == "gpt" else {"7", "8"})
    assert want <= epis, (sorted(epis), pair)
    assert "norm_fwd_row_k" in names and "norm_bwd_dx_row_k" in names, names
    for k in ("attn_fwd_tc", "attn_bwd_dq_tc", "attn_bwd_dkv_tc"):
        assert k in names, (k, names)


@pytest.mark.parametrize("arch,dp,tight", [("gpt-1.3b", 1, False), ("gpt-1.3b", 2, True), ("llama-7b", 2, False),
                                           ("gpt-7b", 1, False)])
def test_bf16_at_bench_width(planner, arch, dp, tight):
    m = WIDTHS[arch]
    plan = make_plan(planner, m, dp, tight)
    assert max(c.context for c in plan.chunks.values()) >= 16384
    if tight:
        assert any(any(v for row in u.ckpt for v in row) for u in plan.units), "ladder inactive"
    loss_sum, cnt, grads, chunk = run_cuda(m, plan, "bf16")
    assert_bench_variants(arch, "bf16")
    ref_loss, ref_grads, per_seq = oracle(arch)
    _, ac_grads, _ = oracle(arch, autocast=True)
    _, pb_grads, _ = oracle(arch, pure_bf16=True)
    assert cnt == plan.total_targets
    assert math.log(m.vocab) * 0.9 < loss_sum / cnt < math.log(m.vocab) * 1.1
    assert abs(loss_sum / cnt - ref_loss) / ref_loss < 2e-3
    ref_chunk = oracle_chunk_losses(plan, per_seq)
    for cid, (s_ref, n_ref) in ref_chunk.items():
        s, n = chunk[cid]
        assert n == n_ref, (cid, n, n_ref)
        assert abs(s - s_ref) <= 2e-3 * abs(s_ref), (cid, s, s_ref)
    worst = []
    for name, g in ref_grads.items():
        ours = rel(grads[name], g)
        yard = rel(ac_grads[name], g)
        pure = rel(pb_grads[name], g)
        worst.append((ours / max(yard, 1e-12), name, ours, yard, pure))
        assert ours <= 2.0 * yard + 1e-3, (name, ours, yard)
        assert ours <= pure, (name, ours, pure)
    worst.sort(reverse=True)
    print(f"{arch} dp={dp} tight={tight}: worst ours/autocast ratio {worst[0]}")


@pytest.mark.parametrize("arch", ["gpt-1.3b", "llama-7b"])
def test_f32_at_bench_width(planner, arch):
    m = WIDTHS[arch]
    plan = make_plan(planner, m, 1, False)
    loss_sum, cnt, grads, chunk = run_cuda(m, plan, "f32")
    assert_bench_variants(arch, "f32")
    ref_loss, ref_grads, per_seq = oracle(arch)
    assert abs(loss_sum / cnt - ref_loss) / ref_loss < 1e-5
    for cid, (s_ref, n_ref) in oracle_chunk_losses(plan, per_seq).items():
        s, n = chunk[cid]
        assert n == n_ref and abs(s - s_ref) <= 1e-5 * abs(s_ref), (cid, s, s_ref)
    for name, g in ref_grads.items():
        assert rel(grads[name], g) < 1e-3, (name, rel(grads[name], g))


@pytest.mark.parametrize("arch,dp", [("gpt-1.3b", 2), ("llama-7b", 1)])
def test_deferred_wgrad_bit_identical(planner, monkeypatch, arch, dp):
    """Weight gradients launched with a deferred dependency wait
    (GemmArgs::defer_wait: they overlap the preceding independent data
    gradient) give the same bits as the fully ordered stream (the stage reads
    EPP_DEFER_WGRAD when it is created)."""
    m = WIDTHS[arch]
    plan = make_plan(planner, m, dp, False)
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("EPP_DEFER_WGRAD", flag)
        out[flag] = run_cuda(m, plan, "bf16")
    (l0, c0, g0, k0), (l1, c1, g1, k1) = out["0"], out["1"]
    assert (l0, c0) == (l1, c1)
    assert k0 == k1
    for name, g in g0.items():
        if name == "embed.weight":
            # the embedding backward scatters rows with float atomics
            # (repeated token ids add in arrival order): run-to-run
            # round-off, independent of the deferral
            assert rel(g1[name], g) < 1e-6, name
            continue
        assert torch.equal(g, g1[name]), name
