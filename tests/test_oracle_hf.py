"""Pins the numerics oracle (oracle/numerics.py) against an independent
implementation of the same model families: Hugging Face transformers'
LlamaForCausalLM (RMSNorm, GQA, SwiGLU, rotate-half RoPE) and
GPTNeoXForCausalLM configured as the GPT of BASELINE.json (sequential
residual, LayerNorm, full rotary, tanh-GELU; its linear biases held at 0).
Same weights, same tokens: per-token losses and every parameter gradient
must agree to fp32 round-off.  The reference itself ships no model
(SURVEY.md §0), so this is the oracle's external pin; the CUDA stages are in
turn held to the oracle (tests/test_gpu_stage.py, test_gpu_bench_shapes.py).
"""
import pytest
import torch

from oracle import numerics as O

transformers = pytest.importorskip("transformers")

LAYERS, D, H, HD, V = 2, 64, 4, 16, 128


def _spec(arch):
    if arch == "llama":
        return O.ModelSpec("llama", LAYERS, D, H, 2, HD, 96, V, rope_theta=10000.0, norm_eps=1e-5)
    return O.ModelSpec("gpt", LAYERS, D, H, H, HD, 128, V, rope_theta=10000.0, norm_eps=1e-5)


def _hf_model(spec):
    torch.manual_seed(0)
    if spec.llama:
        cfg = transformers.LlamaConfig(
            vocab_size=V, hidden_size=D, intermediate_size=spec.ffn, num_hidden_layers=LAYERS,
            num_attention_heads=H, num_key_value_heads=spec.kv_heads, head_dim=HD, rms_norm_eps=spec.norm_eps,
            rope_parameters={"rope_theta": spec.rope_theta, "rope_type": "default"}, attention_bias=False,
            mlp_bias=False, tie_word_embeddings=False, max_position_embeddings=4096)
        cfg._attn_implementation = "eager"
        return transformers.LlamaForCausalLM(cfg).float().eval()
    cfg = transformers.GPTNeoXConfig(
        vocab_size=V, hidden_size=D, intermediate_size=spec.ffn, num_hidden_layers=LAYERS, num_attention_heads=H,
        hidden_act="gelu_pytorch_tanh", layer_norm_eps=spec.norm_eps, use_parallel_residual=False,
        rope_parameters={"rope_theta": spec.rope_theta, "partial_rotary_factor": 1.0, "rope_type": "default"},
        attention_bias=True, tie_word_embeddings=False, max_position_embeddings=4096)
    cfg._attn_implementation = "eager"
    return transformers.GPTNeoXForCausalLM(cfg).float().eval()


def _load(spec, model, params):
    """Our parameters -> the HF module (biases zeroed).  Returns a map our
    name -> function(HF grads) giving the matching gradient."""
    sd = {}
    get = {}
    Hkv = spec.kv_heads
    if spec.llama:
        sd["model.embed_tokens.weight"] = params["embed.weight"]
        get["embed.weight"] = lambda g: g["model.embed_tokens.weight"]
        for j in range(LAYERS):
            p, h = f"layers.{j}.", f"model.layers.{j}."
            w = params[p + "attn.wqkv"]
            sd[h + "self_attn.q_proj.weight"] = w[:H * HD]
            sd[h + "self_attn.k_proj.weight"] = w[H * HD:(H + Hkv) * HD]
            sd[h + "self_attn.v_proj.weight"] = w[(H + Hkv) * HD:]
            sd[h + "self_attn.o_proj.weight"] = params[p + "attn.wo"]
            sd[h + "input_layernorm.weight"] = params[p + "norm1.weight"]
            sd[h + "post_attention_layernorm.weight"] = params[p + "norm2.weight"]
            w13 = params[p + "mlp.w13"]
            sd[h + "mlp.gate_proj.weight"] = w13[:spec.ffn]
            sd[h + "mlp.up_proj.weight"] = w13[spec.ffn:]
            sd[h + "mlp.down_proj.weight"] = params[p + "mlp.w2"]
            get[p + "attn.wqkv"] = (lambda h: lambda g: torch.cat(
                [g[h + "self_attn.q_proj.weight"], g[h + "self_attn.k_proj.weight"],
                 g[h + "self_attn.v_proj.weight"]]))(h)
            get[p + "attn.wo"] = (lambda h: lambda g: g[h + "self_attn.o_proj.weight"])(h)
            get[p + "norm1.weight"] = (lambda h: lambda g: g[h + "input_layernorm.weight"])(h)
            get[p + "norm2.weight"] = (lambda h: lambda g: g[h + "post_attention_layernorm.weight"])(h)
            get[p + "mlp.w13"] = (lambda h: lambda g: torch.cat(
                [g[h + "mlp.gate_proj.weight"], g[h + "mlp.up_proj.weight"]]))(h)
            get[p + "mlp.w2"] = (lambda h: lambda g: g[h + "mlp.down_proj.weight"])(h)
        sd["model.norm.weight"] = params["final_norm.weight"]
        sd["lm_head.weight"] = params["lm_head.weight"]
        get["final_norm.weight"] = lambda g: g["model.norm.weight"]
        get["lm_head.weight"] = lambda g: g["lm_head.weight"]
    else:
        sd["gpt_neox.embed_in.weight"] = params["embed.weight"]
        get["embed.weight"] = lambda g: g["gpt_neox.embed_in.weight"]
        for j in range(LAYERS):
            p, h = f"layers.{j}.", f"gpt_neox.layers.{j}."
            w = params[p + "attn.wqkv"]
            # NeoX fuses q/k/v per head: rows [h][q|k|v][hd]
            q, k, v = (w[i * H * HD:(i + 1) * H * HD].view(H, HD, D) for i in range(3))
            sd[h + "attention.query_key_value.weight"] = torch.stack([q, k, v], 1).reshape(3 * H * HD, D)
            sd[h + "attention.query_key_value.bias"] = torch.zeros(3 * H * HD)
            sd[h + "attention.dense.weight"] = params[p + "attn.wo"]
            sd[h + "attention.dense.bias"] = torch.zeros(D)
            sd[h + "input_layernorm.weight"] = params[p + "norm1.weight"]
            sd[h + "input_layernorm.bias"] = params[p + "norm1.bias"]
            sd[h + "post_attention_layernorm.weight"] = params[p + "norm2.weight"]
            sd[h + "post_attention_layernorm.bias"] = params[p + "norm2.bias"]
            sd[h + "mlp.dense_h_to_4h.weight"] = params[p + "mlp.w1"]
            sd[h + "mlp.dense_h_to_4h.bias"] = torch.zeros(spec.ffn)
            sd[h + "mlp.dense_4h_to_h.weight"] = params[p + "mlp.w2"]
            sd[h + "mlp.dense_4h_to_h.bias"] = torch.zeros(D)

            def qkv_grad(g, h=h):
                t = g[h + "attention.query_key_value.weight"].view(H, 3, HD, D)
                return torch.cat([t[:, i].reshape(H * HD, D) for i in range(3)])
            get[p + "attn.wqkv"] = qkv_grad
            for ours, theirs in (("attn.wo", "attention.dense.weight"), ("norm1.weight", "input_layernorm.weight"),
                                 ("norm1.bias", "input_layernorm.bias"),
                                 ("norm2.weight", "post_attention_layernorm.weight"),
                                 ("norm2.bias", "post_attention_layernorm.bias"),
                                 ("mlp.w1", "mlp.dense_h_to_4h.weight"), ("mlp.w2", "mlp.dense_4h_to_h.weight")):
                get[p + ours] = (lambda key: lambda g: g[key])(h + theirs)
        sd["gpt_neox.final_layer_norm.weight"] = params["final_norm.weight"]
        sd["gpt_neox.final_layer_norm.bias"] = params["final_norm.bias"]
        sd["embed_out.weight"] = params["lm_head.weight"]
        get["final_norm.weight"] = lambda g: g["gpt_neox.final_layer_norm.weight"]
        get["final_norm.bias"] = lambda g: g["gpt_neox.final_layer_norm.bias"]
        get["lm_head.weight"] = lambda g: g["embed_out.weight"]
    missing, unexpected = model.load_state_dict({k: v.float().contiguous() for k, v in sd.items()}, strict=False)
    assert not unexpected, unexpected
    assert all("rotary" in k or "inv_freq" in k for k in missing), missing
    return get


@pytest.mark.parametrize("arch", ["gpt", "llama"])
def test_oracle_matches_transformers(arch):
    spec = _spec(arch)
    params = O.init_params(spec, seed=11)
    model = _hf_model(spec)
    get = _load(spec, model, params)
    g = torch.Generator().manual_seed(5)
    seqs = [torch.randint(0, V, (n,), generator=g) for n in (97, 33, 160)]
    n_targets = sum(len(s) - 1 for s in seqs)
    # HF: per-sequence forward (each attended causally on its own), summed CE / n_targets
    total = 0.0
    for s in seqs:
        logits = model(input_ids=s[None]).logits[0].float()
        hf_tok = torch.nn.functional.cross_entropy(logits[:-1], s[1:], reduction="none")
        ours_tok = O.sequence_token_losses(spec, params, s)[:-1]
        assert torch.allclose(hf_tok, ours_tok, rtol=1e-5, atol=1e-5), float((hf_tok - ours_tok).abs().max())
        (hf_tok.sum() / n_targets).backward()
        total += float(hf_tok.detach().double().sum())
    loss, grads, _ = O.whole_batch_grads(spec, params, seqs)
    assert abs(float(loss) - total / n_targets) < 1e-6 * abs(total / n_targets)
    hf = {k: p.grad for k, p in model.named_parameters() if p.grad is not None}
    assert set(get) == set(grads), set(grads) ^ set(get)
    for name, ours in grads.items():
        theirs = get[name](hf)
        rel = float((ours - theirs).norm() / theirs.norm().clamp_min(1e-30))
        assert rel < 1e-4, (name, rel)
