"""ORACLE / TEST INFRASTRUCTURE ONLY — fp32 CPU numerics of the EPP model path.

Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
leg import this module, as the checker.  The product (paper_2509_21275_b200)
never does.

The reference ships no model execution ("no model, no loss and
no gradients"), so this is a from-scratch restatement with no reference
golden vectors.  What pins it:
  * an independent implementation of the same model families:
    tests/test_oracle_hf.py loads the same weights into Hugging Face
    transformers 5.5.0 LlamaForCausalLM (RMSNorm, GQA, SwiGLU, rotate-half
    RoPE) and GPTNeoXForCausalLM (sequential residual, LayerNorm, full
    rotary, tanh-GELU, zero biases) and requires identical per-token losses
    (max |diff| ~5e-7) and parameter gradients (rel < 1e-4);
  * the chunk semantics are the reference's: slices[0] owns `context`
    (proj/include/epp/chunk.hpp:29-31), Hybrid = tail slice + whole shorts
    (proj/src/processor.cpp:280-299), member order = chunk slice order, a
    non-tail slice's backward follows the next slice's (pipeline.cpp:121-131),
    and attention is causal over the sequence's earlier tokens
    (PAPER.md:180-181);
  * the property test tests/test_oracle.py checks that chunked execution
    through `TorchStage` (any plan, any stage split) reproduces whole-sequence
    autograd loss and gradients to fp32 round-off.

Device-agnostic: the same code runs on CPU (small cases) or, for the
benchmark-width parity tests, on the GPU in fp32 with TF32 off
(tests/test_gpu_bench_shapes.py); attention over long sequences is evaluated
in checkpointed query blocks so its memory stays bounded.

Model (both archs, pre-norm, RoPE rotate-half, no linear biases):
  GPT   : LayerNorm(w,b), MHA, GELU(tanh) MLP ffn
  Llama : RMSNorm(w), GQA, SwiGLU MLP (w13 = [gate; up])
Parameter names/shapes match the CUDA stage (csrc/gpu/stage.cu).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch
import torch.nn.functional as F


@dataclass(frozen=True)
class ModelSpec:
    arch: str            # "gpt" | "llama"
    layers: int
    hidden: int
    heads: int
    kv_heads: int
    head_dim: int
    ffn: int
    vocab: int
    rope_theta: float = 10000.0
    norm_eps: float = 1e-5

    @property
    def llama(self) -> bool:
        return self.arch == "llama"


def param_shapes(spec: ModelSpec, first: int, num: int, has_embed: bool, has_head: bool):
    """(name, shape, kind) in the CUDA stage's parameter order; kind in
    {'w', 'w_out', 'one', 'zero'} drives the init."""
    D, hd = spec.hidden, spec.head_dim
    nq = (spec.heads + 2 * spec.kv_heads) * hd
    f1 = 2 * spec.ffn if spec.llama else spec.ffn
    out = []
    if has_embed:
        out.append(("embed.weight", (spec.vocab, D), "w"))
    for j in range(first, first + num):
        pre = f"layers.{j}."
        out.append((pre + "norm1.weight", (D,), "one"))
        if not spec.llama:
            out.append((pre + "norm1.bias", (D,), "zero"))
        out.append((pre + "attn.wqkv", (nq, D), "w"))
        out.append((pre + "attn.wo", (D, spec.heads * hd), "w_out"))
        out.append((pre + "norm2.weight", (D,), "one"))
        if not spec.llama:
            out.append((pre + "norm2.bias", (D,), "zero"))
        out.append((pre + ("mlp.w13" if spec.llama else "mlp.w1"), (f1, D), "w"))
        out.append((pre + "mlp.w2", (D, spec.ffn), "w_out"))
    if has_head:
        out.append(("final_norm.weight", (D,), "one"))
        if not spec.llama:
            out.append(("final_norm.bias", (D,), "zero"))
        out.append(("lm_head.weight", (spec.vocab, D), "w"))
    return out


def init_params(spec: ModelSpec, seed: int, dtype=torch.float32) -> Dict[str, torch.Tensor]:
    """Whole-model parameters.  Norm weights get a small random perturbation
    around 1 (and biases around 0) so their gradients are exercised."""
    g = torch.Generator().manual_seed(seed)
    out = {}
    for name, shape, kind in param_shapes(spec, 0, spec.layers, True, True):
        if kind == "w":
            t = torch.randn(shape, generator=g, dtype=torch.float64) * 0.02
        elif kind == "w_out":
            t = torch.randn(shape, generator=g, dtype=torch.float64) * (0.02 / math.sqrt(2 * spec.layers))
        elif kind == "one":
            t = 1.0 + 0.1 * torch.randn(shape, generator=g, dtype=torch.float64)
        else:
            t = 0.1 * torch.randn(shape, generator=g, dtype=torch.float64)
        out[name] = t.to(dtype)
    return out


_ROPE_CACHE: Dict[tuple, tuple] = {}


def rope_cos_sin(max_pos: int, hd: int, theta: float):
    """cos/sin [max_pos, hd/2], computed in float64 then rounded to fp32 —
    the same table the CUDA kernels use (elementwise.cu rope_table_k)."""
    key = (max_pos, hd, theta)
    if key not in _ROPE_CACHE:
        half = hd // 2
        j = np.arange(half, dtype=np.float64)
        inv = np.power(theta, -2.0 * j / hd)
        ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
        _ROPE_CACHE[key] = (torch.from_numpy(np.cos(ang).astype(np.float32)),
                            torch.from_numpy(np.sin(ang).astype(np.float32)))
    return _ROPE_CACHE[key]


def apply_rope(x: torch.Tensor, pos: torch.Tensor, theta: float) -> torch.Tensor:
    """x [T, nh, hd]; rotate-half RoPE at integer positions pos [T]."""
    hd = x.shape[-1]
    half = hd // 2
    cos, sin = rope_cos_sin(int(pos.max().item()) + 1, hd, theta)
    pc = pos.cpu()
    c = cos[pc].to(x.device, x.dtype)[:, None, :]
    s = sin[pc].to(x.device, x.dtype)[:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)


def norm(x, w, b, eps, rms):
    if rms:
        return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + eps) * w
    mu = x.mean(-1, keepdim=True)
    var = ((x - mu) ** 2).mean(-1, keepdim=True)
    return (x - mu) * torch.rsqrt(var + eps) * w + b


def gelu_tanh(x):
    return F.gelu(x, approximate="tanh")


def _attend_dense(q, k, v, qpos):
    T, H, hd = q.shape
    S, Hkv, _ = k.shape
    g = H // Hkv
    kk = k.repeat_interleave(g, dim=1)
    vv = v.repeat_interleave(g, dim=1)
    s = torch.einsum("thd,shd->hts", q, kk) / math.sqrt(hd)
    mask = torch.arange(S, device=q.device)[None, :] > qpos.to(q.device)[:, None]
    s = s.masked_fill(mask[None], float("-inf"))
    p = torch.softmax(s, dim=-1)
    return torch.einsum("hts,shd->thd", p, vv)


# score elements per dense evaluation; larger problems go through
# checkpointed query blocks (the backward recomputes each block's scores)
_ATTN_DENSE_LIMIT = 1 << 28


def attend(q, k, v, qpos):
    """q [T,H,hd], k/v [S,Hkv,hd]; query i sees keys j <= qpos[i]."""
    T, H, _ = q.shape
    S = k.shape[0]
    if T * S * H <= _ATTN_DENSE_LIMIT:
        return _attend_dense(q, k, v, qpos)
    from torch.utils.checkpoint import checkpoint
    block = max(64, _ATTN_DENSE_LIMIT // (S * H))
    outs = []
    for i in range(0, T, block):
        qp = qpos[i:i + block]
        kv = int(qp.max().item()) + 1          # keys past the block's last query are masked anyway
        outs.append(checkpoint(_attend_dense, q[i:i + block], k[:kv], v[:kv], qp, use_reentrant=False))
    return torch.cat(outs)


def _p(params, name):
    return params[name]


def mlp(spec, params, pre, x):
    h = norm(x, params[pre + "norm2.weight"], params.get(pre + "norm2.bias"), spec.norm_eps, spec.llama)
    if spec.llama:
        u = h @ params[pre + "mlp.w13"].T
        gate, up = u[:, : spec.ffn], u[:, spec.ffn:]
        a = F.silu(gate) * up
    else:
        a = gelu_tanh(h @ params[pre + "mlp.w1"].T)
    return a @ params[pre + "mlp.w2"].T


def qkv_proj(spec, params, pre, x, pos):
    H, Hkv, hd = spec.heads, spec.kv_heads, spec.head_dim
    h = norm(x, params[pre + "norm1.weight"], params.get(pre + "norm1.bias"), spec.norm_eps, spec.llama)
    qkv = h @ params[pre + "attn.wqkv"].T
    q = qkv[:, : H * hd].reshape(-1, H, hd)
    k = qkv[:, H * hd:(H + Hkv) * hd].reshape(-1, Hkv, hd)
    v = qkv[:, (H + Hkv) * hd:].reshape(-1, Hkv, hd)
    return apply_rope(q, pos, spec.rope_theta), apply_rope(k, pos, spec.rope_theta), v


def head_logits(spec, params, x):
    h = norm(x, params["final_norm.weight"], params.get("final_norm.bias"), spec.norm_eps, spec.llama)
    return h @ params["lm_head.weight"].T


# ---------------------------------------------------------------- whole ---
def sequence_token_losses(spec: ModelSpec, params, tokens: torch.Tensor) -> torch.Tensor:
    """Per-position CE of one whole sequence (next-token targets); the last
    position has no target and gets 0."""
    T = tokens.shape[0]
    dev = params["embed.weight"].device
    tokens = tokens.to(dev)
    pos = torch.arange(T, device=dev)
    x = params["embed.weight"][tokens]
    for j in range(spec.layers):
        pre = f"layers.{j}."
        q, k, v = qkv_proj(spec, params, pre, x, pos)
        o = attend(q, k, v, pos).reshape(T, -1)
        x = x + o @ params[pre + "attn.wo"].T
        x = x + mlp(spec, params, pre, x)
    logits = head_logits(spec, params, x)
    logits = logits.float()
    losses = torch.zeros(T, dtype=logits.dtype, device=dev)
    if T > 1:
        losses = torch.cat([F.cross_entropy(logits[:-1], tokens[1:], reduction="none"),
                            torch.zeros(1, dtype=logits.dtype, device=dev)])
    return losses


def whole_batch_grads(spec: ModelSpec, params: Dict[str, torch.Tensor], sequences: Sequence[torch.Tensor],
                      autocast_bf16: bool = False):
    """Reference loss/grads: mean next-token CE over every target of every
    sequence, each sequence attended independently and causally.  The
    parameters' device decides where it runs.  autocast_bf16 (CUDA): the same
    model under torch.autocast(bfloat16) — the error yardstick the bf16
    executor is held to (tests/test_gpu_bench_shapes.py).  Each sequence is
    back-propagated on its own (bounded memory); gradients accumulate."""
    leaf = {k: v.detach().clone().requires_grad_(True) for k, v in params.items()}
    n_targets = sum(max(0, s.shape[0] - 1) for s in sequences)
    total = 0.0
    per_seq = []
    dev = next(iter(leaf.values())).device
    for s in sequences:
        with torch.autocast(dev.type, dtype=torch.bfloat16, enabled=autocast_bf16):
            l = sequence_token_losses(spec, leaf, s)
        per_seq.append(l.detach())
        (l.sum() / n_targets).backward()
        total += float(l.detach().double().sum())
    loss = torch.tensor(total / n_targets, dtype=torch.float64)
    return loss, {k: v.grad.detach() for k, v in leaf.items()}, per_seq


# --------------------------------------------------------------- chunked ---
@dataclass
class ChunkIO:
    """Executor-side chunk description (mirrors epp_chunk_desc)."""
    id: int
    seq: int                  # -1 for Batched
    kind: int
    tail: bool
    context: int
    seq_len: int
    slices: List[int]
    ckpt_layers: int
    loss_scale: float
    token_ids: torch.Tensor   # [T] int
    target_ids: torch.Tensor  # [T] int, -1 = none


class TorchStage:
    """A pipeline stage executing chunks with the executor's semantics, in
    fp32 torch on CPU.  K/V of a sequence's earlier slices are autograd LEAVES
    here; their .grad accumulates the later slices' contributions exactly like
    the CUDA stage's fp32 dK/dV buffers, and is fed back when the owning chunk
    runs its backward."""

    def __init__(self, spec: ModelSpec, params: Dict[str, torch.Tensor], first: int, num: int,
                 has_embed: bool, has_head: bool):
        self.spec, self.first, self.num = spec, first, num
        self.has_embed, self.has_head = has_embed, has_head
        names = [n for n, _, _ in param_shapes(spec, first, num, has_embed, has_head)]
        self.params = {n: params[n].detach().clone().requires_grad_(True) for n in names}
        self.inflight = {}
        self.kv_leaves: Dict[int, Dict[int, list]] = {}   # seq -> layer -> [(k_leaf, v_leaf, k_graph, v_graph)]
        self.loss_sum = 0.0
        self.loss_count = 0
        self.chunk_losses = {}

    def grads(self):
        return {n: (p.grad.detach().clone() if p.grad is not None else torch.zeros_like(p))
                for n, p in self.params.items()}

    def grad_views(self):
        for p in self.params.values():
            if p.grad is None:
                p.grad = torch.zeros_like(p)
        return {n: p.grad for n, p in self.params.items()}

    def forward(self, c: ChunkIO, act_in: Optional[torch.Tensor]):
        spec, P = self.spec, self.params
        T = sum(c.slices)
        if self.has_embed:
            x_in = None
            x = P["embed.weight"][c.token_ids.long()]
        else:
            x_in = act_in.detach().clone().requires_grad_(True)
            x = x_in
        # segments: (start, len, context, is_seq)
        segs, start = [], 0
        for i, s in enumerate(c.slices):
            segs.append((start, s, c.context if (i == 0 and c.seq >= 0) else 0, i == 0 and c.seq >= 0))
            start += s
        own_kv = []   # graph tensors of this chunk's own sequence K/V per layer
        for j in range(self.num):
            lj = self.first + j
            pre = f"layers.{lj}."
            pos = torch.cat([torch.arange(ctx, ctx + n, device=x.device) for (_, n, ctx, _) in segs])
            q, k, v = qkv_proj(spec, P, pre, x, pos)
            outs = []
            for (st, n, ctx, is_seq) in segs:
                qs, ks, vs = q[st:st + n], k[st:st + n], v[st:st + n]
                if is_seq:
                    store = self.kv_leaves.setdefault(c.seq, {}).setdefault(j, [])
                    prior_k = [e[0] for e in store]
                    prior_v = [e[1] for e in store]
                    kk = torch.cat(prior_k + [ks]) if prior_k else ks
                    vv = torch.cat(prior_v + [vs]) if prior_v else vs
                    assert kk.shape[0] == ctx + n, "context does not match stored slices"
                    leaf_k = ks.detach().clone().requires_grad_(True)
                    leaf_v = vs.detach().clone().requires_grad_(True)
                    store.append((leaf_k, leaf_v))
                    own_kv.append((ks, vs, leaf_k, leaf_v))
                else:
                    kk, vv = ks, vs
                outs.append(attend(qs, kk, vv, torch.arange(ctx, ctx + n, device=x.device)))
            o = torch.cat(outs).reshape(T, -1)
            x = x + o @ P[pre + "attn.wo"].T
            x = x + mlp(spec, P, pre, x)
        state = {"x_in": x_in, "own_kv": own_kv}
        if self.has_head:
            logits = head_logits(spec, P, x)
            tgt = c.target_ids.long()
            valid = tgt >= 0
            ce = F.cross_entropy(logits[valid], tgt[valid], reduction="sum") if valid.any() else logits.sum() * 0
            self.loss_sum += float(ce.detach())
            self.loss_count += int(valid.sum())
            self.chunk_losses[c.id] = (float(ce.detach()), int(valid.sum()))
            state["root"] = ce * c.loss_scale
            out = None
        else:
            state["root"] = x
            out = x.detach().clone()
        self.inflight[c.id] = state
        return out

    def backward(self, c: ChunkIO, grad_in: Optional[torch.Tensor]):
        st = self.inflight.pop(c.id)
        roots, grads = [st["root"]], [None if self.has_head else grad_in]
        if self.has_head:
            grads = [torch.ones_like(st["root"])]
        for (ks, vs, leaf_k, leaf_v) in st["own_kv"]:
            for g_t, leaf in ((ks, leaf_k), (vs, leaf_v)):
                if leaf.grad is not None:
                    roots.append(g_t)
                    grads.append(leaf.grad)
        torch.autograd.backward(roots, grads)
        if c.seq >= 0 and c.context == 0:
            self.kv_leaves.pop(c.seq, None)
        if self.has_embed:
            return None
        return st["x_in"].grad.detach()
