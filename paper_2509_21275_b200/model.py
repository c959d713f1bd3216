"""Model shapes of the BASELINE.json configs and the planner memory/cost
model for them on B200.

The planner only sees a model through SystemConfig (proj/include/epp/
config.hpp:30-60): layers, hidden, bytes per token of activations and model
state per stage.  `planner_config()` derives those numbers from what the CUDA
stage executor (csrc/gpu/stage.cu) actually keeps resident, so the MILP's
memory rows describe the real executor.
"""
from __future__ import annotations

from dataclasses import asdict, dataclass
from typing import List, Dict, Optional


@dataclass(frozen=True)
class ModelConfig:
    name: str
    arch: str            # "gpt" | "llama"
    layers: int
    hidden: int
    heads: int
    kv_heads: int
    ffn: int
    vocab: int
    rope_theta: float = 10000.0
    norm_eps: float = 1e-5

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads

    @property
    def llama(self) -> bool:
        return self.arch == "llama"

    def params_per_layer(self) -> int:
        D, hd = self.hidden, self.head_dim
        qkv = (self.heads + 2 * self.kv_heads) * hd * D
        wo = D * self.heads * hd
        mlp = (3 if self.llama else 2) * D * self.ffn
        norms = (2 if self.llama else 4) * D
        return qkv + wo + mlp + norms

    def num_params(self) -> int:
        return self.layers * self.params_per_layer() + 2 * self.vocab * self.hidden + 2 * self.hidden

    def linear_flops_per_token_layer(self) -> float:
        """Forward matmul FLOPs per token per layer (2 x MACs)."""
        D, hd = self.hidden, self.head_dim
        qkv = 2 * D * (self.heads + 2 * self.kv_heads) * hd
        wo = 2 * self.heads * hd * D
        mlp = 2 * D * self.ffn * (3 if self.llama else 2)
        return qkv + wo + mlp

    def attn_flops_per_pair_layer(self) -> float:
        """Forward FLOPs per (query, visible key) pair per layer: QK^T + PV."""
        return 4.0 * self.heads * self.head_dim

    def to_spec_dict(self) -> Dict:
        d = asdict(self)
        d.pop("name")
        d["head_dim"] = self.head_dim
        return d


MODELS: Dict[str, ModelConfig] = {
    # configs[0]: tiny GPT on the CPU reference (BASELINE.json)
    "tiny": ModelConfig("tiny", "gpt", layers=4, hidden=256, heads=4, kv_heads=4, ffn=1024, vocab=4096),
    # configs[1]: GPT-1.3B shape
    "gpt-1.3b": ModelConfig("gpt-1.3b", "gpt", layers=24, hidden=2048, heads=16, kv_heads=16,
                            ffn=8192, vocab=50304),
    # configs[2]: GPT-7B shape
    "gpt-7b": ModelConfig("gpt-7b", "gpt", layers=32, hidden=4096, heads=32, kv_heads=32,
                          ffn=16384, vocab=50304),
    # configs[3]: Llama-style 7B (GQA, RMSNorm, SwiGLU)
    "llama-7b": ModelConfig("llama-7b", "llama", layers=32, hidden=4096, heads=32, kv_heads=8,
                            ffn=11008, vocab=32000),
    # small test shapes for the GPU parity suite
    "tiny-llama": ModelConfig("tiny-llama", "llama", layers=4, hidden=256, heads=4, kv_heads=2,
                              ffn=512, vocab=4096),
    "small-gpt": ModelConfig("small-gpt", "gpt", layers=4, hidden=512, heads=4, kv_heads=4,
                             ffn=2048, vocab=8192),
}


# Planner memory capacity of one B200 stage, used by both benchmark arms so
# they plan identical documents: the device's HBM as cudaMemGetInfo reports
# it on this pool's B200s (191,502,876,672 bytes), rounded down to 191.0e9.
# SURVEY §8d's 180e9 (the marketing "180 GB") left 11.5 GB of every GPU
# unplanned, which at GPT-7B / 16K on one GPU made the checkpoint MILP re-run
# ~51 layer forwards per step.
# Workspaces, allocator slack and the CUDA context stay covered by the 12 GB
# reserve in stage_state_bytes; bench.py checks the device is at least this big.
B200_MEM_CAPACITY = 191.0e9


def activation_bytes_per_token(m: ModelConfig, elem_bytes: int = 2) -> float:
    """Bytes the CUDA stage keeps per token per NON-checkpointed layer until
    the chunk's backward (stage.cu LayerSaved + chunk-local K/V): layer output
    x (D), q (H*hd), o (H*hd), x_mid (D), h (F or 2F), K and V (2*Hkv*hd),
    plus fp32 norm stats and LSE.  The MLP activation act(h) is transient (the
    backward re-creates it from h for the W2 weight gradient)."""
    D, hd = m.hidden, m.head_dim
    f1 = 2 * m.ffn if m.llama else m.ffn
    elems = D + m.heads * hd + m.heads * hd + D + f1 + 2 * m.kv_heads * hd
    return elems * elem_bytes + 4 * 4 + 4 * m.heads


def head_layer_equivalents(m: "ModelConfig", pairs_per_token: float = 2048.0) -> float:
    """LM head + cross-entropy work of the last stage in units of one
    transformer layer's (matmul FLOPs, attention at `pairs_per_token` visible
    keys per query)."""
    head = 2.0 * m.hidden * m.vocab
    layer = m.linear_flops_per_token_layer() + m.attn_flops_per_pair_layer() * pairs_per_token
    return head / layer


def state_bytes_per_param(dtype: str = "bf16") -> float:
    """fp32 master + fp32 grad + fp32 Adam m, v (+ bf16 working copy)."""
    return 16.0 + (2.0 if dtype == "bf16" else 0.0)


def tail_ckpt_excess_bytes(m: ModelConfig) -> float:
    """Bytes per token per checkpointed layer that a TAIL chunk keeps beyond
    Eq. 10's (3 - 2I) e D l charge (I = 1, e = 4: 4D): the layer input (2D,
    bf16), its K/V rows (4 Hkv hd, bf16, in the sequence / chunk KV buffers
    that recompute rewrites) and 16 B of norm statistics.  Positive for MHA
    models (GPT: 2D + 16), 0 for GQA 4:1 (Llama: 3D + 16 < 4D)."""
    kept = 2 * m.hidden + 4 * m.kv_heads * m.head_dim + 16
    return max(0.0, float(kept - 4 * m.hidden))


def planner_config(m: ModelConfig, pp_degree: int, mem_capacity: float = B200_MEM_CAPACITY,
                   cost: Optional[Dict[str, float]] = None, reserve_bytes: float = 12e9,
                   dtype: str = "bf16", stage_counts: Optional[List[int]] = None,
                   max_seq_len: int = 0) -> Dict:
    """SystemConfig document for the planner (proj/src/config.cpp:76-113).

    token_act_bytes: whole-model, unsharded activation bytes per token;
    stage_state_bytes: parameters/optimizer of each stage + a fixed reserve
    for workspaces (GEMM/attention scratch, logits blocks, allocator slack),
    plus, when max_seq_len is given, what Eq. 10 does not charge for
    checkpointed layers of tail chunks (tail_ckpt_excess_bytes) for two
    in-flight tails of max_seq_len tokens with every stage layer checkpointed.
    The planner's arithmetic is untouched (bit-exactness); only its inputs
    describe the executor.
    """
    L = m.layers
    assert L % pp_degree == 0, "layers must divide by pp_degree"
    counts = list(stage_counts) if stage_counts else [L // pp_degree] * pp_degree
    per_layer = m.params_per_layer()
    sbp = state_bytes_per_param(dtype)
    states = []
    tail_reserve = 2.0 * tail_ckpt_excess_bytes(m) * max(counts) * max(0, int(max_seq_len))
    for p in range(pp_degree):
        n = per_layer * counts[p]
        if p == 0:
            n += m.vocab * m.hidden
        if p == pp_degree - 1:
            n += m.vocab * m.hidden + 2 * m.hidden
        states.append(n * sbp + reserve_bytes + tail_reserve)
    cost = dict(cost or default_cost(m))
    return {
        "cluster": {"num_gpus": pp_degree, "pp_degree": pp_degree, "sp_degree": 1,
                    "mem_capacity": float(mem_capacity),
                    "all2all_bandwidth": {}, "all2all_latency": {}},
        # elem_bytes = 4: Eq. 10 charges the dK/dV accumulators of non-tail
        # chunks as 2 * e * D per token per layer, and the executor keeps them
        # in fp32 (bf16 would lose the cross-slice accumulation).  The
        # checkpointed-layer term (3 - 2I) e D l then covers a NON-tail
        # chunk's kept input + K/V (12D charged vs 2D + 4 Hkv hd + 16 kept);
        # for tails (4D charged) the excess is in stage_state_bytes above.
        "model": {"layers": L, "hidden_dim": m.hidden, "elem_bytes": 4.0,
                  # Eq. 10 charges L/d_p layers per stage; with a head-balanced
                  # split the largest stage holds max(counts), so scale up
                  "token_act_bytes": float(activation_bytes_per_token(m) * L * max(counts) * pp_degree / L),
                  "stage_state_bytes": [float(x) for x in states]},
        "cost": cost,
    }


def default_cost(m: ModelConfig, tflops: float = 700e12, attn_tflops: float = 450e12,
                 fixed_per_layer: float = 60e-6) -> Dict[str, float]:
    """Analytic Eq. 1 coefficients (whole model, per GPU count folded in by
    the cost model) before closed-loop fitting: linear work at `tflops`,
    attention pair work at `attn_tflops`, a fixed per-pass overhead."""
    L = m.layers
    a1 = m.linear_flops_per_token_layer() * L / tflops
    # Eq. 1 charges (C+s)^2 - C^2 = 2Cs + s^2 ~ 2 x causal pairs
    a2 = 0.5 * m.attn_flops_per_pair_layer() * L / attn_tflops
    return {"fwd_sec_per_token2": a2, "fwd_sec_per_token": a1, "fwd_sec_fixed": fixed_per_layer * L,
            "bwd_sec_per_token2": 2.5 * a2, "bwd_sec_per_token": 2.0 * a1,
            "bwd_sec_fixed": 2.0 * fixed_per_layer * L, "layer_fwd_seconds": 0.0}
