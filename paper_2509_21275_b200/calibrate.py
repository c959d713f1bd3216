"""Closed-loop cost model: measured stage times -> Eq. 1 coefficients.

The planner prices every chunk with Eq. 1 (proj/src/cost_model.cpp:12-25),
whose coefficients the paper obtains by offline profiling.
This module measures them on the GPU executor itself:

  1. `TimedStage` wraps a stage (gpu.CudaStage) and records CUDA events
     around every forward / backward call of a step;
  2. `samples()` turns those into fit samples {context, slices, phase,
     seconds} (a backward that re-ran checkpointed layers is charged the
     recompute estimated from its forward: Eq. 1 prices recompute
     separately);
  3. `calibrated_config()` feeds them to fit_cost_params
     (proj/src/cost_model.cpp:143-223, the planner library's C ABI) and returns
     the planner configuration with the fitted coefficients;
  4. `predicted_seconds()` is the planner's simulated makespan of a plan
     (plan_simulated_seconds, planner.cpp:489-493), to compare with the
     measured step time.
"""
from __future__ import annotations

import copy
import json
from typing import Dict, List

import torch

from . import planner


class TimedStage:
    """Delegates to `stage`, timing each forward/backward on the current
    stream (CUDA events; read after the step has been synchronised)."""

    def __init__(self, stage):
        self.stage = stage
        self.records = []   # (op, phase, start event, end event)

    def __getattr__(self, name):
        return getattr(self.stage, name)

    def _timed(self, phase, fn, op, x, **kw):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn(op, x, **kw)
        b.record()
        self.records.append((op, phase, a, b))
        return out

    # keyword arguments (e.g. out_ptr, the P2P mailbox the stage writes into)
    # pass through to the wrapped stage
    def forward(self, op, act_in, **kw):
        return self._timed("forward", self.stage.forward, op, act_in, **kw)

    def backward(self, op, grad_in, **kw):
        return self._timed("backward", self.stage.backward, op, grad_in, **kw)

    def samples(self) -> List[Dict]:
        """Fit samples.  A backward that first re-ran `ckpt` of the stage's
        `num` layers is charged its recompute, estimated from the same
        chunk's measured forward, which Eq. 1 prices separately
        (recompute_time, cost_model.cpp:68-78).  Only the layers' share of
        that forward is scaled: on the last stage the forward call also runs
        the LM head (forward and backward), which recompute never repeats;
        its share is split off by model FLOPs."""
        st = self.stage
        layers = max(1, int(getattr(st, "num", 1)))
        m = getattr(st, "model", None)
        fwd = {}
        for op, phase, a, b in self.records:
            if phase == "forward":
                fwd[op.id] = a.elapsed_time(b) / 1e3
        out = []
        for op, phase, a, b in self.records:
            sec = a.elapsed_time(b) / 1e3
            if phase == "backward" and op.ckpt_layers > 0:
                if op.id not in fwd:
                    continue
                ckpt = _stage_ckpt(st, op.ckpt_layers, layers)
                sec -= _layer_forward_share(m, op, layers, getattr(st, "has_head", False)) * fwd[op.id] * ckpt / layers
            out.append({"context": int(op.context), "slices": [int(s) for s in op.slices], "phase": phase,
                        "seconds": sec})
        return out


def _stage_ckpt(stage, plan_count: int, layers: int) -> int:
    """Layers the stage actually re-ran for a plan count (gpu.CudaStage
    rescales counts of non-uniform stages; never more than the stage has)."""
    f = getattr(stage, "_ckpt_layers", None)
    return int(f(plan_count)) if f else min(int(plan_count), layers)


def _layer_forward_share(m, op, layers: int, has_head: bool) -> float:
    """Fraction of a forward call spent in the transformer layers (model
    FLOPs): 1 except on the last stage, whose forward also runs the LM head
    forward + backward (3 x 2 T D V)."""
    if m is None or not has_head:
        return 1.0
    T = sum(op.slices)
    pairs = sum(s * (op.context if (i == 0 and op.seq >= 0) else 0) + s * (s + 1) / 2
                for i, s in enumerate(op.slices))
    lay = layers * (m.linear_flops_per_token_layer() * T + m.attn_flops_per_pair_layer() * pairs)
    head = 3.0 * 2.0 * T * m.hidden * m.vocab
    return lay / (lay + head) if lay + head > 0 else 1.0


def calibrated_config(cfg: Dict, samples: List[Dict]) -> Dict:
    """`cfg` with Eq. 1 coefficients fitted to `samples` (needs >= 4 samples
    per phase over >= 2 distinct chunk sizes)."""
    fit = planner.fit_cost_params(cfg, samples)
    out = copy.deepcopy(cfg)
    # the least-squares fit is unconstrained; a coefficient that comes out
    # negative (noise around ~0, e.g. a tiny fixed cost) is clamped to 0, the
    # planner's config contract (config.cpp validate: non-negative costs)
    out["cost"].update({k: max(0.0, float(v)) for k, v in fit["cost"].items()})
    out["_fit"] = {"fwd_residual": fit["fwd_residual"], "bwd_residual": fit["bwd_residual"],
                   "samples": len(samples)}
    return out


def planner_config_only(cfg: Dict) -> Dict:
    """Drop bookkeeping keys before handing a config to the planner."""
    return {k: v for k, v in cfg.items() if not k.startswith("_")}


def predicted_seconds(plan_doc) -> float:
    """Simulated makespan summed over the plan's units (seconds)."""
    _, total = planner.simulate_plan_document(plan_doc if isinstance(plan_doc, str) else json.dumps(plan_doc))
    return total
