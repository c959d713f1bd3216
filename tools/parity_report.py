"""Parity report (GPU): the CUDA stage executor against the fp32 CPU oracle
on planned batches (split + packed + hybrid chunks, KV carried across
slices, checkpoint ladder on/off, 1 and 2 stages), fp32 mode and bf16 mode
(reported separately, as north_star asks).  Writes one JSON document.

    python tools/parity_report.py > profiles/r01_parity.json
"""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from oracle import numerics as O  # noqa: E402
from paper_2509_21275_b200 import planner, schedule as S  # noqa: E402
from test_gpu_stage import LENGTHS, cfg_model, make_plan, run_gpu, spec_of  # noqa: E402


def main():
    torch.cuda.set_device(0)
    rows = []
    for arch in ("gpt", "llama"):
        for dp, slices, tight in ((1, 3, False), (2, 3, False), (2, 4, True)):
            m = cfg_model(arch)
            plan = make_plan(planner, m, LENGTHS, dp, slices, tight)
            params = O.init_params(spec_of(m), seed=7)
            tokens = S.synthetic_tokens(LENGTHS, m.vocab, seed=4)
            ref_loss, ref_grads, _ = O.whole_batch_grads(spec_of(m), params,
                                                         [torch.from_numpy(t).long() for t in tokens])
            for dtype in ("f32", "bf16"):
                loss_sum, cnt, grads = run_gpu(m, params, plan, tokens, dtype)
                errs = {k: float((grads[k] - g).norm() / (g.norm() + 1e-30)) for k, g in ref_grads.items()}
                rows.append({
                    "arch": arch, "dtype": dtype, "pp_degree": dp, "slices": slices,
                    "checkpoint_ladder": bool(any(any(v for r in u.ckpt for v in r) for u in plan.units)),
                    "chunks": len(plan.chunks), "tokens": sum(LENGTHS),
                    "loss_rel_err": abs(loss_sum / cnt - ref_loss.item()) / ref_loss.item(),
                    "grad_rel_err_max": max(errs.values()), "grad_rel_err_median": sorted(errs.values())[len(errs) // 2],
                    "worst_param": max(errs, key=errs.get),
                    "tolerance": {"loss": 1e-5 if dtype == "f32" else 5e-3, "grad": 1e-3 if dtype == "f32" else 3e-2},
                })
    print(json.dumps({"oracle": "oracle/numerics.py whole_batch_grads (fp32, torch CPU)",
                      "lengths": LENGTHS, "model": "tests/test_gpu_stage.cfg_model (4 layers, d=256)",
                      "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
