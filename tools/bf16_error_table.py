"""Diagnostics: per-parameter gradient error of the bf16 executor against the
fp32 oracle, next to two torch bf16 yardsticks of the SAME model (oracle run
under torch.autocast(bfloat16), and the oracle with every parameter and
activation in bf16).  Usage: python tools/bf16_error_table.py [gpt-1.3b|llama-7b]
(GPU; prints one JSON line)."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import torch  # noqa: E402

import test_gpu_bench_shapes as T  # noqa: E402
from oracle import numerics as O  # noqa: E402
from paper_2509_21275_b200 import planner, schedule as S  # noqa: E402


def pure_bf16(arch):
    m = T.WIDTHS[arch]
    params = {k: v.cuda().bfloat16() for k, v in O.init_params(T.spec_of(m), seed=11).items()}
    tokens = S.synthetic_tokens(T.LENGTHS, m.vocab, seed=5)
    _, grads, _ = O.whole_batch_grads(T.spec_of(m), params, [torch.from_numpy(t).long().cuda() for t in tokens])
    return {k: g.float() for k, g in grads.items()}


def main():
    arch = sys.argv[1] if len(sys.argv) > 1 else "gpt-1.3b"
    dp = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    m = T.WIDTHS[arch]
    plan = T.make_plan(planner, m, dp, False)
    loss_sum, cnt, grads, _ = T.run_cuda(m, plan, "bf16")
    ref_loss, ref, _ = T.oracle(arch)
    _, ac, _ = T.oracle(arch, autocast=True)
    pb = pure_bf16(arch)
    rows = []
    for k, g in ref.items():
        rows.append({"param": k, "ours": T.rel(grads[k], g), "autocast": T.rel(ac[k], g), "pure_bf16": T.rel(pb[k], g)})
    rows.sort(key=lambda r: -r["ours"] / max(r["autocast"], 1e-12))
    print(json.dumps({"arch": arch, "dp": dp, "loss": loss_sum / cnt, "oracle_loss": ref_loss, "rows": rows}))


if __name__ == "__main__":
    main()
