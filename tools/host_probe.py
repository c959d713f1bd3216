"""Host-side cost of the stage executor: wall time of each epp_stage_forward /
epp_stage_backward call (the C ABI enqueues asynchronously) against the GPU
time of the same call, for one planned batch.  If host >= GPU, the GPU
idles waiting for launches.

    python tools/host_probe.py --model gpt-7b --preset uniform --len 2048 --seqs 32
"""
import argparse
import statistics
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_21275_b200 import gpu, model as M, planner, schedule  # noqa: E402
from paper_2509_21275_b200.executor import _ChunkTokens, _op, stage_layers  # noqa: E402
from paper_2509_21275_b200.schedule import stage_ops  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="gpt-7b")
    ap.add_argument("--preset", default="uniform")
    ap.add_argument("--len", type=int, default=2048)
    ap.add_argument("--cap", type=int, default=32768)
    ap.add_argument("--seqs", type=int, default=32)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    m = M.MODELS[args.model]
    cfg = M.planner_config(m, 1, mem_capacity=float(torch.cuda.mem_get_info()[1]) - 2e9)
    if args.preset == "uniform":
        lengths = planner.generate_workload("uniform", args.seqs, 7, args.len, args.len, args.len)
    else:
        lengths = planner.generate_workload(args.preset, args.seqs, 7, args.cap)
    plan = schedule.parse_plan(planner.make_plan_document(cfg, lengths, None, "main", 8), lengths)
    tokens = schedule.synthetic_tokens(lengths, m.vocab, seed=7)
    st = gpu.CudaStage(m, 0, m.layers, True, True, dtype="bf16")
    st.init_weights(1)
    free_b, _ = torch.cuda.mem_get_info()
    gpu.pool_reserve(free_b - int(6e9))
    dev = torch.device("cuda")
    for rep in range(2):
        toks = _ChunkTokens(plan, tokens, dev, True, True)
        torch.cuda.synchronize()
        host_f, host_b, gpu_f, gpu_b = [], [], [], []
        t_all = time.perf_counter()
        for unit in plan.units:
            for kind, pos in stage_ops(len(unit.chunks), unit.n_prefill, 1, 1, unit.backward_order):
                op = _op(plan, unit, pos, 0, toks)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                t0 = time.perf_counter()
                if kind == "F":
                    st.forward(op, None)
                else:
                    st.backward(op, None)
                t1 = time.perf_counter()
                e1.record()
                (host_f if kind == "F" else host_b).append((t1 - t0) * 1e3)
                (gpu_f if kind == "F" else gpu_b).append((e0, e1))
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t_all) * 1e3
        gf = [a.elapsed_time(b) for a, b in gpu_f]
        gb = [a.elapsed_time(b) for a, b in gpu_b]
        print(f"rep {rep}: chunks {len(host_f)}  wall {wall:.0f} ms  "
              f"fwd host {statistics.mean(host_f):.2f} ms / gpu {statistics.mean(gf):.2f} ms   "
              f"bwd host {statistics.mean(host_b):.2f} ms / gpu {statistics.mean(gb):.2f} ms  "
              f"sum gpu {sum(gf) + sum(gb):.0f} ms")


if __name__ == "__main__":
    main()
