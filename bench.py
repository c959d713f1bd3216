#!/usr/bin/env python
"""EPP training-step benchmark on B200 (BASELINE.json metric: training
tokens/s + MFU, skewed-length GPT EPP at 1/2/4/8 B200).

A step = one global batch of skewed-length sequences (github_like lengths,
seeded uniform tokens, random-init weights), planned by the C++ planner
(sequence processor + elastic 1F1B + checkpoint MILP), executed by the CUDA
stage executors (d_p = number of GPUs, one stage per GPU), followed by the
AdamW step.  Weak scaling: the batch holds `--seqs-per-gpu` x N sequences.

  value : tokens/s with the step's token ids already resident in HBM and the
          plans pre-solved (paper: plans are pre-solved on the host,
          PAPER.md:712-715), timed with CUDA events, max over ranks.
  e2e   : same metric through the public API from host buffers — planning of
          batch i+1 runs on a host thread during step i, token ids are copied
          from pinned host memory each step, the loss is read back each step.

`--impl reference` times the reference's own CPU path on the host cores:
the compiled reference planner (oracle/_ref) on the step's batch plus the
fp32 CPU numerics of the same model on a bounded token sample.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="gpt-1.3b")
    ap.add_argument("--seqs-per-gpu", type=int, default=64)
    ap.add_argument("--cap", type=int, default=32768)
    ap.add_argument("--preset", default="github_like")
    ap.add_argument("--slices", type=int, default=0, help="fixed slice count N (0 = planner auto-N)")
    ap.add_argument("--pp", type=int, default=0,
                    help="pipeline degree d_p (default: --gpus); --gpus / d_p data-parallel replicas")
    ap.add_argument("--no-calibrate", action="store_true",
                    help="keep the analytic Eq. 1 coefficients (default: fit them on warmup step 0)")
    ap.add_argument("--uniform-min", type=int, default=1, help="preset=uniform: shortest length")
    ap.add_argument("--uniform-max", type=int, default=0, help="preset=uniform: longest length")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample-tokens", type=int, default=256)
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["hbm_gbs"], d["bf16_tflops"], d["bf16_tflops_sustained"], "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = ROOT / "gpurun_out" / f"clocks_rank{index}.csv"

    def __enter__(self):
        try:
            self.path.parent.mkdir(exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self):
        if not self.proc:
            return None
        rows = []
        for line in self.path.read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9 and parts[1].isdigit():
                rows.append(parts)
        if not rows:
            return None
        sm = [int(r[1]) for r in rows]
        load = [int(r[1]) for r in rows if float(r[3] or 0) > 200] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": int(rows[0][2]), "reasons": reasons,
                "samples": len(rows)}


def step_flops(m, plan):
    """Model FLOPs of one step (fwd + bwd = 3x fwd, recompute excluded)."""
    lin = m.linear_flops_per_token_layer()
    per_pair = m.attn_flops_per_pair_layer()
    total = 0.0
    for lay in plan.chunks.values():
        T = lay.tokens
        pairs = 0.0
        for i, s in enumerate(lay.slices):
            ctx = lay.context if (i == 0 and lay.seq >= 0) else 0
            pairs += s * ctx + s * (s + 1) / 2
        total += 3 * (m.layers * (lin * T + per_pair * pairs) + 2 * T * m.hidden * m.vocab)
    return total


def make_batches(args, n_batches, world, vocab, replica=0):
    """Synthetic batches of `seqs_per_gpu * world` sequences (world = the
    pipeline's GPUs); data-parallel replicas draw from disjoint seeds."""
    from paper_2509_21275_b200 import planner, schedule
    out = []
    for i in range(n_batches):
        seed = 1000 + i + 100003 * replica
        lengths = planner.generate_workload(args.preset, args.seqs_per_gpu * world, seed, args.cap,
                                            args.uniform_min, args.uniform_max)
        out.append((lengths, schedule.synthetic_tokens(lengths, vocab, seed=seed)))
    return out


def run_ours(args):
    import torch.distributed as dist

    from paper_2509_21275_b200 import calibrate, gpu, model as M, planner, schedule
    from paper_2509_21275_b200.executor import (DistributedPipeline, LocalPipeline, _ChunkTokens, allreduce_grads,
                                                balanced_stage_counts, pipeline_groups, stage_layers)

    world = args.gpus
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
    torch.cuda.set_device(local)     # before the process group: NCCL binds the current device
    dev = torch.device("cuda", local)
    if world > 1:
        # EPP_BENCH_BACKEND=gloo runs the multi-rank code path with several
        # ranks sharing one GPU (messages staged through host memory): a
        # functional check only, never a reported number
        dist.init_process_group(os.environ.get("EPP_BENCH_BACKEND", "nccl"))
        assert dist.get_world_size() == world
    m = M.MODELS[args.model]
    dp = args.pp or world                    # pipeline degree d_p
    assert world % dp == 0, "--gpus must be a multiple of --pp"
    replicas = world // dp
    replica, prank = rank // dp, rank % dp   # data-parallel replica, stage index
    pipes, dp_groups = pipeline_groups(dp, replicas) if world > 1 else ([None], [None])
    free, total_mem = torch.cuda.mem_get_info()
    # the last stage also runs the LM head: give it fewer layers when that
    # lowers the bottleneck stage (GPT-1.3B at d_p 8: 4,3,3,3,3,3,3,2)
    counts = balanced_stage_counts(m.layers, dp, M.head_layer_equivalents(m))
    cfg = M.planner_config(m, dp, mem_capacity=float(total_mem) - 2e9, cost=M.default_cost(m), stage_counts=counts)
    jobs = os.cpu_count() or 8

    batches = make_batches(args, args.warmup + args.steps, dp, m.vocab, replica)

    def plan_all(config, first):
        out, t = [], time.perf_counter()
        for lengths, _ in batches[first:]:
            out.append(schedule.parse_plan(planner.make_plan_document(config, lengths, args.slices or None, "main",
                                                                      jobs), lengths))
        return out, (time.perf_counter() - t) / max(1, len(out))

    plans, planner_s = plan_all(cfg, 0)

    first, num = stage_layers(m.layers, dp, prank, counts)
    stage = gpu.CudaStage(m, first, num, prank == 0, prank == dp - 1, dtype=args.dtype, device=local)
    stage.init_weights(1234)
    timed_stage = calibrate.TimedStage(stage)

    def make_driver(st):
        if dp > 1:
            return DistributedPipeline(st, prank, dp, dev, m.hidden, gpu.TORCH_DTYPES[args.dtype],
                                       pipe=pipes[replica])
        return LocalPipeline([st], dev)

    driver = make_driver(stage)

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    step_no = [0]

    def optimizer():
        step_no[0] += 1
        allreduce_grads(stage, dp_groups[prank], replicas)   # data-parallel replicas (NCCL all-reduce)
        stage.adamw_step(1e-4, step_no[0])

    # ---- warmup -------------------------------------------------------------
    # Reserve the activation pool up front (all but 6 GB of what is free after
    # the stage's weights and optimizer state): steps whose chunks are larger
    # than any earlier step's then never wait for the driver to map memory.
    if os.environ.get("EPP_BENCH_BACKEND", "nccl") == "nccl":   # (ranks own their GPU)
        free_b, _ = torch.cuda.mem_get_info()
        gpu.pool_reserve(free_b - int(6e9))
    cost_report = {"source": "analytic (model.default_cost)"}
    cal_step = args.warmup - 1          # calibrate on the last (warm) warmup step
    for i in range(args.warmup):
        if i == cal_step and not args.no_calibrate:
            # closed loop: time every stage op of the last warmup step, fit
            # Eq. 1 to it (all ranks' samples, so every rank plans
            # identically) and re-plan the timed batches with the fit
            make_driver(timed_stage).run_step(plans[i], batches[i][1])
            optimizer()
            sync_all()
            samples = timed_stage.samples()
            if world > 1:
                gathered = [None] * world
                dist.all_gather_object(gathered, samples)
                samples = [x for part in gathered for x in part]
            try:
                fitted = calibrate.calibrated_config(cfg, samples)
                cfg_fit = calibrate.planner_config_only(fitted)
                rest, planner_s = plan_all(cfg_fit, args.warmup)
                cfg = cfg_fit
                plans = plans[:args.warmup] + rest
                cost_report = {"source": f"fitted on warmup step {i} ({fitted['_fit']['samples']} stage-op samples)",
                               "fwd_residual": fitted["_fit"]["fwd_residual"],
                               "bwd_residual": fitted["_fit"]["bwd_residual"], "cost": cfg["cost"]}
            except planner.Error as e:
                cost_report = {"source": "analytic (fit failed: %s)" % e}
            continue
        driver.run_step(plans[i], batches[i][1])
        optimizer()
    sync_all()
    stage.loss(reset=True)

    # ---- device-resident timed region (value) -------------------------------
    timed = list(range(args.warmup, args.warmup + args.steps))
    pre = [_ChunkTokens(plans[i], batches[i][1], dev, prank == 0, prank == dp - 1) for i in timed]
    sync_all()
    launches0 = gpu.kernel_launches()
    lib = gpu.lib()
    lib.epp_gpu_profile(1)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    trace = os.environ.get("EPP_BENCH_TRACE")   # diagnostics only: a profiler-perturbed run
    tracer = None
    if trace:
        tracer = torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA,
                                                    torch.profiler.ProfilerActivity.CPU])
        tracer.__enter__()
    with ClockSampler(local) as clk:
        sync_all()
        ev0.record()
        for j, i in enumerate(timed):
            driver.run_step(plans[i], batches[i][1], staged=pre[j])
            optimizer()
        ev1.record()
        sync_all()
    if tracer is not None:
        tracer.__exit__(None, None, None)
        tracer.export_chrome_trace(trace)
    lib.epp_gpu_profile(0)
    launches = gpu.kernel_launches() - launches0
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    tokens = sum(sum(plans[i].lengths) for i in timed)
    flops = sum(step_flops(m, plans[i]) for i in timed)
    if replicas > 1:   # every replica's tokens and FLOPs (each counted once, by its stage 0)
        t = torch.tensor([float(tokens) if prank == 0 else 0.0, flops if prank == 0 else 0.0], device=dev,
                         dtype=torch.float64)
        dist.all_reduce(t)
        tokens, flops = int(t[0].item()), float(t[1].item())
    prof = {}
    classes = ((0, "gemm"), (1, "attn_fwd"), (2, "attn_bwd"), (3, "attn_bwd_dq"), (4, "attn_bwd_dkv"),
               (5, "norm_fwd"), (6, "norm_bwd"), (7, "rope"), (8, "act"), (9, "cross_entropy"),
               (10, "adamw"), (11, "embed"), (12, "copy_fill"))
    for cls, name in classes:
        a, b, c = (ctypes_double(), ctypes_double(), ctypes_i64())
        gpu.check(lib.epp_gpu_profile_read(cls, ctypes_ref(a), ctypes_ref(b), ctypes_ref(c), 1))
        prof[name] = {"ms": a.value, "flops": b.value, "launches": c.value}
    loss_sum, loss_cnt = (stage.loss(reset=True) if prank == dp - 1 else (0.0, 0.0))

    # ---- end-to-end timed region (e2e) ---------------------------------------
    e2e = None
    if not args.no_e2e:
        # the same batches as the device-timed leg, re-planned on the fly
        e2e_batches = batches[args.warmup:]
        ahead = {}

        def solve(k):
            lengths = e2e_batches[k][0]
            ahead[k] = schedule.parse_plan(planner.make_plan_document(cfg, lengths, args.slices or None, "main", jobs),
                                           lengths)

        solve(0)    # batch 0's plan is solved during the (untimed) previous step
        h2d = d2h = 0
        # per-step loss: D2H into pinned memory, read one step later (the
        # host enqueues step k+1 before waiting for step k's loss)
        loss_host = torch.zeros((len(e2e_batches), 2), dtype=torch.float32).pin_memory()
        loss_ev = [torch.cuda.Event() for _ in e2e_batches]
        losses = []
        sync_all()
        e0 = time.perf_counter()
        for k in range(len(e2e_batches)):
            th = None
            if k + 1 < len(e2e_batches):
                th = threading.Thread(target=solve, args=(k + 1,))
                th.start()
            st = driver.run_step(ahead.pop(k), e2e_batches[k][1])
            h2d += st["h2d_bytes"]
            optimizer()
            if prank == dp - 1:
                stage.loss_async(loss_host[k], reset=True)
                loss_ev[k].record()
                d2h += 8
                if k > 0:
                    loss_ev[k - 1].synchronize()
                    losses.append(float(loss_host[k - 1, 0] / max(1.0, float(loss_host[k - 1, 1]))))
            if th:
                th.join()
        if prank == dp - 1:
            loss_ev[-1].synchronize()
            losses.append(float(loss_host[-1, 0] / max(1.0, float(loss_host[-1, 1]))))
        sync_all()
        e_s = time.perf_counter() - e0
        if world > 1:
            # slowest rank's wall time; H2D (stage 0) and D2H (last stage)
            # bytes are counted where they happen and summed over ranks
            t = torch.tensor([e_s], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_s = float(t.item())
            b = torch.tensor([float(h2d), float(d2h)], device=dev)
            dist.all_reduce(b, op=dist.ReduceOp.SUM)
            h2d, d2h = int(b[0].item()), int(b[1].item())
        e_tokens = sum(sum(b[0]) for b in e2e_batches)
        if replicas > 1:
            t = torch.tensor([float(e_tokens) if prank == 0 else 0.0], device=dev, dtype=torch.float64)
            dist.all_reduce(t)
            e_tokens = int(t.item())
        nb = len(e2e_batches)
        e2e = {"value": e_tokens / e_s, "unit": "tokens/s", "h2d_bytes_per_step": h2d // nb,
               "d2h_bytes_per_step": d2h // nb}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    hbm, tf_burst, tf_sus, peak_src = peaks()
    # the planner's simulated makespan of the timed plans vs the measured step
    predicted = sum(calibrate.predicted_seconds(plans[i].doc) for i in timed) / len(timed)
    cost_model = dict(cost_report, predicted_step_s=predicted, measured_step_s=ms / 1e3 / args.steps,
                      measured_over_predicted=(ms / 1e3 / args.steps) / predicted if predicted > 0 else None)
    # dominant kernel class by device time in the timed region
    names = {"gemm": "gemm_tc_kernel (tcgen05 BF16 GEMM, fwd/dgrad/wgrad)",
             "attn_fwd": "attn_fwd (slice-causal flash attention forward)",
             "attn_bwd": "attn_bwd (delta + dQ + dK/dV kernels)"}
    dom = max(("gemm", "attn_fwd", "attn_bwd"), key=lambda k: prof[k]["ms"])
    g = prof[dom]
    achieved = g["flops"] / (g["ms"] / 1e3) / 1e12 if g["ms"] > 0 else 0.0
    traffic = None
    summ = ROOT / "profiles" / "ncu_summary.json"
    if summ.exists():
        traffic = json.loads(summ.read_text()).get("dram_bytes_per_launch", {}).get(dom)
    sec = ms / 1e3
    out = {
        "metric": "training tokens/s + MFU, skewed-length GPT EPP at 1/2/4/8 B200",
        "value": tokens / sec,
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": args.dtype,
        "data": "synthetic (seeded github_like lengths, uniform tokens, random-init weights)",
        "config": {"workload": f"{args.model} EPP, {args.preset} lengths cap {args.cap}, "
                               f"{args.seqs_per_gpu} seqs/GPU/step, d_p={dp}",
                   "model": args.model, "global_batch_seqs": args.seqs_per_gpu * world,
                   "tokens_per_step": tokens / args.steps, "seq_len_cap": args.cap,
                   "slices": args.slices or "auto", "stage_layers": counts,
                   "parallelism": f"pp{dp}" + (f"xdp{replicas}" if replicas > 1 else ""), "l2": "inputs larger than L2 (activations GBs/step)"},
        "mfu": flops / (sec * world * tf_burst * 1e12),
        "mfu_vs_sustained": flops / (sec * world * tf_sus * 1e12),
        "model_tflops_per_gpu": flops / sec / world / 1e12,
        "loss": (loss_sum / loss_cnt) if loss_cnt else None,
        "planner_seconds_per_batch": planner_s,
        "cost_model": cost_model,
        "gpu_launches": launches,
        "roofline": {"bound": "tensor", "kernel": names[dom],
                     "achieved": achieved, "peak": tf_sus, "unit": "TFLOP/s",
                     "frac": achieved / tf_sus if tf_sus else None, "traffic": traffic,
                     "peak_source": f"{peak_src} bf16_tflops_sustained (kernel timed inside a long step)",
                     "share_of_step": g["ms"] / ms if ms else None},
        "kernel_classes": {k: {"ms_per_step": v["ms"] / args.steps,
                               ("tflops" if k.startswith(("gemm", "attn")) else "gbs"):
                                   ((v["flops"] / (v["ms"] / 1e3) / 1e12) if k.startswith(("gemm", "attn"))
                                    else (v["flops"] / (v["ms"] / 1e3) / 1e9)) if v["ms"] else 0.0,
                               "launches_per_step": v["launches"] / args.steps}
                           for k, v in prof.items()},
        "unattributed_ms_per_step": (ms - sum(v["ms"] for k, v in prof.items()
                                               if k not in ("attn_bwd_dq", "attn_bwd_dkv"))) / args.steps,
        "clocks": clk.summary(),
        "e2e": e2e,
    }
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args, m, batches[args.warmup][0], cfg)
    print(json.dumps(out))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def ctypes_double():
    import ctypes
    return ctypes.c_double()


def ctypes_ref(x):
    import ctypes
    return ctypes.byref(x)


def ctypes_i64():
    import ctypes
    return ctypes.c_int64()


# ----------------------------------------------------------------- CPU side --
def cpu_numerics_rate(m, sample_tokens: int, threads: int, seed: int = 0):
    """fp32 CPU oracle (oracle/numerics.py) fwd+bwd of the full model on one
    sample sequence of `sample_tokens` tokens; returns (tokens/s, seconds)."""
    from oracle import numerics as O
    torch.set_num_threads(threads)
    spec = O.ModelSpec(m.arch, m.layers, m.hidden, m.heads, m.kv_heads, m.head_dim, m.ffn, m.vocab,
                       m.rope_theta, m.norm_eps)
    g = torch.Generator().manual_seed(seed)
    params = {}
    for name, shape, kind in O.param_shapes(spec, 0, spec.layers, True, True):
        if kind in ("one",):
            params[name] = torch.ones(shape)
        elif kind == "zero":
            params[name] = torch.zeros(shape)
        else:
            params[name] = torch.empty(shape).normal_(0, 0.02, generator=g)
    tokens = torch.randint(0, m.vocab, (sample_tokens,), generator=g)
    t0 = time.perf_counter()
    O.whole_batch_grads(spec, params, [tokens])
    dt = time.perf_counter() - t0
    return sample_tokens / dt, dt


def ref_planner_seconds(cfg, lengths, jobs):
    from paper_2509_21275_b200 import planner
    so = ROOT / "oracle" / "_ref" / "libepp_ref.so"
    if not so.exists():
        return None
    ref = planner._Api(so, prefix="epp_ref_")
    t0 = time.perf_counter()
    planner.make_plan_document(cfg, lengths, None, "main", jobs, _lib=ref)
    return time.perf_counter() - t0


def cpu_baseline(args, m, lengths, cfg):
    cores = os.cpu_count() or 1
    rate, secs = cpu_numerics_rate(m, args.cpu_sample_tokens, cores)
    plan_s = ref_planner_seconds(cfg, lengths, cores)
    tokens = sum(lengths)
    # CPU time for the whole step = reference planning of the batch + fp32
    # numerics of all its tokens at the sampled rate.
    step_s = (plan_s or 0.0) + tokens / rate
    return {"value": tokens / step_s, "unit": "tokens/s", "cores": cores,
            "kind": "reference" if plan_s is not None else "port",
            "sample": f"reference planner (oracle/_ref make_plan, jobs={cores}) on the step's "
                      f"{len(lengths)}-sequence batch ({plan_s:.3f}s) + fp32 torch-CPU oracle "
                      f"fwd+bwd of {args.model} on a {args.cpu_sample_tokens}-token sample "
                      f"({secs:.1f}s, {rate:.1f} tokens/s), extrapolated to the batch's {tokens} tokens"}


def run_reference(args):
    world = args.gpus
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2509_21275_b200 import model as M, planner
    m = M.MODELS[args.model]
    cfg = M.planner_config(m, world, mem_capacity=181e9, cost=M.default_cost(m))
    cores = os.cpu_count() or 1
    batches = make_batches(args, args.warmup + args.steps, world, m.vocab)
    so = ROOT / "oracle" / "_ref" / "libepp_ref.so"
    ref = planner._Api(so, prefix="epp_ref_") if so.exists() else None
    kind = "reference" if ref else "port"
    times, toks = [], []
    for i, (lengths, _) in enumerate(batches):
        t0 = time.perf_counter()
        planner.make_plan_document(cfg, lengths, None, "main", cores, _lib=ref)
        plan_s = time.perf_counter() - t0
        rate, secs = cpu_numerics_rate(m, args.cpu_sample_tokens, cores, seed=i)
        if i >= args.warmup:
            times.append(plan_s + secs)
            toks.append(args.cpu_sample_tokens)
    value = sum(toks) / sum(times)
    sample = (f"per step: reference planner (oracle/_ref, jobs={cores}) on the step's "
              f"{len(batches[0][0])}-sequence batch + fp32 torch-CPU oracle fwd+bwd of {args.model} "
              f"on a {args.cpu_sample_tokens}-token sample; value = sample tokens / step time")
    out = {"metric": "training tokens/s + MFU, skewed-length GPT EPP at 1/2/4/8 B200", "impl": "reference",
           "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f32",
           "data": "synthetic (seeded github_like lengths, uniform tokens, random-init weights)",
           "config": {"workload": f"{args.model} EPP, {args.preset} lengths cap {args.cap}, "
                                  f"{args.seqs_per_gpu} seqs/GPU/step, d_p={world}",
                      "model": args.model, "parallelism": f"pp{world}"},
           "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": kind, "sample": sample},
           "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
