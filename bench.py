#!/usr/bin/env python
"""EPP training-step benchmark on B200 (BASELINE.json metric: training
tokens/s + MFU, skewed-length GPT EPP at 1/2/4/8 B200).

Default workload = configs[2]: GPT-7B shape, github_like lengths capped at
16K, 64 sequences per GPU per step (512 at 8 GPUs), d_p = N
pipeline stages, elastic schedule + chunk-level adaptive checkpointing (at
N=1 the 7B model's optimizer state leaves ~60 GB for activations, so the
checkpoint ladder is active).  A step = one global batch, planned by the C++
planner, executed by the CUDA stage executors, followed by AdamW.

  value : tokens/s with the step's token ids resident in HBM and the plans
          pre-solved, CUDA events, max over ranks.  No
          per-launch instrumentation in this pass.
  e2e   : same metric through the public API from host buffers: batch i+1 is
          planned on a host thread during step i, token ids are copied from
          pinned host memory every step, every step's loss is read back.
  kernel_classes / roofline : a separate instrumented pass over the first
          timed batches (CUDA events around every launch on its stream).
  cpu_baseline : the reference planner (oracle/_ref) + fp32 CPU numerics on
          the host cores (rank 0).

Both arms plan with the same SystemConfig (bench_config): the committed Eq. 1
fit profiles/cost_<model>.json (bench.py --save-cost refreshes it) and
mem_capacity = model.B200_MEM_CAPACITY.  The warmup step is still timed per
stage op and refitted (closed loop, §8f.1); --replan plans the timed batches
with that fresh fit instead.

`--impl reference` times the reference's own CPU path on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

METRIC = "training tokens/s + MFU, skewed-length GPT EPP at 1/2/4/8 B200"
DATA = "synthetic (seeded github_like lengths, uniform tokens, random-init weights)"
REF_SO = ROOT / "oracle" / "_ref" / "libepp_ref.so"
E2E_SEED0 = 7000   # the e2e leg's batches: fresh seeds (never trained on)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="gpt-7b")
    ap.add_argument("--seqs-per-gpu", type=int, default=64)
    ap.add_argument("--cap", type=int, default=16384)
    ap.add_argument("--preset", default="github_like")
    ap.add_argument("--slices", type=int, default=0, help="fixed slice count N (0 = planner auto-N)")
    ap.add_argument("--pp", type=int, default=0,
                    help="pipeline degree d_p (default: --gpus); --gpus / d_p data-parallel replicas")
    ap.add_argument("--cost", default="auto",
                    help="Eq. 1 coefficients: 'auto' (profiles/cost_<model>.json if present, else analytic), "
                         "'analytic', or a JSON path")
    ap.add_argument("--replan", action="store_true",
                    help="plan the timed batches with the fit of the last warmup step (closed loop)")
    ap.add_argument("--save-cost", default="", help="write the warmup fit to this path")
    ap.add_argument("--uniform-min", type=int, default=1, help="preset=uniform: shortest length")
    ap.add_argument("--uniform-max", type=int, default=0, help="preset=uniform: longest length")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--zero", action="store_true", help="ZeRO-1 optimizer-state sharding across replicas")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--prof-steps", type=int, default=2, help="batches re-run in the instrumented pass")
    ap.add_argument("--cpu-sample-tokens", type=int, default=1024)
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
        pw = [float(r[3]) for r in rows if float(r[3] or 0) > 200]
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": int(rows[0][2]), "reasons": reasons,
                "samples": len(rows), "power_w": statistics.median(pw) if pw else None}


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


def bench_config(args, m, dp):
    """(SystemConfig, stage layer counts, cost source): identical in both arms
    (pure Python; loads no native library)."""
    from paper_2509_21275_b200 import model as M
    from paper_2509_21275_b200.executor import balanced_stage_counts
    counts = balanced_stage_counts(m.layers, dp, M.head_layer_equivalents(m))
    src, cost = "analytic (model.default_cost)", M.default_cost(m)
    path = ROOT / "profiles" / f"cost_{args.model}.json" if args.cost == "auto" else Path(args.cost)
    if args.cost != "analytic" and path.exists():
        cost = json.loads(path.read_text())["cost"]
        src = f"{path.relative_to(ROOT) if path.is_relative_to(ROOT) else path} (Eq. 1 fit of GPU stage timings)"
    cfg = M.planner_config(m, dp, mem_capacity=M.B200_MEM_CAPACITY, cost=cost, stage_counts=counts,
                           max_seq_len=args.cap)
    return cfg, counts, src


def make_lengths(args, n_batches, world, replica=0, _lib=None, seed0=1000):
    from paper_2509_21275_b200 import planner
    out = []
    for i in range(n_batches):
        seed = seed0 + i + 100003 * replica
        out.append((seed, planner.generate_workload(args.preset, args.seqs_per_gpu * world, seed, args.cap,
                                                    args.uniform_min, args.uniform_max, _lib=_lib)))
    return out


def make_batches(args, n_batches, world, vocab, replica=0, seed0=1000):
    """Synthetic batches of `seqs_per_gpu * world` sequences (world = the
    pipeline's GPUs); data-parallel replicas draw from disjoint seeds."""
    from paper_2509_21275_b200 import schedule
    return [(lengths, schedule.synthetic_tokens(lengths, vocab, seed=seed))
            for seed, lengths in make_lengths(args, n_batches, world, replica, seed0=seed0)]


def global_targets(args, n_batches, world, replicas, seed0=1000):
    """Next-token targets of every step's WHOLE global batch (all replicas):
    each replica normalises its loss by this, so the replicas' summed
    gradients are the global per-token mean (GradSync)."""
    per = [make_lengths(args, n_batches, world, q, seed0=seed0) for q in range(replicas)]
    return [sum(max(0, n - 1) for q in range(replicas) for n in per[q][i][1]) for i in range(n_batches)]


PROF_CLASSES = ((0, "gemm"), (1, "attn_fwd"), (2, "attn_bwd"), (3, "attn_bwd_dq"), (4, "attn_bwd_dkv"),
                (5, "norm_fwd"), (6, "norm_bwd"), (7, "rope"), (8, "act"), (9, "cross_entropy"),
                (10, "adamw"), (11, "embed"), (12, "copy_fill"),
                (13, "gemm_store"), (14, "gemm_wgrad_accum"), (15, "gemm_addres"), (16, "gemm_store_f32"),
                (17, "gemm_up_gelu"), (18, "gemm_dgrad_gelu"), (19, "gemm_qkv_rope"), (20, "gemm_up_swiglu"),
                (21, "gemm_dgrad_swiglu"))


def read_profile(lib):
    import ctypes
    from paper_2509_21275_b200 import gpu
    out = {}
    for cls, name in PROF_CLASSES:
        a, b, c = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        gpu.check(lib.epp_gpu_profile_read(cls, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), 1))
        out[name] = {"ms": a.value, "flops": b.value, "launches": c.value}
    return out


def run_ours(args):
    import torch.distributed as dist

    from paper_2509_21275_b200 import calibrate, gpu, model as M, planner, schedule
    from paper_2509_21275_b200.executor import (DistributedPipeline, GradSync, LocalPipeline, _ChunkTokens,
                                                pipeline_groups, stage_layers)

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
    assert total_mem >= M.B200_MEM_CAPACITY, "planner capacity exceeds this device"
    cfg, counts, cost_src = bench_config(args, m, dp)
    jobs = os.cpu_count() or 8

    batches = make_batches(args, args.warmup + args.steps, dp, m.vocab, replica)
    targets = global_targets(args, args.warmup + args.steps, dp, replicas)

    def plan_all(config, first):
        out, t = [], time.perf_counter()
        for lengths, _ in batches[first:]:
            out.append(schedule.parse_plan(planner.make_plan_document(config, lengths, args.slices or None, "main",
                                                                      jobs), lengths))
        return out, (time.perf_counter() - t) / max(1, len(out))

    plans, planner_s = plan_all(cfg, 0)

    first, num = stage_layers(m.layers, dp, prank, counts)
    stage = gpu.CudaStage(m, first, num, prank == 0, prank == dp - 1, dtype=args.dtype, device=local,
                          plan_stage_layers=m.layers // dp)
    stage.init_weights(1234)
    timed_stage = calibrate.TimedStage(stage)

    # P2P mailboxes (N > 1) hold two of the largest messages any plan of
    # this run sends: the pre-planned batches, the e2e leg's batches (planned
    # again inside its timed region) and 1.5x headroom for --replan's refit.
    if dp > 1:
        e2e_lengths = [] if args.no_e2e else [b[0] for b in make_batches(args, args.steps, dp, m.vocab, replica,
                                                                         seed0=E2E_SEED0)]
        biggest = max(lay.tokens for pl in plans for lay in pl.chunks.values())
        for lengths in e2e_lengths:
            pl = schedule.parse_plan(planner.make_plan_document(cfg, lengths, args.slices or None, "main", jobs),
                                     lengths)
            biggest = max(biggest, max(lay.tokens for lay in pl.chunks.values()))
        max_tokens = max(int(1.5 * biggest), args.cap)

    def make_driver(st):
        if dp > 1:
            return DistributedPipeline(st, prank, dp, dev, m.hidden, gpu.TORCH_DTYPES[args.dtype],
                                       pipe=pipes[replica], max_tokens=max_tokens)
        return LocalPipeline([st], dev)

    driver = make_driver(stage)

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    step_no = [0]
    # data-parallel replicas: bucketed reductions overlapped with the last
    # backward (NCCL), optional ZeRO-1 optimizer-state sharding
    gsync = GradSync(stage, dp_groups[prank], replicas, zero=args.zero)

    def run(drv, i, staged=None, tgt=None):
        out = drv.run_step(plans[i], batches[i][1], staged=staged,
                           total_targets=(targets[i] if tgt is None else tgt) if replicas > 1 else None)
        gsync.launch()
        return out

    def optimizer():
        step_no[0] += 1
        gsync.finish()
        stage.adamw_step(1e-4, step_no[0])
        gsync.after_step()

    # ---- warmup -------------------------------------------------------------
    # Reserve the activation pool up front (all but 6 GB of what is free after
    # the stage's weights and optimizer state): steps whose chunks are larger
    # than any earlier step's then never wait for the driver to map memory.
    if os.environ.get("EPP_BENCH_BACKEND", "nccl") == "nccl":   # (ranks own their GPU)
        free_b, _ = torch.cuda.mem_get_info()
        gpu.pool_reserve(free_b - int(6e9))
    cost_report = {"source": cost_src}
    cal_step = args.warmup - 1          # time the last (warm) warmup step per stage op
    for i in range(args.warmup):
        if i == cal_step:
            # closed loop: fit Eq. 1 to every stage op of this step (all
            # ranks' samples, so every rank plans identically)
            run(make_driver(timed_stage), i)
            optimizer()
            sync_all()
            samples = timed_stage.samples()
            if world > 1:
                gathered = [None] * world
                dist.all_gather_object(gathered, samples)
                samples = [x for part in gathered for x in part]
            try:
                fitted = calibrate.calibrated_config(cfg, samples)
                cost_report.update({"warmup_fit": {"samples": fitted["_fit"]["samples"],
                                                   "fwd_residual": fitted["_fit"]["fwd_residual"],
                                                   "bwd_residual": fitted["_fit"]["bwd_residual"],
                                                   "cost": fitted["cost"]}})
                if args.save_cost and rank == 0:
                    Path(args.save_cost).write_text(json.dumps(
                        {"model": args.model, "cap": args.cap, "pp": dp, "fitted_on": f"warmup step {i}",
                         "fwd_residual": fitted["_fit"]["fwd_residual"],
                         "bwd_residual": fitted["_fit"]["bwd_residual"], "cost": fitted["cost"]}, indent=1))
                if args.replan:
                    cfg = calibrate.planner_config_only(fitted)
                    rest, planner_s = plan_all(cfg, args.warmup)
                    plans = plans[:args.warmup] + rest
                    cost_report["source"] = f"fitted on warmup step {i} (--replan)"
            except planner.Error as e:
                cost_report["warmup_fit"] = f"fit failed: {e}"
            continue
        run(driver, i)
        optimizer()
    sync_all()
    stage.loss(reset=True)

    # ---- device-resident timed region (value): no instrumentation ----------
    timed = list(range(args.warmup, args.warmup + args.steps))
    pre = [_ChunkTokens(plans[i], batches[i][1], dev, prank == 0, prank == dp - 1) for i in timed]
    sync_all()
    launches0 = gpu.kernel_launches()
    p2p0 = getattr(driver, "p2p_bytes", 0)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        sync_all()
        ev0.record()
        for j, i in enumerate(timed):
            run(driver, i, staged=pre[j])
            optimizer()
        ev1.record()
        sync_all()
    launches = gpu.kernel_launches() - launches0
    p2p_bytes = getattr(driver, "p2p_bytes", 0) - p2p0
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
    loss_sum, loss_cnt = (stage.loss(reset=True) if prank == dp - 1 else (0.0, 0.0))

    # ---- instrumented pass (kernel classes, roofline): first timed batches --
    lib = gpu.lib()
    nprof = max(1, min(args.prof_steps, args.steps))
    read_profile(lib)                         # drop anything recorded so far
    sync_all()
    lib.epp_gpu_profile(1)
    pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pe0.record()
    for j, i in enumerate(timed[:nprof]):
        run(driver, i, staged=pre[j])
        optimizer()
    pe1.record()
    sync_all()
    lib.epp_gpu_profile(0)
    prof = read_profile(lib)
    prof_ms = pe0.elapsed_time(pe1)
    stage.loss(reset=True) if prank == dp - 1 else None

    # ---- measured trace of one step (trace document v1) vs the simulation --
    trace_block = measured_trace_step(args, lambda: run(driver, timed[0], staged=pre[0]), stage, plans[timed[0]],
                                      cfg, optimizer, sync_all, dist, world, rank, dp, prank)

    # ---- end-to-end timed region (e2e) ---------------------------------------
    e2e = None
    if not args.no_e2e:
        # fresh batches (never trained on): the per-step losses are honest
        e2e_batches = make_batches(args, args.steps, dp, m.vocab, replica, seed0=E2E_SEED0)
        e2e_targets = global_targets(args, args.steps, dp, replicas, seed0=E2E_SEED0)

        def e2e_run(k, plan, tokens):
            out = driver.run_step(plan, tokens, total_targets=e2e_targets[k] if replicas > 1 else None)
            gsync.launch()
            return out
        e2e = run_e2e(args, e2e_run, stage, cfg, e2e_batches, jobs, dev, world, dp, prank, replicas,
                      optimizer, sync_all, dist)

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    hbm, tf_burst, tf_sus, peak_src = peaks()
    predicted = sum(calibrate.predicted_seconds(plans[i].doc) for i in timed) / len(timed)
    cost_model = dict(cost_report, predicted_step_s=predicted, measured_step_s=ms / 1e3 / args.steps,
                      measured_over_predicted=(ms / 1e3 / args.steps) / predicted if predicted > 0 else None)
    names = {"gemm": "gemm_tc2_kernel / gemm_tc_kernel (tcgen05 BF16 GEMM, fwd/dgrad/wgrad)",
             "attn_fwd": "attn_fwd_tc (slice-causal flash attention forward)",
             "attn_bwd": "attn_bwd_dq_tc + attn_bwd_dkv_tc (slice-causal flash attention backward)"}
    dom = max(("gemm", "attn_fwd", "attn_bwd"), key=lambda k: prof[k]["ms"])
    g = prof[dom]
    achieved = g["flops"] / (g["ms"] / 1e3) / 1e12 if g["ms"] > 0 else 0.0
    traffic, traffic_src = None, None
    summ = ROOT / "profiles" / "ncu_summary.json"
    if summ.exists():
        sj = json.loads(summ.read_text())
        traffic = sj.get("dram_bytes_per_launch", {}).get(dom)
        traffic_src = sj.get("source")
    sec = ms / 1e3
    gemm_flops_class = {k: v for k, v in prof.items()}
    out = {
        "metric": METRIC,
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
        "data": DATA,
        "config": {"workload": f"{args.model} EPP, {args.preset} lengths cap {args.cap}, "
                               f"{args.seqs_per_gpu} seqs/GPU/step, d_p={dp}",
                   "model": args.model, "global_batch_seqs": args.seqs_per_gpu * world,
                   "tokens_per_step": tokens / args.steps, "seq_len_cap": args.cap,
                   "slices": args.slices or "auto", "stage_layers": counts,
                   "ckpt_layers_per_step": sum(sum(sum(r) for r in u.ckpt) for i in timed for u in plans[i].units)
                                           / args.steps,
                   "parallelism": f"pp{dp}" + (f"xdp{replicas}" if replicas > 1 else "") + ("+zero1" if args.zero and replicas > 1 else ""),
                   "l2": "inputs larger than L2 (activations GBs/step)"},
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
                     "traffic_source": traffic_src,
                     "peak_source": f"{peak_src} bf16_tflops_sustained (kernel timed inside a long step)",
                     "share_of_step": g["ms"] / prof_ms if prof_ms else None,
                     "timed_in": f"instrumented pass over {nprof} of the timed batches"},
        "kernel_classes": {k: {"ms_per_step": v["ms"] / nprof,
                               ("tflops" if k.startswith(("gemm", "attn")) else "gbs"):
                                   ((v["flops"] / (v["ms"] / 1e3) / 1e12) if k.startswith(("gemm", "attn"))
                                    else (v["flops"] / (v["ms"] / 1e3) / 1e9)) if v["ms"] else 0.0,
                               "launches_per_step": v["launches"] / nprof}
                           for k, v in gemm_flops_class.items()},
        "instrumented_ms_per_step": prof_ms / nprof,
        "unattributed_ms_per_step": (prof_ms - sum(v["ms"] for k, v in prof.items()
                                                   if k not in ("attn_bwd_dq", "attn_bwd_dkv")
                                                   and not k.startswith("gemm_"))) / nprof,
        "clocks": clk.summary(),
        "e2e": e2e,
        # the step runs at the board's power cap (sw_power_cap): throughput
        # is energy per token, which this reports (median board power under
        # load x device time per token)
        "energy": None,
        "trace": trace_block,
    }
    if out["clocks"] and out["clocks"].get("power_w") and out["value"]:
        # rank 0's board power, taken as every rank's (whole-job tokens/s)
        out["energy"] = {"power_w_per_gpu": out["clocks"]["power_w"],
                         "joules_per_token": out["clocks"]["power_w"] * world / out["value"]}
    # HBM: what the planner was told against what the stage actually used
    # (weights/grads/Adam state + the activation pool's high-water mark)
    free_b, total_b = torch.cuda.mem_get_info()
    _, pool_peak = stage.memory()
    out["memory"] = {"device_total_bytes": total_b, "planner_mem_capacity": cfg["cluster"]["mem_capacity"],
                     "planner_stage_state_bytes": cfg["model"]["stage_state_bytes"][prank],
                     "planner_token_act_bytes": cfg["model"]["token_act_bytes"],
                     "stage_state_bytes": stage.state_bytes(), "activation_pool_peak_bytes": pool_peak}
    if world > 1:
        # stage-to-stage activations/gradients (this rank's sends; rank 0 is a
        # first stage, so its sends are the forward activations of one hop)
        hop_bytes = p2p_bytes / args.steps
        out["p2p"] = {"transport": getattr(driver, "transport", None), "bytes_per_step_rank0": hop_bytes,
                      "gbs_rank0_avg_over_step": hop_bytes / (sec / args.steps) / 1e9,
                      "nvlink_gbs_per_direction": 900.0,
                      "note": "rank 0's send volume over the whole step time (not per-transfer bandwidth)"}
    if not args.no_cpu_baseline:
        out["cpu_baseline"], out["planner"] = cpu_side(args, m, dp, cfg, tokens / args.steps,
                                                      flops / args.steps / max(1, replicas),
                                                      batches[args.warmup][0], jobs)
    print(json.dumps(out))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def measured_trace_step(args, run_step, stage, plan, cfg, optimizer, sync_all, dist, world, rank, dp, prank):
    """One step with the stages' native per-op trace on (include/epp_gpu.h
    epp_stage_trace): a measured trace document v1 of replica 0, diffed event
    by event against the planner's simulation of the same plan with the same
    cost coefficients (the closed loop's per-op residuals).  Both documents
    go to gpurun_out/."""
    from paper_2509_21275_b200 import planner, trace as TR
    sync_all()
    stage.trace(True)
    run_step()
    optimizer()
    sync_all()
    evs = stage.trace_read()
    stage.trace(False)
    if prank == dp - 1:
        stage.loss(reset=True)
    mine = (rank // dp, prank, evs, stage.state_bytes())
    got = [mine]
    if world > 1:
        got = [None] * world
        dist.all_gather_object(got, mine)
    if rank != 0:
        return None
    per_stage = {p + 1: e for (q, p, e, _) in got if q == 0}
    state = [b for (q, p, _, b) in sorted(got, key=lambda x: x[1]) if q == 0]
    meas = TR.measured_trace(plan, per_stage, state_bytes=state, mem_capacity=cfg["cluster"]["mem_capacity"])
    sim_text, _ = planner.simulate_plan_document(plan.doc)
    res = TR.residuals(meas, sim_text)
    out_dir = ROOT / "gpurun_out"
    out_dir.mkdir(exist_ok=True)
    (out_dir / "trace_measured.json").write_text(json.dumps(meas))
    (out_dir / "trace_simulated.json").write_text(sim_text)
    res["events"] = sum(len(u["events"]) for u in meas["units"])
    res["documents"] = "gpurun_out/trace_measured.json, gpurun_out/trace_simulated.json"
    return res


def run_e2e(args, run_step, stage, cfg, e2e_batches, jobs, dev, world, dp, prank, replicas, optimizer, sync_all,
            dist):
    """Public-API step from host buffers: plans solved on a host thread one
    step ahead, token ids H2D from pinned memory, per-step loss D2H."""
    from paper_2509_21275_b200 import planner, schedule
    ahead = {}

    def solve(k):
        lengths = e2e_batches[k][0]
        ahead[k] = schedule.parse_plan(planner.make_plan_document(cfg, lengths, args.slices or None, "main", jobs),
                                       lengths)

    solve(0)    # batch 0's plan is solved during the (untimed) previous step
    h2d = d2h = 0
    # per-step loss: D2H into pinned memory, read one step later (the host
    # enqueues step k+1 before waiting for step k's loss)
    loss_host = torch.zeros((len(e2e_batches), 2), dtype=torch.float64).pin_memory()
    loss_ev = [torch.cuda.Event() for _ in e2e_batches]
    losses = []
    sync_all()
    e0 = time.perf_counter()
    for k in range(len(e2e_batches)):
        th = None
        if k + 1 < len(e2e_batches):
            th = threading.Thread(target=solve, args=(k + 1,))
            th.start()
        st = run_step(k, ahead.pop(k), e2e_batches[k][1])
        h2d += st["h2d_bytes"]
        optimizer()
        if prank == dp - 1:
            stage.loss_async(loss_host[k], reset=True)
            loss_ev[k].record()
            d2h += 16
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
        # slowest rank's wall time; H2D (stage 0) and D2H (last stage) bytes
        # are counted where they happen and summed over ranks
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
    out = {"value": e_tokens / e_s, "unit": "tokens/s", "h2d_bytes_per_step": h2d // nb,
           "d2h_bytes_per_step": d2h // nb}
    if losses:
        out["loss_per_step"] = losses
    return out


# ----------------------------------------------------------------- CPU side --
def cpu_flops_rate(m, sample_tokens: int, threads: int, seed: int = 0):
    """fp32 CPU oracle (oracle/numerics.py) FLOP rate on the benched model:
    fwd+bwd of ONE transformer layer plus the head (final norm, LM head,
    softmax-CE) on one `sample_tokens`-token sequence.  Returns (model FLOP/s,
    seconds): the whole model's step time is then its FLOP count over this
    rate (same model-FLOP accounting as MFU).  Bounded: two layers' worth of
    parameters, not the whole 7B model."""
    from oracle import numerics as O
    torch.set_num_threads(threads)
    spec = O.ModelSpec(m.arch, 1, m.hidden, m.heads, m.kv_heads, m.head_dim, m.ffn, m.vocab,
                       m.rope_theta, m.norm_eps)
    g = torch.Generator().manual_seed(seed)
    params = {}
    for name, shape, kind in O.param_shapes(spec, 0, 1, True, True):
        if kind == "one":
            params[name] = torch.ones(shape)
        elif kind == "zero":
            params[name] = torch.zeros(shape)
        else:
            params[name] = torch.empty(shape).normal_(0, 0.02, generator=g)
    tokens = torch.randint(0, m.vocab, (sample_tokens,), generator=g)
    t0 = time.perf_counter()
    O.whole_batch_grads(spec, params, [tokens])
    dt = time.perf_counter() - t0
    T = sample_tokens
    flops = 3 * (m.linear_flops_per_token_layer() * T + m.attn_flops_per_pair_layer() * T * (T + 1) / 2
                 + 2 * T * m.hidden * m.vocab)
    return flops / dt, dt


def plan_timed(cfg, lengths, jobs, lib):
    from paper_2509_21275_b200 import planner
    t0 = time.perf_counter()
    doc = planner.make_plan_document(cfg, lengths, None, "main", jobs, _lib=lib)
    return doc, time.perf_counter() - t0


def cpu_side(args, m, dp, cfg, tokens_per_step, flops_per_step, lengths, jobs):
    """(cpu_baseline, planner block) on rank 0's host cores: the reference
    planner (oracle/_ref) at jobs = nproc and 1 on the step's lengths, our
    planner likewise, byte identity of all four documents,
    and the fp32 CPU numerics rate of the benched model."""
    from paper_2509_21275_b200 import planner
    cores = os.cpu_count() or 1
    block = {"cores": cores, "sequences": len(lengths)}
    docs = {}
    if REF_SO.exists():
        ref = planner._Api(REF_SO, prefix="epp_ref_")
        docs["ref_jobs_n"], block["reference_seconds_jobs_n"] = plan_timed(cfg, lengths, cores, ref)
        docs["ref_jobs_1"], block["reference_seconds_jobs_1"] = plan_timed(cfg, lengths, 1, ref)
    docs["ours_jobs_n"], block["ours_seconds_jobs_n"] = plan_timed(cfg, lengths, cores, None)
    docs["ours_jobs_1"], block["ours_seconds_jobs_1"] = plan_timed(cfg, lengths, 1, None)
    block["byte_identical"] = len(set(docs.values())) == 1
    block["documents_compared"] = sorted(docs)
    rate, secs = cpu_flops_rate(m, args.cpu_sample_tokens, cores)
    plan_s = block.get("reference_seconds_jobs_n", block["ours_seconds_jobs_n"])
    step_s = plan_s + flops_per_step / rate
    base = {"value": tokens_per_step / step_s, "unit": "tokens/s", "cores": cores,
            "kind": "reference" if REF_SO.exists() else "port",
            "sample": f"reference planner (oracle/_ref make_plan, jobs={cores}) on the step's {len(lengths)} "
                      f"lengths ({plan_s:.3f} s) + the step's model FLOPs ({flops_per_step:.3e}) at the fp32 "
                      f"torch-CPU oracle rate measured on 1 layer + head of {args.model} over a "
                      f"{args.cpu_sample_tokens}-token sample ({rate / 1e9:.1f} GFLOP/s, {secs:.1f} s)"}
    return base, block


def run_reference(args):
    """The reference's CPU path on the host cores (rank 0 only): per step,
    the compiled reference planner (oracle/_ref, jobs = nproc) on the step's
    batch, generated by the reference's own generate_workload, plus the fp32
    CPU numerics of the same model (1 layer + head sample, scaled by model
    FLOPs).  Loads only oracle/ native code."""
    world = args.gpus
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2509_21275_b200 import model as M, planner
    m = M.MODELS[args.model]
    dp = args.pp or world
    cfg, counts, cost_src = bench_config(args, m, dp)
    cores = os.cpu_count() or 1
    if not REF_SO.exists():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libepp_ref.so not built"}))
        return
    ref = planner._Api(REF_SO, prefix="epp_ref_")
    batches = make_lengths(args, args.warmup + args.steps, dp, _lib=ref)
    times, toks, plan_ts = [], [], []
    for i, (_, lengths) in enumerate(batches):
        doc, plan_s = plan_timed(cfg, lengths, cores, ref)
        flops = step_flops_from_doc(m, doc)
        rate, secs = cpu_flops_rate(m, args.cpu_sample_tokens, cores, seed=i)
        if i >= args.warmup:
            times.append(plan_s + flops / rate)
            toks.append(sum(lengths))
            plan_ts.append(plan_s)
    value = sum(toks) / sum(times)
    sample = (f"per step: reference planner (oracle/_ref, jobs={cores}) on the step's {len(batches[0][1])} "
              f"lengths (mean {statistics.mean(plan_ts):.3f} s) + the step's model FLOPs at the fp32 torch-CPU "
              f"oracle rate measured that step on 1 layer + head of {args.model} over a "
              f"{args.cpu_sample_tokens}-token sample")
    out = {"metric": METRIC, "impl": "reference",
           "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f32", "data": DATA,
           "config": {"workload": f"{args.model} EPP, {args.preset} lengths cap {args.cap}, "
                                  f"{args.seqs_per_gpu} seqs/GPU/step, d_p={dp}",
                      "model": args.model, "parallelism": f"pp{dp}", "stage_layers": counts,
                      "cost": cost_src, "same_config_as_ours": True},
           "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "reference",
                            "sample": sample},
           "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def step_flops_from_doc(m, doc):
    """Model FLOPs of a plan document's chunks (same count as step_flops)."""
    d = json.loads(doc)
    lin, per_pair = m.linear_flops_per_token_layer(), m.attn_flops_per_pair_layer()
    total = 0.0
    for c in d["chunks"]:
        sl = c["slices"]
        T = sum(sl)
        pairs = sum(s * (c["context"] if (i == 0 and "seq" in c) else 0) + s * (s + 1) / 2 for i, s in enumerate(sl))
        total += 3 * (m.layers * (lin * T + per_pair * pairs) + 2 * T * m.hidden * m.vocab)
    return total


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
