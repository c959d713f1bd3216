"""Two processes sharing cuda:0, one CUDA stage each, driven by
DistributedPipeline over the C-ABI P2P channels (include/epp_gpu.h
epp_p2p_*: CUDA IPC mailboxes + stream-ordered flags; on the 8-GPU box the
same code stores over NVLink).  torch.distributed (gloo) only exchanges the
channel handles.  Loss, every per-chunk loss and every parameter gradient are
BIT-identical to the single-process LocalPipeline's, in fp32 and bf16, with a
head-balanced (non-uniform) stage split and an active checkpoint ladder —
except embed.weight, whose backward scatters with float atomics (order-
dependent in the last bit; checked at 1e-6)."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from oracle import numerics as O
from paper_2509_21275_b200 import model as M
from paper_2509_21275_b200 import schedule as S
from paper_2509_21275_b200.executor import DistributedPipeline, LocalPipeline, stage_layers

pytestmark = pytest.mark.gpu

MODEL = M.ModelConfig("t", "llama", layers=4, hidden=256, heads=4, kv_heads=2, ffn=384, vocab=512)
LENGTHS = [900, 37, 210, 90, 5, 64, 380, 1500]
COUNTS = [3, 1]     # head-balanced (non-uniform) stage split


def spec():
    m = MODEL
    return O.ModelSpec(m.arch, m.layers, m.hidden, m.heads, m.kv_heads, m.head_dim, m.ffn, m.vocab,
                       m.rope_theta, m.norm_eps)


def plan_doc(world, tight=False):
    from paper_2509_21275_b200 import planner
    cfg = M.planner_config(MODEL, world, mem_capacity=1e12, reserve_bytes=0)
    if not tight:
        return planner.make_plan_document(cfg, LENGTHS, 3, "main", 1)
    act = cfg["model"]["token_act_bytes"]
    for tokens_fit in (3000, 2500, 2000, 1500, 1200, 1000, 800):
        cfg["cluster"]["mem_capacity"] = max(cfg["model"]["stage_state_bytes"]) + act * tokens_fit / world
        doc = planner.make_plan_document(cfg, LENGTHS, 3, "main", 1)
        if any(any(v for row in u.ckpt for v in row) for u in S.parse_plan(doc, LENGTHS).units):
            return doc
    raise AssertionError("no budget activates the ladder")


def make_stage(rank, world, dtype, params):
    from paper_2509_21275_b200.gpu import CudaStage
    first, num = stage_layers(MODEL.layers, world, rank, COUNTS)
    st = CudaStage(MODEL, first, num, rank == 0, rank == world - 1, dtype=dtype,
                   plan_stage_layers=MODEL.layers // world)
    st.load_weights(params)
    return st


def worker(rank, world, port, doc, dtype, q):
    from paper_2509_21275_b200.gpu import CudaStage
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    plan = S.parse_plan(doc, LENGTHS)
    params = O.init_params(spec(), seed=5)
    st = make_stage(rank, world, dtype, params)
    max_tokens = max(c.tokens for c in plan.chunks.values())
    drv = DistributedPipeline(st, rank, world, torch.device("cuda"), MODEL.hidden,
                              torch.float32 if dtype == "f32" else torch.bfloat16, max_tokens=max_tokens)
    assert drv.p2p and drv.ch, "CUDA stages must use the C-ABI P2P channels"
    drv.run_step(plan, S.synthetic_tokens(LENGTHS, MODEL.vocab, seed=13))
    torch.cuda.synchronize()
    grads = {k: v.cpu().numpy().copy() for k, v in st.grads().items()}   # by value
    loss = st.loss() if rank == world - 1 else None
    chunk = {cid: st.chunk_loss(cid) for cid in plan.chunks} if rank == world - 1 else None
    stats = {k: c.stats() for k, c in drv.ch.items()}
    q.put((rank, grads, loss, chunk, drv.p2p_bytes, stats))
    drv.close()
    torch.distributed.barrier()
    torch.distributed.destroy_process_group()


def collect(q, procs, n, timeout=600):
    """n results from the workers; fails fast when a worker died."""
    import queue
    import time
    out, t0 = [], time.time()
    while len(out) < n:
        try:
            out.append(q.get(timeout=5))
        except queue.Empty:
            dead = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
            if dead or time.time() - t0 > timeout:
                for p in procs:
                    p.kill()
                raise AssertionError(f"worker failed (exit codes {dead})" if dead else "workers timed out")
    return out


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("dtype,tight", [("f32", False), ("bf16", False), ("bf16", True)])
def test_two_rank_cuda_pipeline_matches_local(dtype, tight):
    world = 2
    doc = plan_doc(world, tight)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, doc, dtype, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = collect(q, procs, world)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    plan = S.parse_plan(doc, LENGTHS)
    dist_grads, loss, chunk = {}, None, None
    expect = sum(c.tokens for c in plan.chunks.values()) * MODEL.hidden * (4 if dtype == "f32" else 2)
    for rank, g, ls, ck, nbytes, stats in results:
        dist_grads.update({k: torch.from_numpy(v) for k, v in g.items()})
        # every chunk crosses the stage boundary once forward, once backward
        assert nbytes == expect, (nbytes, expect)
        for k, (n, b) in stats.items():
            assert n == len(plan.chunks) and b == expect, (k, n, b)
        if rank == world - 1:
            loss, chunk = ls, ck
    params = O.init_params(spec(), seed=5)
    stages = [make_stage(p, world, dtype, params) for p in range(world)]
    LocalPipeline(stages, torch.device("cuda")).run_step(plan, S.synthetic_tokens(LENGTHS, MODEL.vocab, seed=13))
    torch.cuda.synchronize()
    local = {}
    for st in stages:
        local.update({k: v.cpu() for k, v in st.grads().items()})
    assert loss == stages[-1].loss()
    assert chunk == {cid: stages[-1].chunk_loss(cid) for cid in plan.chunks}
    for k, v in local.items():
        if k == "embed.weight":
            assert float((dist_grads[k] - v).norm() / v.norm()) < 1e-6
        else:
            assert torch.equal(dist_grads[k], v), (k, float((dist_grads[k] - v).abs().max()))


def test_p2p_channel_roundtrip():
    """The copying forms epp_p2p_send / epp_p2p_recv inside one process
    (raw-pointer mapping): a ring of 5 variable-size messages through a
    2-message arena, wrapping and waiting on releases; payloads arrive
    intact and in order."""
    from paper_2509_21275_b200.gpu import P2PChannel, p2p_init
    p2p_init([0])
    rx = P2PChannel("recv", 3 << 20)
    tx = P2PChannel("send")
    rx.open(tx.handle)
    tx.open(rx.handle)
    sizes = [1 << 20, 700_000, 1 << 20, 123_456, 2_000_000]
    for i, n in enumerate(sizes):
        src = torch.arange(n // 4, device="cuda", dtype=torch.int32) * (i + 1)
        dst = torch.empty_like(src)
        tx.send(src)
        rx.recv(dst)
        torch.cuda.synchronize()
        assert torch.equal(src, dst), i
    assert tx.stats() == (len(sizes), sum(n // 4 * 4 for n in sizes))
    with pytest.raises(Exception, match="larger than the channel"):
        tx.send(torch.empty(4 << 20, device="cuda", dtype=torch.uint8))
    rx.close()
    tx.close()


LENGTHS_R1 = [300, 44, 610, 17, 128]


def dp_worker(rank, world, port, docs, zero, q):
    from paper_2509_21275_b200.executor import GradSync, LocalPipeline
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    group = torch.distributed.new_group(list(range(world)))
    lengths = (LENGTHS, LENGTHS_R1)[rank]
    plan = S.parse_plan(docs[rank], lengths)
    params = O.init_params(spec(), seed=5)
    from paper_2509_21275_b200.gpu import CudaStage
    st = CudaStage(MODEL, 0, MODEL.layers, True, True, dtype="f32")
    st.load_weights(params)
    sync = GradSync(st, group, world, zero=zero)
    LocalPipeline([st], torch.device("cuda")).run_step(plan, S.synthetic_tokens(lengths, MODEL.vocab, seed=21 + rank),
                                                       total_targets=targets_all())
    sync.launch()
    sync.finish()
    grads = st.arena()["grad"].cpu().numpy().copy()
    st.adamw_step(1e-3, 1)
    sync.after_step()
    torch.cuda.synchronize()
    q.put((rank, grads, st.arena()["master"].cpu().numpy().copy(), sync.state_numel))
    torch.distributed.barrier()
    torch.distributed.destroy_process_group()


def targets_all():
    return sum(max(0, n - 1) for n in LENGTHS + LENGTHS_R1)


@pytest.mark.parametrize("zero", [False, True])
def test_data_parallel_gradsync(zero):
    """dp 2 (two processes on cuda:0): bucketed gradient reduction over the
    stage arenas (GradSync) after a step normalised by the global batch's
    targets, then AdamW (ZeRO-1: each replica updates its half of every
    bucket and the masters are all-gathered).  Equals one process running
    both batches into one stage and stepping once."""
    from paper_2509_21275_b200 import planner
    from paper_2509_21275_b200.gpu import CudaStage
    world = 2
    cfg = M.planner_config(MODEL, 1, mem_capacity=1e12, reserve_bytes=0)
    docs = [planner.make_plan_document(cfg, LENGTHS, 3, "main", 1),
            planner.make_plan_document(cfg, LENGTHS_R1, 3, "main", 1)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=dp_worker, args=(r, world, port, docs, zero, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = sorted(collect(q, procs, world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    params = O.init_params(spec(), seed=5)
    st = CudaStage(MODEL, 0, MODEL.layers, True, True, dtype="f32")
    st.load_weights(params)
    drv = LocalPipeline([st], torch.device("cuda"))
    for r, lengths in enumerate((LENGTHS, LENGTHS_R1)):
        drv.run_step(S.parse_plan(docs[r], lengths), S.synthetic_tokens(lengths, MODEL.vocab, seed=21 + r),
                     total_targets=targets_all())
    ref_grad = st.arena()["grad"].cpu()
    st.adamw_step(1e-3, 1)
    ref_master = st.arena()["master"].cpu()
    full = ref_master.numel()
    for rank, g, m, state in results:
        g, m = torch.from_numpy(g), torch.from_numpy(m)
        if not zero:
            assert float((g - ref_grad).norm() / ref_grad.norm()) < 1e-6
        assert float((m - ref_master).norm() / ref_master.norm()) < 1e-6, rank
        assert state == (full // 2 if zero else full)
    assert torch.equal(torch.from_numpy(results[0][2]), torch.from_numpy(results[1][2]))
    st.close()
