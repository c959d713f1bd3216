"""Two processes sharing cuda:0, one CUDA stage each, driven by
DistributedPipeline over gloo (messages staged through host memory; on a
multi-GPU box the same driver sends device tensors over NCCL).  Loss and
every parameter gradient equal the single-process LocalPipeline's (fp32)."""
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


def plan_doc(world):
    from paper_2509_21275_b200 import planner
    cfg = M.planner_config(MODEL, world, mem_capacity=1e12, reserve_bytes=0)
    return planner.make_plan_document(cfg, LENGTHS, 3, "main", 1)


def worker(rank, world, port, doc, q):
    from paper_2509_21275_b200.gpu import CudaStage
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    plan = S.parse_plan(doc, LENGTHS)
    params = O.init_params(spec(), seed=5)
    first, num = stage_layers(MODEL.layers, world, rank, COUNTS)
    st = CudaStage(MODEL, first, num, rank == 0, rank == world - 1, dtype="f32")
    st.load_weights(params)
    drv = DistributedPipeline(st, rank, world, torch.device("cuda"), MODEL.hidden, torch.float32)
    drv.run_step(plan, S.synthetic_tokens(LENGTHS, MODEL.vocab, seed=13))
    torch.cuda.synchronize()
    grads = {k: v.cpu().numpy().copy() for k, v in st.grads().items()}   # by value
    loss = st.loss()[0] if rank == world - 1 else None
    q.put((rank, grads, loss, drv.p2p_bytes))
    torch.distributed.barrier()
    torch.distributed.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_cuda_pipeline_matches_local():
    from paper_2509_21275_b200.gpu import CudaStage
    world = 2
    doc = plan_doc(world)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, doc, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    dist_grads, loss = {}, None
    for rank, g, ls, nbytes in results:
        dist_grads.update({k: torch.from_numpy(v) for k, v in g.items()})
        assert nbytes > 0
        if rank == world - 1:
            loss = ls
    plan = S.parse_plan(doc, LENGTHS)
    params = O.init_params(spec(), seed=5)
    stages = []
    for p in range(world):
        st = CudaStage(MODEL, *stage_layers(MODEL.layers, world, p, COUNTS), p == 0, p == world - 1, dtype="f32")
        st.load_weights(params)
        stages.append(st)
    LocalPipeline(stages, torch.device("cuda")).run_step(plan, S.synthetic_tokens(LENGTHS, MODEL.vocab, seed=13))
    torch.cuda.synchronize()
    local = {}
    for st in stages:
        local.update({k: v.cpu() for k, v in st.grads().items()})
    ref_loss = stages[-1].loss()[0]
    assert abs(loss - ref_loss) <= 1e-5 * abs(ref_loss)
    for k, v in local.items():
        err = float((dist_grads[k] - v).norm() / (v.norm() + 1e-30))
        assert err < 1e-5, (k, err)
