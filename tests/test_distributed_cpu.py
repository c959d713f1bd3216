"""World-size-2 gloo run of the one-stage-per-rank executor
(DistributedPipeline) on CPU, with the oracle's TorchStage standing in for
the CUDA stage: gradients equal the single-process LocalPipeline's."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from oracle import numerics as O
from paper_2509_21275_b200 import model as M
from paper_2509_21275_b200 import schedule as S
from paper_2509_21275_b200.executor import DistributedPipeline, LocalPipeline, stage_layers

MODEL = M.ModelConfig("t", "gpt", layers=4, hidden=64, heads=4, kv_heads=4, ffn=128, vocab=256)
LENGTHS = [300, 37, 21, 90, 5, 64, 180]


def spec():
    m = MODEL
    return O.ModelSpec(m.arch, m.layers, m.hidden, m.heads, m.kv_heads, m.head_dim, m.ffn, m.vocab)


def plan_doc(world):
    from paper_2509_21275_b200 import planner
    cfg = M.planner_config(MODEL, world, mem_capacity=1e12, reserve_bytes=0)
    return planner.make_plan_document(cfg, LENGTHS, 3, "main", 1)


def counts_for(world):
    # head-balanced (non-uniform) split for world 2: the last stage gets fewer layers
    return [3, 1] if world == 2 else None


class ClaimsP2P(O.TorchStage):
    """A CPU stage that claims the C-ABI P2P transport: opening the channels
    fails here (no GPU), so every rank must fall back to torch.distributed
    together."""
    supports_p2p = True


def worker(rank, world, port, doc, q, claim_p2p=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    plan = S.parse_plan(doc, LENGTHS)
    params = O.init_params(spec(), seed=3)
    first, num = stage_layers(MODEL.layers, world, rank, counts_for(world))
    cls = ClaimsP2P if claim_p2p else O.TorchStage
    st = cls(spec(), params, first, num, rank == 0, rank == world - 1)
    drv = DistributedPipeline(st, rank, world, torch.device("cpu"), MODEL.hidden, torch.float32)
    if claim_p2p:
        assert not drv.p2p and drv.transport.startswith("torch.distributed (P2P channels failed"), drv.transport
    drv.run_step(plan, S.synthetic_tokens(LENGTHS, MODEL.vocab, seed=11))
    # by value (numpy): shared-memory tensors would vanish with the exiting worker
    q.put((rank, {k: v.numpy().copy() for k, v in st.grads().items()}, float(st.loss_sum), drv.p2p_bytes))
    torch.distributed.barrier()
    torch.distributed.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,claim_p2p", [(2, False), (4, False), (2, True)])
def test_gloo_pipeline_matches_local(world, claim_p2p):
    doc = plan_doc(world)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, doc, q, claim_p2p)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    dist_grads = {}
    loss = None
    for rank, g, ls, nbytes in results:
        dist_grads.update({k: torch.from_numpy(v) for k, v in g.items()})
        if rank == world - 1:
            loss = ls
        if 0 < rank < world - 1:
            assert nbytes > 0
    plan = S.parse_plan(doc, LENGTHS)
    params = O.init_params(spec(), seed=3)
    stages = [O.TorchStage(spec(), params, *stage_layers(MODEL.layers, world, p, counts_for(world)), p == 0,
                           p == world - 1)
              for p in range(world)]
    LocalPipeline(stages, torch.device("cpu")).run_step(plan, S.synthetic_tokens(LENGTHS, MODEL.vocab, seed=11))
    local = {}
    for st in stages:
        local.update(st.grads())
    assert abs(loss - stages[-1].loss_sum) < 1e-4
    for k, v in local.items():
        assert torch.allclose(dist_grads[k], v, rtol=1e-5, atol=1e-8), k


LENGTHS_B = [120, 260, 33, 75, 9, 140]


def dp_worker(rank, world, pp, port, docs, q):
    from paper_2509_21275_b200.executor import GradSync, pipeline_groups
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    replicas = world // pp
    pipes, dp_groups = pipeline_groups(pp, replicas)
    replica, p = rank // pp, rank % pp
    lengths = (LENGTHS, LENGTHS_B)[replica]
    plan = S.parse_plan(docs[replica], lengths)
    params = O.init_params(spec(), seed=3)
    first, num = stage_layers(MODEL.layers, pp, p)
    st = O.TorchStage(spec(), params, first, num, p == 0, p == pp - 1)
    drv = DistributedPipeline(st, p, pp, torch.device("cpu"), MODEL.hidden, torch.float32, pipe=pipes[replica])
    sync = GradSync(st, dp_groups[p], replicas)
    drv.run_step(plan, S.synthetic_tokens(lengths, MODEL.vocab, seed=11 + replica), total_targets=global_targets())
    sync.launch()
    sync.finish()
    q.put((rank, {k: v.numpy().copy() for k, v in st.grads().items()}))   # by value: the worker exits
    torch.distributed.barrier()
    torch.distributed.destroy_process_group()


def global_targets():
    return sum(max(0, n - 1) for n in LENGTHS + LENGTHS_B)


def test_gloo_pipeline_data_parallel_replicas():
    """pp 2 x dp 2: each replica pipelines its own batch with the loss
    normalised by the targets of the WHOLE global batch, then the stage
    gradients are summed across replicas (GradSync): the global per-token
    mean, whatever each replica's share of targets."""
    from paper_2509_21275_b200 import planner
    pp, world = 2, 4
    cfg = M.planner_config(MODEL, pp, mem_capacity=1e12, reserve_bytes=0)
    docs = [planner.make_plan_document(cfg, LENGTHS, 3, "main", 1),
            planner.make_plan_document(cfg, LENGTHS_B, 3, "main", 1)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=dp_worker, args=(r, world, pp, port, docs, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = {r: {k: torch.from_numpy(v) for k, v in g.items()} for r, g in (q.get(timeout=300) for _ in range(world))}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # reference: each replica's batch through a local pipeline, grads averaged
    ref = {}
    for replica, lengths in enumerate((LENGTHS, LENGTHS_B)):
        params = O.init_params(spec(), seed=3)
        stages = [O.TorchStage(spec(), params, *stage_layers(MODEL.layers, pp, p), p == 0, p == pp - 1)
                  for p in range(pp)]
        LocalPipeline(stages, torch.device("cpu")).run_step(S.parse_plan(docs[replica], lengths),
                                                           S.synthetic_tokens(lengths, MODEL.vocab, seed=11 + replica),
                                                           total_targets=global_targets())
        for st in stages:
            for k, v in st.grads().items():
                ref[k] = ref.get(k, 0) + v
    for rank in range(world):
        p = rank % pp
        for k, v in results[rank].items():
            assert torch.allclose(v, ref[k], rtol=1e-5, atol=1e-8), (rank, k)
    # both replicas of a stage hold identical summed gradients
    for p in range(pp):
        for k in results[p]:
            assert torch.equal(results[p][k], results[pp + p][k])
