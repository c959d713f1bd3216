"""Replays a plan document on stage executors — the EPP training step.

    plan_{i} = planner.make_plan(lengths_i)        (CPU, can be pre-solved)
    for unit in plan.units:                        (sequential 1F1B pipelines,
        every stage runs stage_ops(...)             gradient-accumulated)
    optimizer step on every stage

Two drivers share the op-list logic (schedule.stage_ops):
  * LocalPipeline — every stage in this process (one GPU running d_p stages,
    or the d_p = 1 single-GPU configuration); ops are issued in a
    dependency-respecting round robin over the stages' op lists.
  * DistributedPipeline — one stage per rank (torch.distributed, NCCL on
    B200s, gloo in the CPU tests).  Activations go p -> p+1 and gradients
    p+1 -> p over two separate process groups per adjacent pair, so the
    forward and backward streams of messages can never block each other;
    both sides derive every message size from the plan, no handshake.

A stage is any object with forward(chunk, act_in) / backward(chunk, grad_in)
(gpu.CudaStage on the product path).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

from .schedule import ChunkLayout, Plan, chunk_token_arrays, stage_ops


@dataclass
class ChunkOp:
    """Per-(stage, chunk) call arguments (mirrors epp_chunk_desc)."""
    id: int
    seq: int
    kind: int
    tail: bool
    context: int
    seq_len: int
    slices: List[int]
    ckpt_layers: int
    loss_scale: float
    token_ids: Optional[torch.Tensor]
    target_ids: Optional[torch.Tensor]


def stage_layers(layers: int, pp_degree: int, stage: int, counts: Optional[Sequence[int]] = None):
    """(first layer, count) of 0-based `stage`: contiguous blocks, L/d_p each
    (proj/src/config.cpp:25-26 requires L % d_p == 0) unless explicit
    per-stage `counts` (balanced_stage_counts) are given."""
    if counts is None:
        per = layers // pp_degree
        return stage * per, per
    assert len(counts) == pp_degree and sum(counts) == layers
    return sum(counts[:stage]), counts[stage]


def balanced_stage_counts(layers: int, pp_degree: int, head_layers: float) -> List[int]:
    """Layers per stage when the last stage also runs the LM head and
    cross-entropy, worth `head_layers` transformer layers of work: start from
    the uniform split and move single layers from the most to the least
    loaded stage while that lowers the pipeline's bottleneck stage.  The
    planner still prices uniform stages (its contract); the executor's memory
    model is made conservative for the largest stage (model.planner_config)."""
    counts = [layers // pp_degree] * pp_degree
    if pp_degree == 1:
        return counts

    def load(i):
        return counts[i] + (head_layers if i == pp_degree - 1 else 0.0)

    while True:
        hi = max(range(pp_degree), key=load)
        lo = min(range(pp_degree), key=load)
        if counts[hi] <= 1 or load(lo) + 1 >= load(hi):
            return counts
        counts[hi] -= 1
        counts[lo] += 1


class _ChunkTokens:
    """Token ids / targets of every chunk of a step, staged from pinned host
    memory to the device (counted as the step's H2D bytes)."""

    def __init__(self, plan: Plan, tokens: Sequence[np.ndarray], device: torch.device, need_ids: bool,
                 need_targets: bool):
        self.ids: Dict[int, torch.Tensor] = {}
        self.tgt: Dict[int, torch.Tensor] = {}
        self.h2d_bytes = 0
        pin = device.type == "cuda"
        for cid, lay in plan.chunks.items():
            ids, tgt = chunk_token_arrays(lay, tokens)
            if need_ids:
                t = torch.from_numpy(ids)
                if pin:
                    t = t.pin_memory()
                self.ids[cid] = t.to(device, non_blocking=True)
                self.h2d_bytes += t.numel() * 4
            if need_targets:
                t = torch.from_numpy(tgt)
                if pin:
                    t = t.pin_memory()
                self.tgt[cid] = t.to(device, non_blocking=True)
                self.h2d_bytes += t.numel() * 4


def _op(plan: Plan, unit, pos: int, stage: int, toks: _ChunkTokens, total_targets: Optional[int] = None) -> ChunkOp:
    """total_targets: the loss normaliser (default: this plan's targets; with
    data-parallel replicas, the targets of the whole global batch, so the
    summed replica gradients are the global per-token mean)."""
    lay: ChunkLayout = plan.chunks[unit.chunks[pos]]
    n = plan.total_targets if total_targets is None else total_targets
    return ChunkOp(lay.id, lay.seq, lay.kind, lay.tail, lay.context, lay.seq_len, lay.slices,
                   unit.ckpt[stage][pos], 1.0 / max(1, n),
                   toks.ids.get(lay.id), toks.tgt.get(lay.id))


class LocalPipeline:
    def __init__(self, stages: Sequence, device: torch.device):
        self.stages = list(stages)
        self.device = device

    def run_step(self, plan: Plan, tokens: Sequence[np.ndarray], staged: Optional[_ChunkTokens] = None,
                 total_targets: Optional[int] = None) -> dict:
        """One global batch.  `staged`: token tensors already on the device
        (the device-resident benchmark mode); otherwise they are copied from
        pinned host memory here.  total_targets: see _op."""
        dp = len(self.stages)
        if dp != plan.pp_degree:
            raise ValueError(f"plan is for {plan.pp_degree} stages, executor has {dp}")
        toks = staged or _ChunkTokens(plan, tokens, self.device, True, True)
        self._targets = total_targets
        for unit in plan.units:
            self._run_unit(plan, unit, toks)
        return {"h2d_bytes": toks.h2d_bytes}

    def _run_unit(self, plan: Plan, unit, toks: _ChunkTokens):
        dp = len(self.stages)
        n = len(unit.chunks)
        order = unit.backward_order
        ops = [stage_ops(n, unit.n_prefill, dp, p + 1, order) for p in range(dp)]
        idx = [0] * dp
        acts: Dict[tuple, torch.Tensor] = {}
        grads: Dict[tuple, torch.Tensor] = {}
        remaining = sum(len(o) for o in ops)
        while remaining:
            progressed = False
            for p in range(dp):
                while idx[p] < len(ops[p]):
                    kind, pos = ops[p][idx[p]]
                    if kind == "F":
                        if p > 0 and (p - 1, pos) not in acts:
                            break
                        act_in = acts.pop((p - 1, pos)) if p > 0 else None
                        out = self.stages[p].forward(_op(plan, unit, pos, p, toks, self._targets), act_in)
                        if p + 1 < dp:
                            acts[(p, pos)] = out
                    else:
                        if p + 1 < dp and (p + 1, pos) not in grads:
                            break
                        g_in = grads.pop((p + 1, pos)) if p + 1 < dp else None
                        g_out = self.stages[p].backward(_op(plan, unit, pos, p, toks, self._targets), g_in)
                        if p > 0:
                            grads[(p, pos)] = g_out
                    idx[p] += 1
                    remaining -= 1
                    progressed = True
            if not progressed:
                raise RuntimeError("pipeline op lists deadlocked (plan/op-list mismatch)")


def pipeline_groups(pp: int, replicas: int = 1):
    """Process groups of `replicas` data-parallel copies of a `pp`-stage
    pipeline (global rank = replica * pp + stage).  Collective: every rank
    calls it with the same arguments (torch's new_group is).

    Returns (pipes, dp_groups): pipes[q] = (ranks, fwd_groups, bwd_groups) of
    replica q, one group per adjacent stage pair and direction; dp_groups[p]
    = the group of stage p across replicas (None without replicas)."""
    import torch.distributed as dist
    pipes = []
    for q in range(replicas):
        ranks = [q * pp + p for p in range(pp)]
        fwd, bwd = [], []
        for p in range(pp - 1):
            fwd.append(dist.new_group([ranks[p], ranks[p + 1]]))
            bwd.append(dist.new_group([ranks[p], ranks[p + 1]]))
        pipes.append((ranks, fwd, bwd))
    dp_groups = [dist.new_group([q * pp + p for q in range(replicas)]) if replicas > 1 else None
                 for p in range(pp)]
    return pipes, dp_groups


class GradSync:
    """Data-parallel gradient reduction of one stage across its replicas
    (the paper's data parallelism across pipeline replicas).

    * Gradients are SUMMED: every replica normalises its loss by the targets
      of the whole global batch (run_step(total_targets=...)), so the sum is
      the global per-token mean whatever each replica's share of targets.
    * CUDA stages: one collective per bucket (embedding | layer | head, each a
      contiguous arena range, include/epp_gpu.h), issued on a side stream in
      readiness order (head, last layer, ..., first layer, embedding) right
      after the step's last backward has been ENQUEUED; each waits only for
      its bucket's event, so reducing layer j overlaps the backward of the
      layers below it.  finish() makes the compute stream wait for all.
    * zero=True (ZeRO-1): reduce-scatter instead of all-reduce, Adam state
      only for this replica's 1/R slice of every bucket (epp_stage_opt_shard),
      and after the optimizer step the updated fp32 masters are all-gathered
      and the working copies re-derived (after_step).
    * Other stages (the CPU oracle stages of the gloo tests): one all-reduce
      per gradient tensor, no overlap (zero is ignored: no optimizer there).
    gloo groups (the 2-processes-on-one-GPU tests) reduce-scatter via an
    all-reduce and all-gather via a list; NCCL uses the native collectives."""

    def __init__(self, stage, group, replicas: int, zero: bool = False):
        import torch.distributed as dist
        self.dist, self.stage, self.group, self.R = dist, stage, group, int(replicas)
        self.active = group is not None and self.R > 1
        self.rank = dist.get_rank(group) if self.active else 0
        self.cuda = hasattr(stage, "arena")
        self.zero = bool(zero) and self.cuda and self.active
        self.works = []
        self.native = self.active and dist.get_backend(group) == "nccl"
        if self.cuda:
            a = stage.arena()
            self.grad, self.master = a["grad"], a["master"]
            self.off = stage.buckets()
            stage.grad_events(True)
            self.side = torch.cuda.Stream(device=stage.device)
            self.state_numel = stage.opt_shard(self.rank, self.R) if self.zero else self.master.numel()

    def _slice(self, t: torch.Tensor) -> torch.Tensor:
        n = t.numel() // self.R
        return t[self.rank * n:(self.rank + 1) * n]

    def launch(self) -> None:
        """Issue the reductions; call right after the stage's last backward of
        the step was enqueued (e.g. after run_step returned)."""
        if not self.active:
            return
        if not self.cuda:
            for t in self.stage.grad_views().values():
                self.dist.all_reduce(t, group=self.group)
            return
        with torch.cuda.stream(self.side):
            for b in reversed(range(len(self.off) - 1)):
                self.stage.bucket_wait(b, self.side)
                g = self.grad[self.off[b]:self.off[b + 1]]
                if self.zero and self.native:
                    w = self.dist.reduce_scatter_tensor(self._slice(g), g, group=self.group, async_op=True)
                else:
                    w = self.dist.all_reduce(g, group=self.group, async_op=True)
                self.works.append(w)

    def finish(self) -> None:
        """The current stream waits for every reduction (before the optimizer)."""
        for w in self.works:
            w.wait()
        self.works = []

    def after_step(self) -> None:
        """ZeRO-1: all-gather the updated master slices, then re-derive the
        working copies."""
        if not self.zero:
            return
        for b in range(len(self.off) - 1):
            m = self.master[self.off[b]:self.off[b + 1]]
            mine = self._slice(m)
            if self.native:
                self.dist.all_gather_into_tensor(m, mine, group=self.group)
            else:
                parts = list(m.chunk(self.R))
                self.dist.all_gather(parts, mine.clone(), group=self.group)
                m.copy_(torch.cat(parts))
        self.stage.sync_weights()


def allreduce_grads(stage, group, replicas: int) -> None:
    """Blocking per-tensor sum of one stage's gradients over its replicas
    (the un-bucketed baseline; GradSync is the overlapped path)."""
    if group is None or replicas <= 1:
        return
    import torch.distributed as dist
    for t in stage.grad_views().values():
        dist.all_reduce(t, group=group)


class DistributedPipeline:
    """One stage per rank (rank = stage) of a pipeline.

    Transport:
      * CUDA stages (gpu.CudaStage): the C-ABI P2P channels over peer memory
        (include/epp_gpu.h epp_p2p_*; NVLink between the 8 B200s, CUDA IPC
        between processes).  The sending stage's last kernel stores its
        output straight into the receiver's mailbox, the receiver copies an
        activation into its own input buffer (a gradient is read in place)
        and releases the slot; all waits are stream-ordered, the host never
        blocks, nothing stays alive after the call that consumed it.
        torch.distributed only exchanges the channel handles at setup.
      * other stages (the CPU oracle stages in the gloo tests):
        torch.distributed isend / irecv, two groups per adjacent pair so the
        forward and backward message streams never block each other.
    Both sides derive every message size from the plan, no handshake.
    `pipe` = (global ranks of the stages, fwd groups, bwd groups) from
    pipeline_groups(); by default the whole world is one pipeline.
    `max_tokens`: the largest chunk any plan will send (sizes the mailboxes:
    two such messages per channel)."""

    def __init__(self, stage, rank: int, world: int, device: torch.device, hidden: int,
                 act_dtype: torch.dtype, pipe=None, max_tokens: int = 0):
        import torch.distributed as dist
        self.dist = dist
        self.stage, self.rank, self.world = stage, rank, world
        self.device, self.hidden, self.act_dtype = device, hidden, act_dtype
        if pipe is None:
            (pipe,), _ = pipeline_groups(world, 1)
        self.ranks, self.fwd_groups, self.bwd_groups = pipe
        self.p2p_bytes = 0
        self.p2p = bool(getattr(stage, "supports_p2p", False))
        self.ch = {}
        self.transport = "torch.distributed"
        if self.p2p:
            # every rank must agree on the transport: if any endpoint cannot
            # map its peer (e.g. no CUDA IPC between the two processes), all
            # ranks use torch.distributed (NCCL) send / recv instead
            err = self._open_channels(max_tokens)
            errs = [None] * self.dist.get_world_size()
            self.dist.all_gather_object(errs, err)
            bad = [e for e in errs if e]
            if bad:
                import sys
                print(f"epp: P2P channels unavailable ({bad[0]}); stage transfers use torch.distributed",
                      file=sys.stderr)
                self.close()
                self.p2p = False
                self.transport = f"torch.distributed (P2P channels failed: {bad[0]})"
            else:
                self.transport = "epp_p2p channels (peer memory)"

    def _open_channels(self, max_tokens: int) -> str:
        """Endpoints: 'fin' (activations from p-1), 'fout' (to p+1), 'bin'
        (gradients from p+1), 'bout' (to p-1).  Receivers own the arenas.
        Every rank takes part in the handle exchange even if its own
        endpoints failed; returns this rank's error ('' = fine)."""
        from .gpu import P2PChannel
        p, dp = self.rank, self.world
        err = ""
        try:
            esz = torch.tensor([], dtype=self.act_dtype).element_size()
            arena = 2 * max(1, int(max_tokens)) * self.hidden * esz
            if p > 0:
                self.ch["fin"] = P2PChannel("recv", arena)
                self.ch["bout"] = P2PChannel("send")
            if p + 1 < dp:
                self.ch["fout"] = P2PChannel("send")
                self.ch["bin"] = P2PChannel("recv", arena)
            mine = {k: c.handle for k, c in self.ch.items()}
        except Exception as e:  # noqa: BLE001
            err, mine = f"{type(e).__name__}: {e}", None
        got = [None] * self.dist.get_world_size()
        self.dist.all_gather_object(got, (self.ranks[p], mine))
        by_rank = {r: h for (r, h) in got}
        if err:
            return err
        peer = {"fin": (p - 1, "fout"), "bout": (p - 1, "bin"), "fout": (p + 1, "fin"), "bin": (p + 1, "bout")}
        try:
            for k, c in self.ch.items():
                q, their = peer[k]
                h = by_rank[self.ranks[q]]
                if h is None:
                    return f"stage {q} has no P2P endpoints"
                c.open(h[their])
        except Exception as e:  # noqa: BLE001
            return f"{type(e).__name__}: {e}"
        return ""

    def close(self):
        for c in self.ch.values():
            c.close()
        self.ch = {}

    # -- torch.distributed transport (CPU oracle stages) ----------------------
    def _recv(self, T: int, src: int, group) -> torch.Tensor:
        buf = torch.empty((T, self.hidden), dtype=self.act_dtype, device=self.device)
        self.dist.irecv(buf, src=src, group=group).wait()
        return buf

    def _send(self, t: torch.Tensor, dst: int, group, pending: list):
        pending.append((self.dist.isend(t, dst=dst, group=group), t))
        self.p2p_bytes += t.numel() * t.element_size()

    def run_step(self, plan: Plan, tokens: Sequence[np.ndarray], staged: Optional[_ChunkTokens] = None,
                 total_targets: Optional[int] = None) -> dict:
        p, dp = self.rank, self.world
        if dp != plan.pp_degree:
            raise ValueError(f"plan is for {plan.pp_degree} stages, world size is {dp}")
        toks = staged or _ChunkTokens(plan, tokens, self.device, need_ids=(p == 0), need_targets=(p == dp - 1))
        self._targets = total_targets
        for unit in plan.units:
            if self.p2p:
                self._run_unit_p2p(plan, unit, toks)
            else:
                self._run_unit_dist(plan, unit, toks)
        return {"h2d_bytes": toks.h2d_bytes}

    def _run_unit_p2p(self, plan: Plan, unit, toks: _ChunkTokens):
        p, dp, ch = self.rank, self.world, self.ch
        for kind, pos in stage_ops(len(unit.chunks), unit.n_prefill, dp, p + 1, unit.backward_order):
            op = _op(plan, unit, pos, p, toks, self._targets)
            nbytes = self.stage.act_bytes(op)
            if kind == "F":
                src = ch["fin"].recv_wait(nbytes) if p > 0 else None
                dst = ch["fout"].send_reserve(nbytes) if p + 1 < dp else None
                self.stage.forward(op, src, out_ptr=dst)
                if src is not None:
                    ch["fin"].recv_release()      # the stage copied it (stream-ordered)
                if dst is not None:
                    ch["fout"].send_commit()
                    self.p2p_bytes += nbytes
            else:
                g = ch["bin"].recv_wait(nbytes) if p + 1 < dp else None
                dst = ch["bout"].send_reserve(nbytes) if p > 0 else None
                self.stage.backward(op, g, out_ptr=dst)
                if g is not None:
                    ch["bin"].recv_release()
                if dst is not None:
                    ch["bout"].send_commit()
                    self.p2p_bytes += nbytes

    def _run_unit_dist(self, plan: Plan, unit, toks: _ChunkTokens):
        p, dp = self.rank, self.world
        pending = []
        for kind, pos in stage_ops(len(unit.chunks), unit.n_prefill, dp, p + 1, unit.backward_order):
            T = plan.chunks[unit.chunks[pos]].tokens
            op = _op(plan, unit, pos, p, toks, self._targets)
            if kind == "F":
                act_in = self._recv(T, self.ranks[p - 1], self.fwd_groups[p - 1]) if p > 0 else None
                out = self.stage.forward(op, act_in)
                if p + 1 < dp:
                    self._send(out, self.ranks[p + 1], self.fwd_groups[p], pending)
            else:
                g_in = self._recv(T, self.ranks[p + 1], self.bwd_groups[p]) if p + 1 < dp else None
                g_out = self.stage.backward(op, g_in)
                if p > 0:
                    self._send(g_out, self.ranks[p - 1], self.bwd_groups[p - 1], pending)
            # a send's buffer is released as soon as it completed
            pending = [(w, t) for (w, t) in pending if not w.is_completed()]
        for w, _ in pending:
            w.wait()
