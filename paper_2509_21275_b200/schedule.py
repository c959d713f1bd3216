"""Plan document (v1) -> what each stage executor replays.

  * per-stage op lists of every unit: the reference's event-driven 1F1B
    (proj/src/pipeline.cpp:96-297) issues, on stage p (1-based),
    warmup_p = min(d_p - p + n_prefill - 1, n) forwards, then a forward
    whenever fwd_issued - warmup == bwd_issued, else the next backward in the
    dry-run backward order (identical on every stage, f2b^-1).  That closed
    form is what `stage_ops` returns (SURVEY.md §3.3 verified it against
    simulate_plan with 0 mismatches; tests/test_schedule.py re-checks it
    against the planner's own trace documents).
  * token layout of every chunk: slices[0] is tokens [context, context+s0)
    of `seq`; the remaining slices are whole short sequences, in the packer's
    member order (processor.cpp:179-184 sort, :212 placement: tokens desc,
    seq asc; arrival order for the no_wbc packer, :363-381).
  * checkpointed layer counts ckpt[stage][pos] (plan_io.cpp:91-100).
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

KIND = {"batched": 0, "split": 1, "hybrid": 2}


@dataclass
class ChunkLayout:
    id: int
    kind: int
    seq: int                 # -1 for batched
    context: int
    tail: bool
    slices: List[int]
    members: List[Tuple[int, int, int]]   # (sequence, start token, length) per slice
    seq_len: int             # length of `seq` (0 if none)

    @property
    def tokens(self) -> int:
        return sum(self.slices)


@dataclass
class Unit:
    chunks: List[int]        # chunk ids, forward order
    n_prefill: int
    f2b: List[int]
    ckpt: List[List[int]]    # [stage][pos]

    @property
    def backward_order(self) -> List[int]:
        order = [0] * len(self.f2b)
        for k, j in enumerate(self.f2b):
            order[j] = k
        return order


@dataclass
class Plan:
    doc: dict
    pp_degree: int
    layers: int
    chunks: Dict[int, ChunkLayout]
    units: List[Unit]
    lengths: List[int]

    @property
    def total_tokens(self) -> int:
        return sum(self.lengths)

    @property
    def total_targets(self) -> int:
        return sum(max(0, n - 1) for n in self.lengths)


def stage_ops(n: int, n_prefill: int, pp_degree: int, stage: int,
              backward_order: Sequence[int]) -> List[Tuple[str, int]]:
    """Op list of `stage` (1-based) for one unit: ('F', pos) / ('B', pos)."""
    warmup = min(pp_degree - stage + n_prefill - 1, n)
    ops, f, b = [], 0, 0
    while f < n or b < n:
        if f < warmup or (f < n and f - warmup == b):
            ops.append(("F", f))
            f += 1
        else:
            ops.append(("B", backward_order[b]))
            b += 1
    return ops


def parse_plan(doc_text_or_dict, lengths: Sequence[int]) -> Plan:
    doc = json.loads(doc_text_or_dict) if isinstance(doc_text_or_dict, (str, bytes)) else doc_text_or_dict
    if doc.get("kind") != "plan" or doc.get("version") != 1:
        raise ValueError("not a v1 plan document")
    lengths = [int(x) for x in lengths]
    per_seq = doc["per_sequence"]
    if len(per_seq) != len(lengths):
        raise ValueError("plan and length list disagree on the number of sequences")
    owners: Dict[int, List[int]] = {}
    for s, ids in enumerate(per_seq):
        for cid in ids:
            owners.setdefault(cid, []).append(s)
    arrival = doc["mode"] == "no_wbc"
    chunks = {}
    for cj in doc["chunks"]:
        cid = cj["id"]
        seq = cj.get("seq", -1)
        slices = [int(x) for x in cj["slices"]]
        shorts = [s for s in owners.get(cid, []) if s != seq]
        if arrival:
            shorts.sort()
        else:
            shorts.sort(key=lambda s: (-lengths[s], s))
        members = []
        rest = slices
        if seq >= 0:
            members.append((seq, int(cj["context"]), slices[0]))
            rest = slices[1:]
        if sorted(lengths[s] for s in shorts) != sorted(rest):
            raise ValueError(f"chunk {cid}: packed members do not match its slices")
        # assign members to slices respecting the slice order
        pool = list(shorts)
        for n in rest:
            s = next(x for x in pool if lengths[x] == n)
            pool.remove(s)
            members.append((s, 0, n))
        chunks[cid] = ChunkLayout(cid, KIND[cj["kind"]], seq, int(cj["context"]), bool(cj["tail"]),
                                  slices, members, lengths[seq] if seq >= 0 else 0)
    units = [Unit([int(x) for x in u["chunks"]], int(u["n_prefill"]), [int(x) for x in u["f2b"]],
                  [[int(x) for x in row] for row in u["ckpt"]]) for u in doc["units"]]
    cfg = doc["config"]
    return Plan(doc, int(cfg["cluster"]["pp_degree"]), int(cfg["model"]["layers"]), chunks, units,
                lengths)


# ------------------------------------------------------------- tokens ----
def _splitmix64(state: np.uint64, n: int) -> np.ndarray:
    """n outputs of splitmix64 starting from `state` (vectorised)."""
    with np.errstate(over="ignore"):
        idx = np.arange(1, n + 1, dtype=np.uint64)
        z = np.uint64(state) + idx * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def synthetic_tokens(lengths: Sequence[int], vocab: int, seed: int) -> List[np.ndarray]:
    """Seeded uniform token ids in [0, vocab) per sequence."""
    out = []
    for s, n in enumerate(lengths):
        r = _splitmix64(np.uint64((seed * 1000003 + s) & 0xFFFFFFFFFFFFFFFF), int(n))
        out.append((r % np.uint64(vocab)).astype(np.int32))
    return out


def chunk_token_arrays(layout: ChunkLayout, tokens: Sequence[np.ndarray]):
    """(token ids, next-token targets with -1 where the sequence ends)."""
    ids, tgt = [], []
    for (s, start, n) in layout.members:
        seq = tokens[s]
        ids.append(seq[start:start + n])
        t = np.full(n, -1, dtype=np.int32)
        avail = min(n, len(seq) - start - 1)
        if avail > 0:
            t[:avail] = seq[start + 1:start + 1 + avail]
        tgt.append(t)
    return np.concatenate(ids).astype(np.int32), np.concatenate(tgt).astype(np.int32)
