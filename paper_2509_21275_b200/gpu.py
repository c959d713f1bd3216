"""ctypes binding of libepp_gpu.so (include/epp_gpu.h) with torch plumbing.

torch provides device memory and streams; all compute goes through the CUDA
library.  Loading fails loudly when the library is missing — there is no CPU
fallback on the product path.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path
from typing import Dict, Optional

import numpy as np
import torch

from .model import ModelConfig

_LIB_PATH = Path(__file__).resolve().parent / "libepp_gpu.so"
_lib = None

DTYPES = {"f32": 0, "bf16": 1}
TORCH_DTYPES = {"f32": torch.float32, "bf16": torch.bfloat16}


class EppGpuError(RuntimeError):
    pass


class ModelDesc(ctypes.Structure):
    _fields_ = [("arch", ctypes.c_int32), ("layers", ctypes.c_int32), ("hidden", ctypes.c_int32),
                ("heads", ctypes.c_int32), ("kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("ffn", ctypes.c_int32), ("vocab", ctypes.c_int32), ("rope_theta", ctypes.c_float),
                ("norm_eps", ctypes.c_float)]


class ChunkDesc(ctypes.Structure):
    _fields_ = [("id", ctypes.c_int32), ("seq", ctypes.c_int32), ("kind", ctypes.c_int32),
                ("tail", ctypes.c_int32), ("context", ctypes.c_int64), ("seq_len", ctypes.c_int64),
                ("nslices", ctypes.c_int32), ("slices", ctypes.POINTER(ctypes.c_int64)),
                ("ckpt_layers", ctypes.c_int32), ("loss_scale", ctypes.c_float),
                ("token_ids", ctypes.c_void_p), ("target_ids", ctypes.c_void_p)]


class TraceEvent(ctypes.Structure):
    _fields_ = [("chunk_id", ctypes.c_int32), ("op", ctypes.c_int32), ("start_s", ctypes.c_double),
                ("end_s", ctypes.c_double), ("live_bytes", ctypes.c_int64)]


class ParamInfo(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("numel", ctypes.c_int64), ("master", ctypes.c_void_p),
                ("work", ctypes.c_void_p), ("grad", ctypes.c_void_p)]


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise ImportError(f"{_LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback)")
        L = ctypes.CDLL(str(_LIB_PATH), mode=os.RTLD_LOCAL)
        vp, i32, i64, f32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float
        sig = {
            "epp_gpu_set_device": [ctypes.c_int],
            "epp_stage_create": [ctypes.POINTER(ModelDesc), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)],
            "epp_stage_destroy": [vp],
            "epp_stage_init_weights": [vp, ctypes.c_uint64, vp],
            "epp_stage_num_params": [vp, ctypes.POINTER(i32)],
            "epp_stage_param": [vp, i32, ctypes.POINTER(ParamInfo)],
            "epp_stage_sync_weights": [vp, vp],
            "epp_stage_forward": [vp, ctypes.POINTER(ChunkDesc), vp, vp, vp],
            "epp_stage_backward": [vp, ctypes.POINTER(ChunkDesc), vp, vp, vp],
            "epp_seq_release": [vp, i32],
            "epp_stage_loss": [vp, ctypes.POINTER(ctypes.c_double), i32, vp],
            "epp_stage_loss_async": [vp, vp, i32, vp],
            "epp_gpu_pool_reserve": [ctypes.c_uint64, vp],
            "epp_stage_zero_grads": [vp, vp],
            "epp_stage_adamw_step": [vp, f32, f32, f32, f32, f32, i32, vp],
            "epp_stage_memory": [vp, ctypes.POINTER(i64), ctypes.POINTER(i64)],
            "epp_gpu_profile": [i32],
            "epp_stage_trace": [vp, i32, vp],
            "epp_stage_arena": [vp, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(i64)],
            "epp_stage_buckets": [vp, ctypes.POINTER(i64), i32, ctypes.POINTER(i32)],
            "epp_stage_grad_events": [vp, i32],
            "epp_stage_bucket_wait": [vp, i32, vp],
            "epp_stage_opt_shard": [vp, i32, i32, ctypes.POINTER(i64)],
            "epp_stage_trace_read": [vp, ctypes.POINTER(TraceEvent), i32, ctypes.POINTER(i32)],
            "epp_stage_chunk_loss": [vp, i32, ctypes.POINTER(ctypes.c_double), vp],
            "epp_gpu_profile_read": [i32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                     ctypes.POINTER(i64), i32],
            "epp_kernel_gemm": [i32, i32, i32, vp, i64, i32, vp, i64, i32, vp, i64, vp, i64, i32, i32, vp],
            "epp_kernel_gemm_ex": [i32, i32, i32, vp, i64, i32, vp, i64, i32, vp, i64, vp, i64, vp, i64, i32, i32,
                                   vp],
            "epp_kernel_attention_fwd": [i32, i32, i32, i32, f32, i32, ctypes.POINTER(i32),
                                         ctypes.POINTER(i32), ctypes.POINTER(i32),
                                         ctypes.POINTER(vp), ctypes.POINTER(vp), vp, vp, vp, i32, vp],
            "epp_kernel_attention_bwd": [i32, i32, i32, i32, f32, i32, ctypes.POINTER(i32),
                                         ctypes.POINTER(i32), ctypes.POINTER(i32),
                                         ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp),
                                         ctypes.POINTER(vp), vp, vp, vp, vp, vp, i32, vp],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        p2p = {
            "epp_p2p_init": [ctypes.c_int, ctypes.POINTER(ctypes.c_int)],
            "epp_p2p_create": [ctypes.c_int, ctypes.c_uint64, ctypes.POINTER(vp), ctypes.c_char_p],
            "epp_p2p_open": [vp, ctypes.c_char_p],
            "epp_p2p_send_reserve": [vp, ctypes.c_uint64, vp, ctypes.POINTER(vp)],
            "epp_p2p_send_commit": [vp, vp],
            "epp_p2p_recv_wait": [vp, ctypes.c_uint64, vp, ctypes.POINTER(vp)],
            "epp_p2p_recv_release": [vp, vp],
            "epp_p2p_send": [vp, vp, ctypes.c_uint64, vp],
            "epp_p2p_recv": [vp, vp, ctypes.c_uint64, vp],
            "epp_p2p_stats": [vp, ctypes.POINTER(i64), ctypes.POINTER(i64)],
            "epp_p2p_destroy": [vp],
        }
        for name, args in p2p.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        L.epp_gpu_kernel_stats.argtypes = [i32, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(i64)]
        L.epp_gpu_kernel_stats.restype = ctypes.c_int
        L.epp_gpu_last_error.restype = ctypes.c_char_p
        L.epp_gpu_kernel_launches.restype = ctypes.c_int64
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        raise EppGpuError(lib().epp_gpu_last_error().decode())


def pool_reserve(nbytes: int) -> None:
    """Pre-reserve device memory for stage activations (see epp_gpu.h)."""
    check(lib().epp_gpu_pool_reserve(int(max(0, nbytes)), stream_ptr()))


def kernel_launches() -> int:
    return int(lib().epp_gpu_kernel_launches())


def kernel_stats() -> Dict[str, int]:
    """{demangled kernel name: launches so far} of this library's kernels."""
    L, out, i = lib(), {}, 0
    name, cnt = ctypes.c_char_p(), ctypes.c_int64()
    while L.epp_gpu_kernel_stats(i, ctypes.byref(name), ctypes.byref(cnt)) == 0:
        out[name.value.decode()] = int(cnt.value)
        i += 1
    return out


def stream_ptr(stream: Optional[torch.cuda.Stream] = None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t) -> Optional[int]:
    """Device address of a tensor, or an address passed as an int (e.g. a
    P2P mailbox slot)."""
    if t is None or isinstance(t, int):
        return t
    return t.data_ptr()


P2P_HANDLE_BYTES = 256


class P2PChannel:
    """One endpoint of a directed stage-to-stage message stream over peer
    memory (include/epp_gpu.h epp_p2p_*): role 'send' or 'recv'; the
    receiver owns the mailbox arena (>= the largest message).  Exchange
    `.handle` with the peer out of band, then open(peer_handle)."""

    def __init__(self, role: str, arena_bytes: int = 0):
        self.role = role
        buf = ctypes.create_string_buffer(P2P_HANDLE_BYTES)
        h = ctypes.c_void_p()
        check(lib().epp_p2p_create({"send": 0, "recv": 1}[role], int(arena_bytes), ctypes.byref(h), buf))
        self.h = h
        self.handle = buf.raw

    def open(self, peer_handle: bytes):
        check(lib().epp_p2p_open(self.h, peer_handle))

    def send_reserve(self, nbytes: int) -> int:
        p = ctypes.c_void_p()
        check(lib().epp_p2p_send_reserve(self.h, int(nbytes), stream_ptr(), ctypes.byref(p)))
        return p.value

    def send_commit(self):
        check(lib().epp_p2p_send_commit(self.h, stream_ptr()))

    def recv_wait(self, nbytes: int) -> int:
        p = ctypes.c_void_p()
        check(lib().epp_p2p_recv_wait(self.h, int(nbytes), stream_ptr(), ctypes.byref(p)))
        return p.value

    def recv_release(self):
        check(lib().epp_p2p_recv_release(self.h, stream_ptr()))

    def send(self, t: torch.Tensor):
        check(lib().epp_p2p_send(self.h, ctypes.c_void_p(t.data_ptr()), t.numel() * t.element_size(),
                                 stream_ptr()))

    def recv(self, t: torch.Tensor):
        check(lib().epp_p2p_recv(self.h, ctypes.c_void_p(t.data_ptr()), t.numel() * t.element_size(),
                                 stream_ptr()))

    def stats(self):
        n, b = ctypes.c_int64(), ctypes.c_int64()
        check(lib().epp_p2p_stats(self.h, ctypes.byref(n), ctypes.byref(b)))
        return n.value, b.value

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            check(lib().epp_p2p_destroy(self.h))
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def p2p_init(devices) -> None:
    """Enable peer access among `devices` (one process driving several GPUs)."""
    arr = (ctypes.c_int * len(devices))(*devices)
    check(lib().epp_p2p_init(len(devices), arr))


class CudaStage:
    """One pipeline stage on the current CUDA device (the CUDA executor)."""

    def __init__(self, model: ModelConfig, first: int, num: int, has_embed: bool, has_head: bool,
                 dtype: str = "bf16", device: Optional[int] = None, plan_stage_layers: Optional[int] = None):
        """plan_stage_layers: the per-stage layer count the planner priced
        (L / d_p; Eq. 10 assumes uniform stages).  With a head-balanced split
        this stage may hold `num` != that; checkpoint counts from the plan are
        rescaled so the full-activation layers kept never exceed what the
        planner charged (see _ckpt_layers)."""
        self.model, self.first, self.num = model, first, num
        self.plan_layers = int(plan_stage_layers or num)
        self.has_embed, self.has_head = has_embed, has_head
        self.dtype = dtype
        self.tdtype = TORCH_DTYPES[dtype]
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        L = lib()
        check(L.epp_gpu_set_device(self.device.index))
        desc = ModelDesc(1 if model.llama else 0, model.layers, model.hidden, model.heads,
                         model.kv_heads, model.head_dim, model.ffn, model.vocab,
                         model.rope_theta, model.norm_eps)
        h = ctypes.c_void_p()
        check(L.epp_stage_create(ctypes.byref(desc), first, num, int(has_embed), int(has_head),
                                 DTYPES[dtype], ctypes.byref(h)))
        self.h = h
        self._keep = {}

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            check(lib().epp_stage_destroy(self.h))
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- parameters ----------------------------------------------------------
    def params(self) -> Dict[str, dict]:
        L = lib()
        n = ctypes.c_int32()
        check(L.epp_stage_num_params(self.h, ctypes.byref(n)))
        out = {}
        for i in range(n.value):
            info = ParamInfo()
            check(L.epp_stage_param(self.h, i, ctypes.byref(info)))
            out[info.name.decode()] = {"numel": info.numel, "master": info.master, "work": info.work,
                                       "grad": info.grad}
        return out

    def init_weights(self, seed: int):
        check(lib().epp_stage_init_weights(self.h, seed, stream_ptr()))

    def load_weights(self, weights: Dict[str, torch.Tensor]):
        for name, p in self.params().items():
            src = weights[name].detach().to(self.device, torch.float32).contiguous().view(-1)
            assert src.numel() == p["numel"], name
            _wrap_ptr(p["master"], p["numel"], torch.float32, self.device).copy_(src)
        check(lib().epp_stage_sync_weights(self.h, stream_ptr()))

    def grads(self) -> Dict[str, torch.Tensor]:
        return {name: _wrap_ptr(p["grad"], p["numel"], torch.float32, self.device).clone()
                for name, p in self.params().items()}

    def grad_views(self) -> Dict[str, torch.Tensor]:
        """Zero-copy fp32 views of the accumulated gradients (in-place
        collectives, e.g. the data-parallel all-reduce)."""
        return {name: _wrap_ptr(p["grad"], p["numel"], torch.float32, self.device)
                for name, p in self.params().items()}

    # -- data-parallel buckets (include/epp_gpu.h, data parallelism) ---------
    def arena(self) -> Dict[str, torch.Tensor]:
        """Zero-copy flat views of the fp32 master and gradient arenas."""
        m, w, g, n = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int64()
        check(lib().epp_stage_arena(self.h, ctypes.byref(m), ctypes.byref(w), ctypes.byref(g), ctypes.byref(n)))
        return {"master": _wrap_ptr(m.value, n.value, torch.float32, self.device),
                "grad": _wrap_ptr(g.value, n.value, torch.float32, self.device)}

    def buckets(self):
        """Arena element offsets of the gradient buckets ([embedding],
        layers, [head]): nbuckets + 1 values."""
        nb = ctypes.c_int32()
        check(lib().epp_stage_buckets(self.h, None, 0, ctypes.byref(nb)))
        arr = (ctypes.c_int64 * (nb.value + 1))()
        check(lib().epp_stage_buckets(self.h, arr, nb.value + 1, ctypes.byref(nb)))
        return list(arr)

    def grad_events(self, enable: bool = True):
        check(lib().epp_stage_grad_events(self.h, int(enable)))

    def bucket_wait(self, bucket: int, stream: Optional[torch.cuda.Stream] = None):
        """`stream` waits until bucket's gradients of the latest backward are final."""
        check(lib().epp_stage_bucket_wait(self.h, int(bucket), stream_ptr(stream)))

    def opt_shard(self, rank: int, nranks: int) -> int:
        """ZeRO-1: keep Adam state for slice `rank` of `nranks` of every bucket;
        returns the state elements held."""
        n = ctypes.c_int64()
        check(lib().epp_stage_opt_shard(self.h, int(rank), int(nranks), ctypes.byref(n)))
        return n.value

    def sync_weights(self):
        check(lib().epp_stage_sync_weights(self.h, stream_ptr()))

    def zero_grads(self):
        check(lib().epp_stage_zero_grads(self.h, stream_ptr()))

    def adamw_step(self, lr, step, b1=0.9, b2=0.95, eps=1e-8, wd=0.1):
        check(lib().epp_stage_adamw_step(self.h, lr, b1, b2, eps, wd, step, stream_ptr()))

    def loss(self, reset: bool = False):
        out = (ctypes.c_double * 2)()
        check(lib().epp_stage_loss(self.h, out, int(reset), stream_ptr()))
        return out[0], out[1]

    def loss_async(self, out2: torch.Tensor, reset: bool = False):
        """Enqueue a copy of (loss sum, #targets) into `out2` (2 fp64, pinned
        host or device) on the current stream; the caller synchronises."""
        assert out2.dtype == torch.float64 and out2.numel() >= 2
        check(lib().epp_stage_loss_async(self.h, ctypes.c_void_p(out2.data_ptr()), int(reset), stream_ptr()))

    def chunk_loss(self, chunk_id: int):
        """(sum of token losses, #targets) of one micro-batch (epp::Chunk),
        its latest forward since the last loss reset (fp64)."""
        out = (ctypes.c_double * 2)()
        check(lib().epp_stage_chunk_loss(self.h, int(chunk_id), out, stream_ptr()))
        return out[0], out[1]

    def trace(self, enable: bool = True):
        """Start (clear + t = 0 on the current stream) or stop recording the
        measured per-op trace (include/epp_gpu.h epp_stage_trace)."""
        check(lib().epp_stage_trace(self.h, int(enable), stream_ptr()))

    def trace_read(self):
        """Recorded events [{chunk, op 'F'/'B'/'R', start, end (s), live}]
        (synchronises on the last one)."""
        n = ctypes.c_int32()
        check(lib().epp_stage_trace_read(self.h, None, 0, ctypes.byref(n)))
        buf = (TraceEvent * max(1, n.value))()
        check(lib().epp_stage_trace_read(self.h, buf, n.value, ctypes.byref(n)))
        ops = {0: "F", 1: "B", 2: "R"}
        return [{"chunk": e.chunk_id, "op": ops[e.op], "start": e.start_s, "end": e.end_s,
                 "live": e.live_bytes} for e in buf[:n.value]]

    def state_bytes(self) -> int:
        """Resident bytes of weights, fp32 grads and Adam state."""
        per = 16 + (2 if self.dtype == "bf16" else 0)
        return sum(p["numel"] for p in self.params().values()) * per

    def memory(self):
        live, peak = ctypes.c_int64(), ctypes.c_int64()
        check(lib().epp_stage_memory(self.h, ctypes.byref(live), ctypes.byref(peak)))
        return live.value, peak.value

    # -- chunk ops -------------------------------------------------------------
    def _ckpt_layers(self, c: int) -> int:
        """Layers to checkpoint for a plan count c of a uniform stage of
        plan_layers layers: the planner charges (plan_layers - c) /
        plan_layers of the stage's full activations (model.planner_config
        scales token_act_bytes to the LARGEST stage), so this stage keeps at
        most floor((plan_layers - c) * num / plan_layers) full layers."""
        P, n = self.plan_layers, self.num
        c = max(0, min(int(c), P))
        if P == n:
            return c
        return max(0, min(n, n - ((P - c) * n) // P))

    def _desc(self, c) -> ChunkDesc:
        slices = (ctypes.c_int64 * len(c.slices))(*c.slices)
        self._keep[c.id] = slices
        ckpt = self._ckpt_layers(c.ckpt_layers)
        return ChunkDesc(c.id, c.seq, c.kind, int(c.tail), c.context, c.seq_len, len(c.slices),
                         slices, ckpt, c.loss_scale, _ptr(c.token_ids), _ptr(c.target_ids))

    supports_p2p = True

    def act_bytes(self, c) -> int:
        """Bytes of one [T, hidden] activation / gradient of chunk c."""
        return sum(c.slices) * self.model.hidden * (4 if self.dtype == "f32" else 2)

    def forward(self, c, act_in, out_ptr: Optional[int] = None) -> Optional[torch.Tensor]:
        """act_in: tensor or device address (read before the call's work
        ends; the stage copies it).  out_ptr: where the stage output goes
        (e.g. the next stage's P2P mailbox); default: a new tensor, returned."""
        T = sum(c.slices)
        out = None
        if not self.has_head and out_ptr is None:
            out = torch.empty((T, self.model.hidden), dtype=self.tdtype, device=self.device)
        d = self._desc(c)
        check(lib().epp_stage_forward(self.h, ctypes.byref(d), _ptr(act_in),
                                      out_ptr if out_ptr is not None else _ptr(out), stream_ptr()))
        return out

    def backward(self, c, grad_in, out_ptr: Optional[int] = None) -> Optional[torch.Tensor]:
        """grad_in: tensor or device address, read in place by the last
        layer's backward.  out_ptr: destination of d(stage input) (e.g. the
        previous stage's mailbox); default: a new tensor, returned."""
        T = sum(c.slices)
        out = None
        if not self.has_embed and out_ptr is None:
            out = torch.empty((T, self.model.hidden), dtype=self.tdtype, device=self.device)
        d = self._desc(c)
        check(lib().epp_stage_backward(self.h, ctypes.byref(d), _ptr(grad_in),
                                       out_ptr if out_ptr is not None else _ptr(out), stream_ptr()))
        self._keep.pop(c.id, None)
        return out


def _wrap_ptr(ptr: int, numel: int, dtype: torch.dtype, device: torch.device) -> torch.Tensor:
    """Zero-copy tensor over device memory owned by the library."""
    class _Holder:
        pass
    h = _Holder()
    h.__cuda_array_interface__ = {
        "shape": (int(numel),),
        "typestr": {torch.float32: "<f4", torch.bfloat16: "<V2"}[dtype],
        "data": (int(ptr), False),
        "version": 3,
        "strides": None,
    }
    if dtype == torch.bfloat16:
        raw = torch.as_tensor(_I16Holder(ptr, numel), device=device)
        return raw.view(torch.bfloat16)
    return torch.as_tensor(h, device=device)


class _I16Holder:
    def __init__(self, ptr, numel):
        self.__cuda_array_interface__ = {"shape": (int(numel),), "typestr": "<i2",
                                         "data": (int(ptr), False), "version": 3, "strides": None}
