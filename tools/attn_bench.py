"""Attention kernel microbenchmark (GPU): the tcgen05 forward / dQ / dK-dV
kernels on representative segment layouts, timed by the library's own
per-launch CUDA events (epp_gpu_profile).  Rates are ALGORITHMIC: 4*H*hd
FLOP per visible (query, key) pair forward, 8*H*hd backward.

    python tools/attn_bench.py [--reps 5] [--check]
"""
import argparse
import ctypes
import json
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_21275_b200 import gpu  # noqa: E402

CASES = {
    "long16k": dict(H=16, Hkv=16, hd=128, segs=[(0, 16384, 0)]),
    "ctx12k+4k": dict(H=16, Hkv=16, hd=128, segs=[(0, 4096, 12288)]),
    "packed": dict(H=16, Hkv=16, hd=128, segs=None),
    "gqa8k": dict(H=32, Hkv=8, hd=128, segs=[(0, 8192, 0)]),
    "long32k": dict(H=16, Hkv=16, hd=128, segs=[(0, 32768, 0)]),
    "seq4k": dict(H=16, Hkv=16, hd=128, segs=[(0, 4096, 0)]),
    "seq2k": dict(H=16, Hkv=16, hd=128, segs=[(0, 2048, 0)]),
    "seq1k_x8": dict(H=16, Hkv=16, hd=128, segs=[(i * 1024, 1024, 0) for i in range(8)]),
    # GPT-7B (H=32, hd=128) at the default bench workload: a whole 16K
    # sequence, and a split slice + packed short (14926 + 1316)
    "gpt7b_16k": dict(H=32, Hkv=32, hd=128, segs=[(0, 16384, 0)]),
    "gpt7b_hybrid": dict(H=32, Hkv=32, hd=128, segs=[(0, 14926, 0), (14926, 1316, 0)]),
    "gpt7b_ctx": dict(H=32, Hkv=32, hd=128, segs=[(0, 5349, 10571)]),
    # Llama-7B (GQA 32/8) at 64K split into 8 slices: the last slice, and a middle one
    "llama_ctx56k": dict(H=32, Hkv=8, hd=128, segs=[(0, 8192, 57344)]),
    "llama_ctx24k": dict(H=32, Hkv=8, hd=128, segs=[(0, 8192, 24576)]),
}


def packed_segs(total=16384, seed=0):
    g = torch.Generator().manual_seed(seed)
    segs, q = [], 0
    while q < total:
        n = int(min(total - q, max(16, math.exp(torch.empty(1).uniform_(math.log(64), math.log(4096),
                                                                         generator=g).item()))))
        segs.append((q, n, 0))
        q += n
    return segs


def run(case, reps):
    lib = gpu.lib()
    H, Hkv, hd = case["H"], case["Hkv"], case["hd"]
    segs = case["segs"] or packed_segs()
    T = sum(s[1] for s in segs)
    torch.manual_seed(0)
    dev = "cuda"
    q = torch.randn(T, H, hd, device=dev).bfloat16()
    ks = [torch.randn(c + n, Hkv, hd, device=dev).bfloat16() for (_, n, c) in segs]
    vs = [torch.randn(c + n, Hkv, hd, device=dev).bfloat16() for (_, n, c) in segs]
    o = torch.empty(T, H, hd, device=dev, dtype=torch.bfloat16)
    lse = torch.empty(H, T, device=dev)
    do = torch.randn(T, H, hd, device=dev).bfloat16()
    dks = [torch.zeros(k.shape, device=dev) for k in ks]
    dvs = [torch.zeros(v.shape, device=dev) for v in vs]
    dq = torch.empty(T, H, hd, device=dev)
    n = len(segs)
    I32, VP = ctypes.c_int32 * n, ctypes.c_void_p * n
    qs, ql, cx = I32(*[s[0] for s in segs]), I32(*[s[1] for s in segs]), I32(*[s[2] for s in segs])
    kp, vp = VP(*[k.data_ptr() for k in ks]), VP(*[v.data_ptr() for v in vs])
    dkp, dvp = VP(*[d.data_ptr() for d in dks]), VP(*[d.data_ptr() for d in dvs])
    scale = 1.0 / math.sqrt(hd)

    def once():
        gpu.check(lib.epp_kernel_attention_fwd(T, H, Hkv, hd, scale, n, qs, ql, cx, kp, vp, q.data_ptr(),
                                               o.data_ptr(), lse.data_ptr(), 1, gpu.stream_ptr()))
        gpu.check(lib.epp_kernel_attention_bwd(T, H, Hkv, hd, scale, n, qs, ql, cx, kp, vp, dkp, dvp,
                                               q.data_ptr(), o.data_ptr(), lse.data_ptr(), do.data_ptr(),
                                               dq.data_ptr(), 1, gpu.stream_ptr()))

    once()
    torch.cuda.synchronize()
    lib.epp_gpu_profile(1)
    for _ in range(reps):
        once()
    torch.cuda.synchronize()
    lib.epp_gpu_profile(0)
    out = {"T": T, "nseg": n}
    for cls, name in ((1, "fwd"), (3, "bwd_dq"), (4, "bwd_dkv"), (2, "bwd")):
        a, b, c = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        gpu.check(lib.epp_gpu_profile_read(cls, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), 1))
        if c.value:
            out[name] = {"ms": round(a.value / c.value, 4), "tflops": round(b.value / a.value / 1e9, 1)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cases", default=",".join(CASES))
    ap.add_argument("--lib", default=None, help="alternative libepp_gpu.so (A/B runs)")
    args = ap.parse_args()
    if args.lib:
        gpu._LIB_PATH = Path(args.lib)
    torch.cuda.set_device(0)
    res = {k: run(CASES[k], args.reps) for k in args.cases.split(",")}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
