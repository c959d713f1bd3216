"""GEMM microbenchmark (GPU): the tcgen05 GEMM on the stage executor's
shapes (GPT-1.3B, T tokens per chunk): forward X W^T, data-gradient dY W and
weight-gradient dY^T X, timed by the library's per-launch CUDA events.

    python tools/gemm_bench.py [--T 16384] [--reps 10]
"""
import argparse
import ctypes
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_21275_b200 import gpu  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=16384)
    ap.add_argument("--D", type=int, default=2048)
    ap.add_argument("--F", type=int, default=8192)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--lib", default=None, help="alternative libepp_gpu.so (A/B runs)")
    args = ap.parse_args()
    if args.lib:
        gpu._LIB_PATH = Path(args.lib)
    torch.cuda.set_device(0)
    lib = gpu.lib()
    gpu.pool_reserve(8 << 30)   # as the stage does: workspaces never wait on the driver to map memory
    T, D, F = args.T, args.D, args.F
    bf = torch.bfloat16
    out = {}
    # (name, M, N, K, a_kmajor, b_kmajor, epi): A is [M,K] (K-major) or [K,M]; B is [N,K] or [K,N]
    cases = [("fwd_qkv", T, 3 * D, D, 1, 1, 0), ("fwd_up", T, F, D, 1, 1, 0), ("fwd_down", T, D, F, 1, 1, 0),
             ("dgrad_up", T, D, F, 1, 0, 0), ("wgrad_up", F, D, T, 0, 0, 1), ("wgrad_down", D, F, T, 0, 0, 1)]
    for name, M, N, K, ak, bk, epi in cases:
        A = torch.randn((M, K) if ak else (K, M), device="cuda").to(bf)
        B = torch.randn((N, K) if bk else (K, N), device="cuda").to(bf)
        C = torch.zeros((M, N), device="cuda", dtype=torch.float32 if epi == 1 else bf)

        def once():
            gpu.check(lib.epp_kernel_gemm(M, N, K, A.data_ptr(), A.shape[1], ak, B.data_ptr(), B.shape[1], bk,
                                          C.data_ptr(), N, None, 0, epi, 1, gpu.stream_ptr()))

        once()
        torch.cuda.synchronize()
        lib.epp_gpu_profile(1)
        for _ in range(args.reps):
            once()
        torch.cuda.synchronize()
        lib.epp_gpu_profile(0)
        a, b, c = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        gpu.check(lib.epp_gpu_profile_read(0, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), 1))
        out[name] = {"ms": round(a.value / c.value, 4), "tflops": round(b.value / a.value / 1e9, 1)}
    # fused-epilogue data gradients: GELU' (R = h, C2 = gelu(h)) and SwiGLU'
    # (R = h = [g | u], C = dh [T, 2F], C2 = silu(g) u)
    # *_store: the same operands and layout with a plain bf16 store (isolates
    # the epilogue); *_kmajor: the same epilogue with a K-major weight operand
    # (epilogue cost split: addres = R load + store; storegelu = math + C2
    # store; gelu_noc2 = R load + math + store)
    for name, epi, wk in (("dgrad_gelu", 5, 0), ("dgrad_swiglu", 8, 0), ("dgrad_gelu_store", 0, 0),
                          ("dgrad_gelu_kmajor", 5, 1), ("dgrad_store_kmajor", 0, 1), ("dgrad_addres", 2, 0),
                          ("dgrad_storegelu", 4, 0), ("dgrad_gelu_noc2", 5, 0)):
        M, N, K = T, F, D
        dy = torch.randn((M, K), device="cuda").to(bf)
        W = torch.randn((N, K) if wk else (K, N), device="cuda").to(bf)
        h = torch.randn((M, 2 * N if epi == 8 else N), device="cuda").to(bf)
        C = torch.empty((M, 2 * N if epi == 8 else N), device="cuda", dtype=bf)
        C2 = torch.empty((M, N), device="cuda", dtype=bf)

        def once2():
            gpu.check(lib.epp_kernel_gemm_ex(M, N, K, dy.data_ptr(), K, 1, W.data_ptr(), W.shape[1], wk, C.data_ptr(),
                                             C.shape[1], h.data_ptr(), h.shape[1], None if name.endswith("noc2") else C2.data_ptr(), N, epi, 1,
                                             gpu.stream_ptr()))

        once2()
        torch.cuda.synchronize()
        lib.epp_gpu_profile(1)
        for _ in range(args.reps):
            once2()
        torch.cuda.synchronize()
        lib.epp_gpu_profile(0)
        a, b, c = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        gpu.check(lib.epp_gpu_profile_read(0, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), 1))
        out[name] = {"ms": round(a.value / c.value, 4), "tflops": round(b.value / a.value / 1e9, 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
