"""Does running a layer's weight-gradient GEMM concurrently with its
data-gradient GEMM (two streams) fill the waves that short chunks leave
empty?  Times, per Llama-7B / GPT-7B backward projection at T tokens, the
pair serially on one stream vs forked onto two streams (CUDA events on the
joining stream).

    python tools/overlap_bench.py [--T 1700] [--model llama]
"""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_21275_b200 import gpu  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=1700)
    ap.add_argument("--model", default="llama", choices=["llama", "gpt"])
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    lib = gpu.lib()
    gpu.pool_reserve(8 << 30)
    T = args.T
    D = 4096
    F = 11008 if args.model == "llama" else 16384
    qkv = 6144 if args.model == "llama" else 3 * D
    up = 2 * F if args.model == "llama" else F
    bf = torch.bfloat16
    # (name, out, in): W [out, in]; dgrad dX[T,in] = dY[T,out] W; wgrad dW[out,in] += dY^T X
    projs = [("qkv", qkv, D), ("o", D, D), ("up", up, D), ("down", D, F)]
    side = torch.cuda.Stream()
    main_s = torch.cuda.current_stream()
    res = {}
    for name, out, inn in projs:
        dY = torch.randn(T, out, device="cuda").to(bf)
        X = torch.randn(T, inn, device="cuda").to(bf)
        W = torch.randn(out, inn, device="cuda").to(bf)
        dX = torch.empty(T, inn, device="cuda", dtype=bf)
        dW = torch.zeros(out, inn, device="cuda", dtype=torch.float32)

        def dgrad(s):
            gpu.check(lib.epp_kernel_gemm(T, inn, out, dY.data_ptr(), out, 1, W.data_ptr(), inn, 0, dX.data_ptr(),
                                          inn, None, 0, 0, 1, gpu.stream_ptr(s)))

        def wgrad(s):
            gpu.check(lib.epp_kernel_gemm(out, inn, T, dY.data_ptr(), out, 0, X.data_ptr(), inn, 0, dW.data_ptr(),
                                          inn, None, 0, 1, 1, gpu.stream_ptr(s)))

        def serial():
            dgrad(main_s)
            wgrad(main_s)

        def forked():
            ev = torch.cuda.Event()
            ev.record(main_s)
            side.wait_event(ev)
            wgrad(side)
            dgrad(main_s)
            ev2 = torch.cuda.Event()
            ev2.record(side)
            main_s.wait_event(ev2)

        out_r = {}
        for label, fn in (("serial", serial), ("forked", forked), ("dgrad", lambda: dgrad(main_s)),
                          ("wgrad", lambda: wgrad(main_s))):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(main_s)
            for _ in range(args.reps):
                fn()
            b.record(main_s)
            torch.cuda.synchronize()
            out_r[label] = round(a.elapsed_time(b) / args.reps * 1e3, 1)   # us
        flops = 2.0 * 2 * T * out * inn
        out_r["tflops_serial"] = round(flops / out_r["serial"] / 1e6, 1)
        out_r["tflops_forked"] = round(flops / out_r["forked"] / 1e6, 1)
        res[name] = out_r
    print(json.dumps({"T": T, "model": args.model, "us": res}))


if __name__ == "__main__":
    main()
