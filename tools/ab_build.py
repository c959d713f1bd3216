"""Build an A/B variant of libepp_gpu.so: one source recompiled with extra
nvcc defines, linked against the current build's other objects.

    python tools/ab_build.py --src gemm.cu -D EPP_PAIR_EPI_WARPS=4 --out tools/_ab/epi4.so
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_21275_b200 import _build as b  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--src", required=True, help="file under csrc/gpu to recompile")
    ap.add_argument("--from-file", default=None, help="compile this file in its place (e.g. a git show of HEAD)")
    ap.add_argument("-D", action="append", default=[], dest="defs")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    b.build_gpu()
    objdir = b.BUILD / "gpu"
    out = Path(a.out).resolve()
    out.parent.mkdir(parents=True, exist_ok=True)
    src = b.CSRC / "gpu" / a.src
    variant = out.with_suffix(".o")
    text = Path(a.from_file) if a.from_file else src
    b._run([b.NVCC] + b.NVCC_FLAGS + [f"-D{d}" for d in a.defs] + ["-c", str(text), "-o", str(variant)])
    objs = [str(variant) if o.stem == src.stem else str(o) for o in sorted(objdir.glob("*.o"))]
    b._run([b.NVCC, "-shared"] + b.GPU_ARCH + ["-o", str(out)] + objs)
    variant.unlink()
    print(out)


if __name__ == "__main__":
    main()
