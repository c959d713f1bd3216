"""In-tree build of the native libraries (no JIT cache; the .so files travel
with the repo snapshot to the GPU box).

  libepp_planner.so  - C++ planner (include/epp/*.hpp API + include/epp_c.h)
  libepp_gpu.so      - sm_100a stage executor + kernels (include/epp_gpu.h)

The oracle (oracle/_ref/libepp_ref.so) is built by oracle/Makefile; see
build_oracle().  Compiler flags are part of the parity contract: the
planner is compiled like the reference (-O3, no -march, no FMA contraction)
so float64 plan arithmetic is bit-identical.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build"
CXX = "/usr/bin/g++" if Path("/usr/bin/g++").exists() else (shutil.which("g++") or "g++")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
CUDA_HOME = Path(NVCC).resolve().parent.parent

PLANNER_SO = PKG / "libepp_planner.so"
GPU_SO = PKG / "libepp_gpu.so"

PLANNER_FLAGS = ["-std=gnu++20", "-O3", "-DNDEBUG", "-fPIC", "-ffp-contract=off",
                 "-pthread", "-Wall", "-Wextra",
                 f"-I{ROOT / 'include'}", f"-I{ROOT / 'third_party'}"]

GPU_ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC",
              "--expt-relaxed-constexpr", "-DNDEBUG",
              f"-I{ROOT / 'include'}", f"-I{CSRC / 'gpu'}"] + GPU_ARCH


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(map(str, cmd))}\n{r.stdout}\n{r.stderr}")
    return r


def _headers(*dirs):
    out = []
    for d in dirs:
        out += list(Path(d).rglob("*.h")) + list(Path(d).rglob("*.hpp")) + list(Path(d).rglob("*.cuh"))
    return out


def build_planner(force: bool = False) -> Path:
    srcs = sorted((CSRC / "planner").glob("*.cpp"))
    hdrs = _headers(ROOT / "include")
    objdir = BUILD / "planner"
    objdir.mkdir(parents=True, exist_ok=True)
    jobs = []
    objs = []
    for s in srcs:
        o = objdir / (s.stem + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            jobs.append([CXX] + PLANNER_FLAGS + ["-c", str(s), "-o", str(o)])
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(_run, jobs))
    if force or jobs or _stale(PLANNER_SO, objs):
        _run([CXX, "-shared", "-pthread", "-o", str(PLANNER_SO)] + [str(o) for o in objs])
    return PLANNER_SO


def build_gpu(force: bool = False) -> Path | None:
    gdir = CSRC / "gpu"
    srcs = sorted(gdir.glob("*.cu")) + sorted(gdir.glob("*.cpp"))
    if not srcs:
        return None
    hdrs = _headers(ROOT / "include", gdir)
    objdir = BUILD / "gpu"
    objdir.mkdir(parents=True, exist_ok=True)
    jobs = []
    objs = []
    for s in srcs:
        o = objdir / (s.stem + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            jobs.append([NVCC] + NVCC_FLAGS + ["-c", str(s), "-o", str(o)])
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(_run, jobs))
    if force or jobs or _stale(GPU_SO, objs):
        _run([NVCC, "-shared"] + GPU_ARCH + ["-o", str(GPU_SO)] + [str(o) for o in objs]
 )
    return GPU_SO


def build_oracle(force: bool = False) -> Path | None:
    """Compile oracle/_ref from /root/reference (present only in the build
    container; the GPU box uses the prebuilt .so that travels with the repo)."""
    ref = Path("/root/reference/proj/src")
    out = ROOT / "oracle" / "_ref" / "libepp_ref.so"
    if not ref.exists():
        return out if out.exists() else None
    cmd = ["make", "-C", str(ROOT / "oracle"), "-j", str(os.cpu_count() or 4)]
    if force:
        _run(["make", "-C", str(ROOT / "oracle"), "clean"])
    _run(cmd)
    return out


def build_all(force: bool = False) -> None:
    build_planner(force)
    build_gpu(force)
    build_oracle(force)


if __name__ == "__main__":
    import sys
    build_all(force="--force" in sys.argv)
    print("built:", PLANNER_SO, GPU_SO if GPU_SO.exists() else "(no gpu lib)")
