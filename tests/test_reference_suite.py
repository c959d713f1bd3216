"""Runs the reference's own planner unit tests (proj/tests/*.cpp, compiled
from /root/reference, never copied) against libepp_planner.so through a
doctest-compatible shim (tests/cpp/doctest_shim).  Also compiles our own
known-answer checks (tests/cpp/test_kat.cpp), which need no reference."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REF_TESTS = Path("/root/reference/proj/tests")
CXX = "/usr/bin/g++" if Path("/usr/bin/g++").exists() else shutil.which("g++")
FLAGS = ["-std=gnu++20", "-O1", "-ffp-contract=off", f"-I{ROOT / 'tests/cpp/doctest_shim'}",
         f"-I{ROOT / 'include'}", f"-I{ROOT / 'third_party'}"]
LINK = [f"-L{ROOT / 'paper_2509_21275_b200'}", "-lepp_planner",
        f"-Wl,-rpath,{ROOT / 'paper_2509_21275_b200'}", "-pthread"]


def build_and_run(tmp_path, sources, extra_inc=()):
    objs = []
    procs = []
    for src in sources:
        obj = tmp_path / (Path(src).stem + ".o")
        procs.append(subprocess.Popen([CXX] + FLAGS + [f"-I{d}" for d in extra_inc] +
                                      ["-c", str(src), "-o", str(obj)], stderr=subprocess.PIPE, text=True))
        objs.append(obj)
    for p in procs:
        _, err = p.communicate()
        assert p.returncode == 0, err[-3000:]
    exe = tmp_path / "suite"
    r = subprocess.run([CXX, "-o", str(exe)] + [str(o) for o in objs] + LINK, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    return r


@pytest.mark.skipif(not REF_TESTS.exists(), reason="/root/reference not present")
def test_reference_doctest_suite(tmp_path):
    srcs = sorted(REF_TESTS.glob("test_*.cpp")) + [ROOT / "tests/cpp/shim_main.cpp"]
    r = build_and_run(tmp_path, srcs, extra_inc=[REF_TESTS])
    assert r.returncode == 0, r.stdout + r.stderr[-4000:]
    assert "97 passed | 0 failed" in r.stdout, r.stdout


def test_known_answers(tmp_path):
    r = build_and_run(tmp_path, [ROOT / "tests/cpp/test_kat.cpp", ROOT / "tests/cpp/shim_main.cpp"])
    assert r.returncode == 0, r.stdout + r.stderr[-4000:]


def test_shim_detects_failures(tmp_path):
    canary = tmp_path / "canary.cpp"
    canary.write_text('#include <doctest.h>\nTEST_CASE("canary") { CHECK(1 == 2); }\n')
    r = build_and_run(tmp_path, [canary, ROOT / "tests/cpp/shim_main.cpp"])
    assert r.returncode != 0 and "1 failed" in r.stdout
