"""The C-ABI libraries load and export every function include/*.h declares
(no GPU needed: symbols only, no compute calls)."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared(header: str):
    text = (ROOT / "include" / header).read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(epp_[a-z0-9_]+)\s*\(", text)))


@pytest.mark.parametrize("header,lib", [("epp_c.h", "libepp_planner.so"), ("epp_gpu.h", "libepp_gpu.so")])
def test_exports(header, lib):
    path = ROOT / "paper_2509_21275_b200" / lib
    assert path.exists(), f"{lib} not built (run __graft_entry__.build())"
    so = ctypes.CDLL(str(path))
    names = declared(header)
    assert len(names) >= 5
    missing = [n for n in names if not hasattr(so, n)]
    assert not missing, missing


def test_cpp_api_exported():
    """The C++ drop-in API (include/epp/*.hpp) is exported too: the reference
    test-suite links against it (tests/test_reference_suite.py)."""
    import subprocess
    out = subprocess.run(["nm", "-DC", "--defined-only", str(ROOT / "paper_2509_21275_b200/libepp_planner.so")],
                         capture_output=True, text=True).stdout
    for sym in ["epp::make_plan(", "epp::milp::solve(", "epp::detail::run_schedule(", "epp::split_longest(",
                "epp::plan_to_json(", "epp::fit_cost_params(", "epp::generate_workload(", "epp::render_svg("]:
        assert sym.rstrip("(") in out, sym


def test_planner_error_codes(planner):
    with pytest.raises(planner.ConfigError):
        planner.make_plan_document({"cluster": {}}, [1, 2], None)
    with pytest.raises(planner.ParseError):
        planner.make_plan_document("{not json", [1, 2], None)
    with pytest.raises(planner.ContractError):
        planner.generate_workload("github_like", 0, 0, 10)
