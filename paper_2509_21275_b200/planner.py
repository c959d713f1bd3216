"""Python binding of the C++ planner (libepp_planner.so, include/epp_c.h).

Mirrors the reference's planner entry points (proj/include/epp/planner.hpp,
plan_io.hpp, workload.hpp) with the same argument meaning and the same error
classes (re-raised as Python exceptions of the same names).  Documents are the
reference's JSON v1 byte streams.
"""
from __future__ import annotations

import ctypes
import json
import os
from pathlib import Path
from typing import Iterable, Optional, Sequence

_PKG = Path(__file__).resolve().parent
_LIB_PATH = _PKG / "libepp_planner.so"

MODES = {"main": 0, "no_wbc": 1, "no_ckpt": 2, "full_ckpt": 3}


class Error(RuntimeError):
    """epp::Error"""


class ConfigError(Error):
    pass


class ParseError(Error):
    pass


class InfeasibleError(Error):
    pass


class IoError(Error):
    pass


class ContractError(Error):
    pass


class FitError(Error):
    pass


_CODE_TO_EXC = {1: Error, 2: ConfigError, 3: ParseError, 4: InfeasibleError,
                5: IoError, 6: ContractError, 7: FitError, 8: Error}


class _Api:
    """ctypes view of one planner library (the product, or the oracle with
    prefix 'epp_ref_' — the latter only from tests/bench)."""

    def __init__(self, path: Path, prefix: str = "epp_"):
        if not Path(path).exists():
            raise ImportError(f"planner library missing: {path} (run __graft_entry__.build())")
        self.lib = ctypes.CDLL(str(path), mode=os.RTLD_LOCAL)
        f = lambda name: getattr(self.lib, prefix + name)  # noqa: E731
        self.plan = f("plan_json")
        self.plan.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int64), ctypes.c_size_t,
                              ctypes.c_int, ctypes.c_int, ctypes.c_int,
                              ctypes.POINTER(ctypes.c_void_p)]
        self.simulate = f("simulate_json")
        self.simulate.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p),
                                  ctypes.POINTER(ctypes.c_double)]
        self.gen = f("generate_workload")
        self.gen.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_int64,
                             ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]
        self.fit = f("fit_cost_json")
        self.fit.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
        self.render = f("render_svg")
        self.render.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
        self.last_error = f("last_error")
        self.last_error.restype = ctypes.c_char_p
        self.free = f("free")
        self.free.argtypes = [ctypes.c_void_p]
        for fn in (self.plan, self.simulate, self.gen, self.fit, self.render):
            fn.restype = ctypes.c_int

    def check(self, rc: int) -> None:
        if rc != 0:
            raise _CODE_TO_EXC.get(rc, Error)(self.last_error().decode())

    def take_string(self, ptr: ctypes.c_void_p) -> str:
        try:
            return ctypes.string_at(ptr.value).decode()
        finally:
            self.free(ptr)


_api: Optional[_Api] = None


def api() -> _Api:
    global _api
    if _api is None:
        _api = _Api(_LIB_PATH)
    return _api


def _as_text(doc) -> bytes:
    if isinstance(doc, (bytes, bytearray)):
        return bytes(doc)
    if isinstance(doc, str):
        return doc.encode()
    return json.dumps(doc).encode()


def make_plan_document(config, lengths: Sequence[int], slices: Optional[int] = None,
                       mode: str = "main", jobs: int = 1, _lib: Optional[_Api] = None) -> str:
    """epp::make_plan + dump_document(plan_to_json(...)) -> plan v1 text."""
    a = _lib or api()
    arr = (ctypes.c_int64 * len(lengths))(*[int(x) for x in lengths])
    out = ctypes.c_void_p()
    a.check(a.plan(_as_text(config), arr, len(lengths), int(slices or 0), MODES[mode],
                   int(jobs), ctypes.byref(out)))
    return a.take_string(out)


def simulate_plan_document(plan_doc, _lib: Optional[_Api] = None):
    """simulate_plan + trace_to_json -> (trace v1 text, plan_simulated_seconds)."""
    a = _lib or api()
    out = ctypes.c_void_p()
    total = ctypes.c_double()
    a.check(a.simulate(_as_text(plan_doc), ctypes.byref(out), ctypes.byref(total)))
    return a.take_string(out), total.value


def generate_workload(preset: str, count: int, seed: int, context_cap: int,
                      uniform_min: int = 1, uniform_max: int = 0,
                      _lib: Optional[_Api] = None) -> list:
    """epp::generate_workload -> list of lengths."""
    a = _lib or api()
    arr = (ctypes.c_int64 * count)()
    a.check(a.gen(preset.encode(), int(count), int(seed), int(context_cap), int(uniform_min),
                  int(uniform_max), arr))
    return list(arr)


def fit_cost_params(config, samples: Iterable[dict], _lib: Optional[_Api] = None) -> dict:
    """epp::fit_cost_params from measured (chunk, phase, seconds) samples."""
    a = _lib or api()
    out = ctypes.c_void_p()
    a.check(a.fit(_as_text(config), json.dumps(list(samples)).encode(), ctypes.byref(out)))
    return json.loads(a.take_string(out))


def render_svg(trace_doc, _lib: Optional[_Api] = None) -> str:
    a = _lib or api()
    out = ctypes.c_void_p()
    a.check(a.render(_as_text(trace_doc), ctypes.byref(out)))
    return a.take_string(out)


def system_config(*, pp_degree: int, layers: int, hidden_dim: int, mem_capacity: float,
                  token_act_bytes: float, stage_state_bytes: Sequence[float],
                  cost: dict, sp_degree: int = 1, elem_bytes: float = 2.0) -> dict:
    """Builds a SystemConfig JSON document (reference proj/src/config.cpp:76-142)."""
    return {
        "cluster": {"num_gpus": pp_degree * sp_degree, "pp_degree": pp_degree,
                    "sp_degree": sp_degree, "mem_capacity": float(mem_capacity),
                    "all2all_bandwidth": {}, "all2all_latency": {}},
        "model": {"layers": layers, "hidden_dim": hidden_dim, "elem_bytes": float(elem_bytes),
                  "token_act_bytes": float(token_act_bytes),
                  "stage_state_bytes": [float(x) for x in stage_state_bytes]},
        "cost": dict(cost),
    }
