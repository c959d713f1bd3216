"""Generates the committed golden fixtures from the REFERENCE planner
(oracle/_ref/libepp_ref.so, compiled from /root/reference by oracle/Makefile).

    python tests/golden/make_golden.py

Each fixture stores the inputs and the reference's exact output bytes; the
product library must reproduce them byte for byte (tests/test_golden.py),
including on the GPU box where /root/reference does not exist."""
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

from paper_2509_21275_b200 import model as M  # noqa: E402
from paper_2509_21275_b200 import planner as P  # noqa: E402

REF = P._Api(ROOT / "oracle" / "_ref" / "libepp_ref.so", prefix="epp_ref_")

DESK8 = {"cluster": {"num_gpus": 32, "pp_degree": 8, "sp_degree": 4, "mem_capacity": 80e9,
                     "all2all_bandwidth": {"2": 2.4e11, "4": 1.5e11, "8": 1.1e11},
                     "all2all_latency": {"2": 1.5e-5, "4": 3e-5, "8": 5e-5}},
         "model": {"layers": 48, "hidden_dim": 6144, "elem_bytes": 2, "token_act_bytes": 1.1796480e7,
                   "stage_state_bytes": [15.5e9, 15e9, 15e9, 15e9, 15e9, 15e9, 15e9, 15.3e9]},
         "cost": {"fwd_sec_per_token2": 3.78e-10, "fwd_sec_per_token": 2.787e-4, "fwd_sec_fixed": 6e-4,
                  "bwd_sec_per_token2": 7.56e-10, "bwd_sec_per_token": 5.574e-4, "bwd_sec_fixed": 1.2e-3,
                  "layer_fwd_seconds": 0}}
TIGHT8 = json.loads(json.dumps(DESK8))
TIGHT8["cluster"]["mem_capacity"] = 40e9
WORKED = {"cluster": {"num_gpus": 2, "pp_degree": 2, "sp_degree": 1, "mem_capacity": 1e12,
                      "all2all_bandwidth": {}, "all2all_latency": {}},
          "model": {"layers": 4, "hidden_dim": 256, "elem_bytes": 2, "token_act_bytes": 1e5,
                    "stage_state_bytes": [2e9, 2e9]},
          "cost": {"fwd_sec_per_token2": 1e-9, "fwd_sec_per_token": 1e-5, "fwd_sec_fixed": 2e-3,
                   "bwd_sec_per_token2": 2e-9, "bwd_sec_per_token": 2e-5, "bwd_sec_fixed": 4e-3,
                   "layer_fwd_seconds": 0}}


def cases():
    out = []
    out.append(("worked_example", WORKED, [9000, 300, 200, 1500, 700], 3, "main"))
    tiny = M.planner_config(M.MODELS["tiny"], 2, mem_capacity=180e9)
    out.append(("tiny_cpu_case", tiny, P.generate_workload("uniform", 64, 0, 4096, 128, 4096, _lib=REF), None, "main"))
    for seed in (0, 1):
        lens = P.generate_workload("github_like", 96, seed, 196608, _lib=REF)
        out.append((f"desk8_s{seed}", DESK8, lens, None, "main"))
        out.append((f"tight8_s{seed}", TIGHT8, lens, None, "main"))
    lens = P.generate_workload("github_like", 64, 5, 65536, _lib=REF)
    for mode in ("no_wbc", "no_ckpt", "full_ckpt"):
        out.append((f"desk8_{mode}", DESK8, lens, 4, mode))
    g13 = M.planner_config(M.MODELS["gpt-1.3b"], 8, mem_capacity=180e9)
    out.append(("gpt13b_pp8", g13, P.generate_workload("github_like", 128, 3, 32768, _lib=REF), None, "main"))
    l7 = M.planner_config(M.MODELS["llama-7b"], 8, mem_capacity=80e9)
    out.append(("llama7b_64k_s8", l7, P.generate_workload("github_like", 64, 4, 65536, _lib=REF), 8, "main"))
    return out


def main():
    fixtures = []
    for name, cfg, lengths, slices, mode in cases():
        try:
            doc = P.make_plan_document(cfg, lengths, slices, mode, 4, _lib=REF)
            err = None
        except P.Error as e:
            doc, err = None, [type(e).__name__, str(e)]
        trace = None
        if doc is not None and name in ("worked_example", "tiny_cpu_case", "desk8_s0"):
            trace, total = P.simulate_plan_document(doc, _lib=REF)
        fixtures.append({"name": name, "config": cfg, "lengths": list(map(int, lengths)), "slices": slices,
                         "mode": mode, "plan": doc, "error": err, "trace": trace})
    work = {f"github_like_{s}": P.generate_workload("github_like", 512, s, 196608, _lib=REF) for s in (0, 1)}
    work["commoncrawl_like_7"] = P.generate_workload("commoncrawl_like", 300, 7, 131072, _lib=REF)
    work["uniform_3"] = P.generate_workload("uniform", 100, 3, 8192, 100, 0, _lib=REF)
    (HERE / "planner_fixtures.json").write_text(json.dumps({"fixtures": fixtures, "workloads": work}))
    print(f"wrote {len(fixtures)} plan fixtures, {len(work)} workloads")


if __name__ == "__main__":
    main()
