"""Summarise an ncu capture pass (tools/ncu_capture.sh) into profiles/:
  profiles/<tag>_ncu_launches.csv      the launch list (copied)
  profiles/<tag>_ncu_full_<kernel>.csv raw-page metrics of each full capture
  profiles/ncu_summary.json            per-kernel headline counters, DRAM bytes
                                       per launch (bench.py's roofline.traffic)
                                       and each kernel's share of the launch list.
    python tools/ncu_summarize.py r01b
"""
import csv
import json
import re
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"
CLASS = {"gemm_tc2_kernel": "gemm", "gemm_tc2_wgrad": "gemm_wgrad_accum", "attn_fwd_tc": "attn_fwd",
         "attn_bwd_dq_tc": "attn_bwd_dq", "attn_bwd_dkv_tc": "attn_bwd_dkv", "norm_bwd_dx_row_k": "norm_bwd",
         "norm_fwd_row_k": "norm_fwd", "ce_k": "cross_entropy", "adamw_multi_k": "adamw"}
KEYS = {"duration": "gpu__time_duration.sum",
        "dram_read_bytes": "dram__bytes_read.sum", "dram_write_bytes": "dram__bytes_write.sum",
        "tensor_pipe_active_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smem_tc_pct": "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "smem_lsu_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "registers": "launch__registers_per_thread", "grid": "launch__grid_size",
        "sm_clock_ghz": "sm__cycles_elapsed.avg.per_second"}


def raw(rep):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    return rows[0], rows[1], rows[2:]


def main():
    tag = sys.argv[1]
    summ = {"round": 2, "tag": tag,
            "note": "ncu --set full --clock-control none, one launch per kernel class from `python bench.py "
                    "--steps 1 --warmup 1 --seqs-per-gpu 16 --prof-steps 1` (GPT-7B, github_like <= 16K, "
                    "d_p=1; tools/ncu_capture.sh); launch list: --metrics gpu__time_duration.sum, same command "
                    "(cold-cache, serialised: compare shares)",
            "kernels": {}, "dram_bytes_per_launch": {}}
    for k, cls in CLASS.items():
        rep = OUT / f"prof_{tag}_{k}.ncu-rep"
        if not rep.exists():
            continue
        hdr, units, rows = raw(rep)
        if not rows:
            continue
        d = dict(zip(hdr, rows[0]))
        u = dict(zip(hdr, units))
        with open(PROF / f"{tag}_ncu_full_{k}.csv", "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(hdr)
            w.writerow(units)
            w.writerow(rows[0])
        ent = {"name": d.get("Kernel Name", "")}
        for name, key in KEYS.items():
            if key in d:
                v = d[key]
                try:
                    v = float(v.replace(",", ""))
                except ValueError:
                    pass
                ent[name] = v
                if u.get(key):
                    ent[name + "_unit"] = u[key]
        # bytes: ncu reports in the unit shown (byte / Kbyte / Mbyte / Gbyte)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot = 0.0
        for side in ("dram_read_bytes", "dram_write_bytes"):
            if side in ent:
                tot += ent[side] * scale.get(ent.get(side + "_unit", "byte"), 1)
        summ["kernels"][k] = ent
        summ["dram_bytes_per_launch"][cls] = tot
    lst = OUT / f"launches_{tag}.csv"
    if lst.exists():
        shutil.copy(lst, PROF / f"{tag}_ncu_launches.csv")
        rows = [r for r in csv.reader(open(lst)) if len(r) > 10]
        hdr = rows[0]
        ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
        share, total = {}, 0.0
        for r in rows[1:]:
            v = float(r[iv].replace(",", ""))
            v = v / 1e6 if r[iu] in ("ns", "nsecond") else (v / 1e3 if r[iu] in ("us", "usecond") else v)
            name = re.sub(r"\(.*", "", r[ik]).replace("void ", "").split("<")[0].strip()
            e = share.setdefault(name, {"ms": 0.0, "launches": 0})
            e["ms"] += v
            e["launches"] += 1
            total += v
        for e in share.values():
            e["pct"] = round(100 * e["ms"] / total, 2)
            e["ms"] = round(e["ms"], 3)
        summ["launch_list"] = {"source": f"profiles/{tag}_ncu_launches.csv", "total_ms": round(total, 3),
                               "launches": sum(e["launches"] for e in share.values()),
                               "share": dict(sorted(share.items(), key=lambda kv: -kv[1]["ms"]))}
    (PROF / "ncu_summary.json").write_text(json.dumps(summ, indent=1))
    print(json.dumps({k: {x: v.get(x) for x in ("duration", "tensor_pipe_active_pct", "dram_throughput_pct")}
                      for k, v in summ["kernels"].items()}, indent=1))


if __name__ == "__main__":
    main()
