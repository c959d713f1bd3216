"""Warp-stall samples of one kernel in an ncu report, attributed to CUDA
source lines (needs -lineinfo + --import-source):
    python tools/ncu_lines.py report.ncu-rep kernel_regex [top]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda", "-k",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = None
per_line = defaultdict(lambda: [0, 0, ""])
cur_line, cur_src = None, ""
for r in rows:
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 5:
        continue
    if r[0]:
        cur_line, cur_src = r[0], r[1]
    try:
        s_all, s_ni = int(r[4] or 0), int(r[5] or 0)
    except ValueError:
        continue
    e = per_line[cur_line]
    e[0] += s_all
    e[1] += s_ni
    e[2] = cur_src
tot = sum(v[0] for v in per_line.values())
print("total samples", tot)
for line, (a, n, src) in sorted(per_line.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{a:7d} {100.0 * a / max(1, tot):5.1f}%  L{line:5s} {src.strip()[:100]}")
