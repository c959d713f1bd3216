"""One-screen summary of bench.py JSON lines: value, MFU, clocks and the
per-class kernel times.   python tools/bench_brief.py file.json [...]"""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    print(f"{f}: {d['value']:.0f} tok/s  e2e {(d.get('e2e') or {}).get('value', 0):.0f}  mfu {d.get('mfu', 0):.3f}  "
          f"{d['ms_per_step']:.0f} ms/step  clock {d.get('clocks', {}).get('sm_mhz')}  "
          f"ckpt {d['config'].get('ckpt_layers_per_step')}  loss {d.get('loss', 0):.4f}")
    for k, v in d.get("kernel_classes", {}).items():
        if v.get("ms_per_step"):
            rate = f"{v['tflops']:.0f} TF/s" if "tflops" in v else f"{v.get('gbs', 0):.0f} GB/s"
            print(f"   {k:18s} {v['ms_per_step']:8.1f} ms  {rate:>12s}  x{v['launches_per_step']:.0f}")
    print(f"   unattributed {d.get('unattributed_ms_per_step', 0):.1f} ms")
