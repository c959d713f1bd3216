"""Idle-time breakdown of a bench step from a torch.profiler chrome trace
(`EPP_BENCH_TRACE=trace.json python bench.py ...`): kernel busy time vs span
on the busiest stream, the largest gaps and the kernels they follow, and
device time per kernel name.

    python tools/trace_gaps.py gpurun_out/trace.json [--top 20]
"""
import argparse
import collections
import json


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("trace")
    ap.add_argument("--top", type=int, default=20)
    args = ap.parse_args()
    ev = json.load(open(args.trace))
    ev = ev["traceEvents"] if isinstance(ev, dict) else ev
    kern = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    by_stream = collections.defaultdict(list)
    for e in kern:
        by_stream[(e.get("pid"), e.get("tid"))].append(e)
    sid, ks = max(by_stream.items(), key=lambda kv: sum(e["dur"] for e in kv[1]))
    ks.sort(key=lambda e: e["ts"])
    span = ks[-1]["ts"] + ks[-1]["dur"] - ks[0]["ts"]
    busy = sum(e["dur"] for e in ks)
    gaps = []
    for a, b in zip(ks, ks[1:]):
        g = b["ts"] - (a["ts"] + a["dur"])
        if g > 0:
            gaps.append((g, a["name"][:70], b["name"][:70]))
    gaps.sort(reverse=True)
    hist = collections.Counter()
    for g, _, _ in gaps:
        hist["<2us" if g < 2 else "<10us" if g < 10 else "<100us" if g < 100 else ">=100us"] += g
    per = collections.defaultdict(lambda: [0.0, 0])
    for e in ks:
        per[e["name"][:70]][0] += e["dur"]
        per[e["name"][:70]][1] += 1
    print(json.dumps({"stream": str(sid), "kernels": len(ks), "span_ms": span / 1e3, "busy_ms": busy / 1e3,
                      "idle_ms": (span - busy) / 1e3, "idle_by_gap_size_ms": {k: v / 1e3 for k, v in hist.items()},
                      "other_streams_ms": {str(k): sum(e["dur"] for e in v) / 1e3
                                           for k, v in by_stream.items() if k != sid}}, indent=1))
    print("largest gaps (us, after -> before):")
    for g, a, b in gaps[:args.top]:
        print(f"{g:9.1f}  {a}  ->  {b}")
    trans = collections.defaultdict(lambda: [0.0, 0])
    for a, b in zip(ks, ks[1:]):
        g = max(0.0, b["ts"] - (a["ts"] + a["dur"]))
        key = (a["name"].split("(")[0][-40:], b["name"].split("(")[0][-40:])
        trans[key][0] += g
        trans[key][1] += 1
    print("idle by transition (total ms, count, mean us):")
    for (a, b), (g, n) in sorted(trans.items(), key=lambda kv: -kv[1][0])[:args.top]:
        print(f"{g / 1e3:8.2f} {n:6d} {g / n:7.1f}  {a}  ->  {b}")
    # host launch vs device start: a kernel that starts right after its
    # launch call returned found the GPU idle (the host was the bottleneck)
    rt = {e["args"]["correlation"]: e for e in ev
          if e.get("ph") == "X" and e.get("cat") == "cuda_runtime" and "correlation" in e.get("args", {})}
    slack = []
    for e in ks:
        c = e.get("args", {}).get("correlation")
        if c in rt:
            slack.append(e["ts"] - (rt[c]["ts"] + rt[c]["dur"]))
    if slack:
        slack.sort()
        starved = [x for x in slack if x < 20]
        print(f"launch->start slack: n={len(slack)} median {slack[len(slack) // 2]:.0f} us, "
              f"{len(starved)} kernels started < 20 us after their launch call (host-bound)")
    print("device time by kernel (ms, launches):")
    for name, (d, n) in sorted(per.items(), key=lambda kv: -kv[1][0])[:args.top]:
        print(f"{d / 1e3:9.2f} {n:6d}  {name}")


if __name__ == "__main__":
    main()
