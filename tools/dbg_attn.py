import sys, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from test_gpu_kernels import run_attention, rel, SEGS
for case in ["multi_tile", "packed", "long"]:
    for hd, H, Hkv in [(64, 4, 4), (128, 4, 2)]:
        got, ref = run_attention("bf16", hd, H, Hkv, SEGS[case])
        o, lse, dq, dks, dvs = got; ro, rlse, rdq, rdks, rdvs = ref
        print(case, hd, H, Hkv, "dq %.4f" % rel(dq, rdq), end=" ")
        for si, (a, b, c, d) in enumerate(zip(dks, rdks, dvs, rdvs)):
            ek = ((a - b).norm(dim=(1, 2)) / (b.norm(dim=(1, 2)) + 1e-6))
            ev = ((c - d).norm(dim=(1, 2)) / (d.norm(dim=(1, 2)) + 1e-6))
            bad = (ev > 0.05).nonzero().flatten().tolist()
            print(f"| seg{si} dk {rel(a,b):.4f} dv {rel(c,d):.4f} badrows {bad[:8]}{'...' if len(bad)>8 else ''} n={len(bad)}", end=" ")
        print()
