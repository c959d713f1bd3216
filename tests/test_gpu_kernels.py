"""Kernel-level numerics on the GPU, through the C ABI (libepp_gpu.so):
tcgen05 GEMMs in every operand layout / epilogue vs a fp32 torch reference,
slice-causal attention fwd/bwd vs the fp32 oracle math."""
import ctypes
import math

import pytest
import torch

pytestmark = pytest.mark.gpu


def G():
    from paper_2509_21275_b200 import gpu
    return gpu


def ref_gemm(A, B, a_k, b_k, M, N, K):
    Am = A.float() if a_k else A.float().T
    Bm = B.float() if b_k else B.float().T
    return Am[:M, :K] @ Bm[:N, :K].T


def test_gemm_rejects_unaligned_pitch():
    g = G()
    A = torch.zeros((64, 300), device="cuda", dtype=torch.bfloat16)
    with pytest.raises(g.EppGpuError, match="multiples of 8"):
        g.check(g.lib().epp_kernel_gemm(300, 64, 64, A.data_ptr(), 300, 0, A.data_ptr(), 300, 1,
                                        A.data_ptr(), 64, None, 0, 0, 1, g.stream_ptr()))


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("a_k,b_k", [(True, True), (True, False), (False, True), (False, False)])
@pytest.mark.parametrize("M,N,K", [(256, 512, 256), (300, 384, 320), (1000, 256, 192), (4096, 1024, 1024),
                                   (2312, 4096, 576)])   # the last two take the CTA-pair (cta_group::2) kernel
def test_gemm_layouts(dtype, a_k, b_k, M, N, K):
    g = G()
    td = torch.bfloat16 if dtype == "bf16" else torch.float32
    torch.manual_seed(0)
    pad = lambda n: (n + 7) // 8 * 8   # TMA row pitch: 16-byte multiple
    A = (torch.randn((M, pad(K)) if a_k else (K, pad(M)), device="cuda") * 0.5).to(td)
    B = (torch.randn((N, pad(K)) if b_k else (K, pad(N)), device="cuda") * 0.5).to(td)
    C = torch.empty((M, N), device="cuda", dtype=td)
    lda = A.shape[1]
    ldb = B.shape[1]
    g.check(g.lib().epp_kernel_gemm(M, N, K, A.data_ptr(), lda, int(a_k), B.data_ptr(), ldb, int(b_k),
                                    C.data_ptr(), N, None, 0, 0, g.DTYPES[dtype], g.stream_ptr()))
    torch.cuda.synchronize()
    ref = ref_gemm(A, B, a_k, b_k, M, N, K)
    err = (C.float() - ref).norm() / ref.norm()
    assert err < (8e-3 if dtype == "bf16" else 1e-5), float(err)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_gemm_epilogues(dtype):
    g = G()
    td = torch.bfloat16 if dtype == "bf16" else torch.float32
    M, N, K = 384, 768, 512
    A = torch.randn((K, M), device="cuda").to(td)      # MN-major (wgrad shape)
    B = torch.randn((K, N), device="cuda").to(td)
    C = torch.randn((M, N), device="cuda", dtype=torch.float32)
    C0 = C.clone()
    g.check(g.lib().epp_kernel_gemm(M, N, K, A.data_ptr(), M, 0, B.data_ptr(), N, 0, C.data_ptr(), N,
                                    None, 0, 1, g.DTYPES[dtype], g.stream_ptr()))
    torch.cuda.synchronize()
    ref = C0 + A.float().T @ B.float()
    assert ((C - ref).norm() / ref.norm()) < (5e-3 if dtype == "bf16" else 1e-5)
    # residual add
    A2 = torch.randn((M, K), device="cuda").to(td)
    B2 = torch.randn((N, K), device="cuda").to(td)
    R = torch.randn((M, N), device="cuda").to(td)
    C2 = torch.empty((M, N), device="cuda", dtype=td)
    g.check(g.lib().epp_kernel_gemm(M, N, K, A2.data_ptr(), K, 1, B2.data_ptr(), K, 1, C2.data_ptr(), N,
                                    R.data_ptr(), N, 2, g.DTYPES[dtype], g.stream_ptr()))
    torch.cuda.synchronize()
    ref2 = A2.float() @ B2.float().T + R.float()
    assert ((C2.float() - ref2).norm() / ref2.norm()) < (8e-3 if dtype == "bf16" else 1e-5)




def test_gemm_swiglu_epilogues():
    """The fused SwiGLU epilogues at Llama-7B's FFN width (F = 11008) against
    fp64: the up-projection (tiles pair w13's gate rows j.. with its up rows
    F+j..; C = h = [g | u], C2 = silu(g) u) and the W2 data gradient (acc =
    dA; dh = [dA u silu'(g) | dA silu(g)], C2 = silu(g) u from the bf16 h)."""
    g = G()
    torch.manual_seed(4)
    M, F, D = 2000, 11008, 512
    x = torch.randn((M, D), device="cuda").bfloat16()
    w13 = (torch.randn((2 * F, D), device="cuda") * 0.05).bfloat16()
    h = torch.empty((M, 2 * F), device="cuda", dtype=torch.bfloat16)
    act = torch.empty((M, F), device="cuda", dtype=torch.bfloat16)
    g.check(g.lib().epp_kernel_gemm_ex(M, 2 * F, D, x.data_ptr(), D, 1, w13.data_ptr(), D, 1, h.data_ptr(), 2 * F,
                                       None, 0, act.data_ptr(), F, 7, g.DTYPES["bf16"], g.stream_ptr()))
    torch.cuda.synchronize()
    hd = x.double() @ w13.double().T
    assert ((h.double() - hd).norm() / hd.norm()) < 8e-3
    ga, ua = hd[:, :F], hd[:, F:]
    ref_act = torch.nn.functional.silu(ga) * ua
    assert ((act.double() - ref_act).norm() / ref_act.norm()) < 1e-2
    # backward: dA = dY W2 with W2 = [D, F] (MN-major B), R = the bf16 h
    dy = torch.randn((M, D), device="cuda").bfloat16()
    w2 = (torch.randn((D, F), device="cuda") * 0.05).bfloat16()
    dh = torch.full((M, 2 * F), 3.0, device="cuda").bfloat16()
    act2 = torch.empty((M, F), device="cuda", dtype=torch.bfloat16)
    g.check(g.lib().epp_kernel_gemm_ex(M, F, D, dy.data_ptr(), D, 1, w2.data_ptr(), F, 0, dh.data_ptr(), 2 * F,
                                       h.data_ptr(), 2 * F, act2.data_ptr(), F, 8, g.DTYPES["bf16"],
                                       g.stream_ptr()))
    torch.cuda.synchronize()
    da = dy.double() @ w2.double()
    gh, uh = h.double()[:, :F], h.double()[:, F:]
    sg = torch.sigmoid(gh)
    ref_dg = da * uh * sg * (1 + gh * (1 - sg))
    ref_du = da * gh * sg
    for got, ref in ((dh.double()[:, :F], ref_dg), (dh.double()[:, F:], ref_du), (act2.double(), gh * sg * uh)):
        assert ((got - ref).norm() / ref.norm()) < 1e-2

@pytest.mark.parametrize("ak,bk", [(1, 1), (0, 0)])
def test_gemm_pair_ragged_n(ak, bk):
    """The CTA-pair kernel with N % 256 != 0 (the LM head: N = V = 50304;
    the last column tile is half empty): K-major operands (head forward) and
    MN-major ones (weight-gradient layout), bf16 store against fp64."""
    g = G()
    torch.manual_seed(3)
    M, N, K = 1528, 50304, 512   # ragged M as well (1528 = 5 x 256 + 248)
    A = torch.randn((M, K) if ak else (K, M), device="cuda").bfloat16()
    B = (torch.randn((N, K) if bk else (K, N), device="cuda") * 0.05).bfloat16()
    C = torch.full((M, N + 32), 7.0, device="cuda").bfloat16()
    before = g.kernel_stats()
    g.check(g.lib().epp_kernel_gemm(M, N, K, A.data_ptr(), A.shape[1], ak, B.data_ptr(), B.shape[1], bk,
                                    C.data_ptr(), N + 32, None, 0, 0, g.DTYPES["bf16"], g.stream_ptr()))
    torch.cuda.synchronize()
    Ad = A.double() if ak else A.double().T
    Bd = B.double().T if bk else B.double()
    ref = Ad @ Bd
    assert ((C[:, :N].double() - ref).norm() / ref.norm()) < 8e-3
    assert torch.all(C[:, N:] == 7.0)
    after = g.kernel_stats()
    assert any("gemm_tc2_kernel<" in k and after[k] > before.get(k, 0) for k in after), "pair kernel not used"

@pytest.mark.parametrize("epi", [0, 1, 2, 3, 4, 5])
def test_gemm_pair_epilogues(epi):
    """Every epilogue on the CTA-pair kernel (>= 60 pair tiles, N % 256 == 0)
    at the GPT-1.3B up-projection / W2-dgrad widths, with a ragged M edge:
    0 Store, 1 AccumF32 (wgrad, MN-major operands), 2 AddRes, 3 StoreF32,
    4 StoreGelu (C and gelu(C)), 5 GeluBwd (C * gelu'(R) and gelu(R)).  The fp32-output
    epilogues (1, 3) are held to 1e-5 against an fp64 product of the same
    bf16 operands: only the accumulation order differs."""
    g = G()
    torch.manual_seed(1)
    M, N, K = 2200, 2048 if epi in (0, 1, 2, 3) else 8192, 768
    if epi == 1:
        A = torch.randn((K, M), device="cuda").bfloat16()
        B = torch.randn((K, N), device="cuda").bfloat16()
        # C is a column slice of a wider buffer (ldc > N): the TMA reduce-add
        # epilogue must respect the row pitch and leave the other columns alone
        Cw = torch.randn((M, N + 64), device="cuda")
        Cw0 = Cw.clone()
        g.check(g.lib().epp_kernel_gemm(M, N, K, A.data_ptr(), M, 0, B.data_ptr(), N, 0, Cw.data_ptr(), N + 64,
                                        None, 0, 1, g.DTYPES["bf16"], g.stream_ptr()))
        torch.cuda.synchronize()
        ref = Cw0[:, :N].double() + A.double().T @ B.double()
        assert ((Cw[:, :N].double() - ref).norm() / ref.norm()) < 1e-5
        assert torch.equal(Cw[:, N:], Cw0[:, N:])
        return
    A = torch.randn((M, K), device="cuda").bfloat16()
    B = torch.randn((N, K), device="cuda").bfloat16() * 0.05
    acc = A.double() @ B.double().T
    R = torch.randn((M, N), device="cuda").bfloat16()
    out_dt = torch.float32 if epi == 3 else torch.bfloat16
    C = torch.empty((M, N), device="cuda", dtype=out_dt)
    C2 = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
    g.check(g.lib().epp_kernel_gemm_ex(M, N, K, A.data_ptr(), K, 1, B.data_ptr(), K, 1, C.data_ptr(), N,
                                       R.data_ptr() if epi in (2, 5) else None, N,
                                       C2.data_ptr() if epi in (4, 5) else None, N, epi, g.DTYPES["bf16"],
                                       g.stream_ptr()))
    torch.cuda.synchronize()
    gelu = lambda x: torch.nn.functional.gelu(x, approximate="tanh")
    if epi == 0:
        checks = [(C, acc, 8e-3)]
    elif epi == 2:
        checks = [(C, acc + R.double(), 8e-3)]
    elif epi == 3:
        checks = [(C, acc, 1e-5)]
    elif epi == 4:
        checks = [(C, acc, 8e-3), (C2, gelu(acc.bfloat16().double()), 8e-3)]
    else:
        r = R.double().requires_grad_()
        gelu(r).backward(torch.ones_like(r))
        # C2: the activation gelu(R) the W2 weight gradient re-uses
        checks = [(C, acc * r.grad, 8e-3), (C2, gelu(R.double()), 8e-3)]
    for got, ref, tol in checks:
        err = float((got.double() - ref).norm() / ref.norm())
        assert err < tol, (epi, err)


def attn_reference(q, ks, vs, segs, scale):
    """fp32 reference: q [T,H,hd]; ks/vs per segment [S_i, Hkv, hd]."""
    T, H, hd = q.shape
    out = torch.zeros(T, H, hd, device=q.device)
    lse = torch.zeros(H, T, device=q.device)
    for (qs, ql, ctx), k, v in zip(segs, ks, vs):
        g = H // k.shape[1]
        kk = k.float().repeat_interleave(g, 1)
        vv = v.float().repeat_interleave(g, 1)
        s = torch.einsum("thd,shd->hts", q[qs:qs + ql].float(), kk) * scale
        qpos = torch.arange(ctx, ctx + ql, device=q.device)
        mask = torch.arange(kk.shape[0], device=q.device)[None, :] > qpos[:, None]
        s = s.masked_fill(mask[None], float("-inf"))
        lse[:, qs:qs + ql] = torch.logsumexp(s, -1) / math.log(2)
        out[qs:qs + ql] = torch.einsum("hts,shd->thd", torch.softmax(s, -1), vv)
    return out, lse


def run_attention(dtype, hd, H, Hkv, segs, seed=0):
    g = G()
    td = torch.bfloat16 if dtype == "bf16" else torch.float32
    torch.manual_seed(seed)
    T = sum(ql for (_, ql, _) in segs)
    q = torch.randn(T, H, hd, device="cuda").to(td)
    ks = [torch.randn(ctx + ql, Hkv, hd, device="cuda").to(td) for (_, ql, ctx) in segs]
    vs = [torch.randn(ctx + ql, Hkv, hd, device="cuda").to(td) for (_, ql, ctx) in segs]
    o = torch.empty(T, H, hd, device="cuda", dtype=td)
    lse = torch.empty(H, T, device="cuda")
    n = len(segs)
    I32 = ctypes.c_int32 * n
    VP = ctypes.c_void_p * n
    qs_, ql_, cx_ = I32(*[s[0] for s in segs]), I32(*[s[1] for s in segs]), I32(*[s[2] for s in segs])
    kp, vp = VP(*[k.data_ptr() for k in ks]), VP(*[v.data_ptr() for v in vs])
    scale = 1.0 / math.sqrt(hd)
    g.check(g.lib().epp_kernel_attention_fwd(T, H, Hkv, hd, scale, n, qs_, ql_, cx_, kp, vp, q.data_ptr(),
                                             o.data_ptr(), lse.data_ptr(), g.DTYPES[dtype], g.stream_ptr()))
    # backward
    do = torch.randn(T, H, hd, device="cuda").to(td)
    dks = [torch.zeros(k.shape, device="cuda") for k in ks]
    dvs = [torch.zeros(v.shape, device="cuda") for v in vs]
    dq = torch.empty(T, H, hd, device="cuda")
    FP = ctypes.c_void_p * n
    g.check(g.lib().epp_kernel_attention_bwd(T, H, Hkv, hd, scale, n, qs_, ql_, cx_, kp, vp,
                                             FP(*[d.data_ptr() for d in dks]),
                                             FP(*[d.data_ptr() for d in dvs]), q.data_ptr(), o.data_ptr(),
                                             lse.data_ptr(), do.data_ptr(), dq.data_ptr(),
                                             g.DTYPES[dtype], g.stream_ptr()))
    torch.cuda.synchronize()
    # reference with autograd
    qr = q.float().requires_grad_()
    kr = [k.float().requires_grad_() for k in ks]
    vr = [v.float().requires_grad_() for v in vs]
    ref_o, ref_lse = attn_reference(qr, kr, vr, segs, scale)
    ref_o.backward(do.float())
    return (o, lse, dq, dks, dvs), (ref_o.detach(), ref_lse.detach(), qr.grad, [k.grad for k in kr],
                                   [v.grad for v in vr])


def rel(a, b):
    return float((a.float() - b.float()).norm() / (b.float().norm() + 1e-30))


SEGS = {
    "packed": [(0, 100, 0), (100, 37, 0), (137, 200, 0), (337, 1, 0)],
    "multi_tile": [(0, 300, 0), (300, 129, 0), (429, 257, 600)],
    "slice_ctx": [(0, 150, 333)],
    "hybrid": [(0, 90, 1000), (90, 64, 0), (154, 17, 0)],
    "long": [(0, 1024, 2048)],
}


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("hd,H,Hkv", [(64, 4, 4), (128, 4, 2), (128, 8, 8), (128, 8, 2)])
@pytest.mark.parametrize("case", list(SEGS))
def test_attention(dtype, hd, H, Hkv, case):
    got, ref = run_attention(dtype, hd, H, Hkv, SEGS[case])
    check_attention(got, ref, dtype)


def check_attention(got, ref, dtype):
    tol = 2e-2 if dtype == "bf16" else 1e-4
    o, lse, dq, dks, dvs = got
    ro, rlse, rdq, rdks, rdvs = ref
    assert rel(o, ro) < tol, ("o", rel(o, ro))
    assert (lse - rlse).abs().max() < (2e-2 if dtype == "bf16" else 1e-4)
    assert rel(dq, rdq) < 2 * tol, ("dq", rel(dq, rdq))
    # a 1-token segment has exactly-zero dK: measure over all segments
    cat = lambda xs: torch.cat([x.reshape(-1) for x in xs])
    assert rel(cat(dks), cat(rdks)) < 2 * tol, ("dk", rel(cat(dks), cat(rdks)))
    assert rel(cat(dvs), cat(rdvs)) < 2 * tol, ("dv", rel(cat(dvs), cat(rdvs)))


@pytest.mark.parametrize("H,Hkv", [(8, 2), (32, 8)])
@pytest.mark.parametrize("case", ["ctx32k", "hybrid32k"])
def test_attention_long_context(H, Hkv, case):
    """The benchmark's regime: a late slice of a 32K sequence (queries at
    positions 31K..32K over the whole cached context) and a hybrid chunk whose
    tail slice sits at 16K context followed by packed documents; GQA 4:1 as
    in Llama-7B (32 query / 8 KV heads), head_dim 128, tcgen05 kernels."""
    segs = {"ctx32k": [(0, 1024, 31744)],
            "hybrid32k": [(0, 700, 16384), (700, 1500, 0), (2200, 301, 0)]}[case]
    got, ref = run_attention("bf16", 128, H, Hkv, segs, seed=3)
    check_attention(got, ref, "bf16")
