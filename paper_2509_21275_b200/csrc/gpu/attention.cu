// epp-b200: slice-causal attention dispatch + the fp32 parity kernels.
//
// A chunk is a list of segments (kernels.h: AttnSeg).  Segment 0 of a
// Split/Hybrid chunk is a slice of a long sequence: its queries sit at key
// positions [C, C+s0) of the sequence's per-stage KV buffer, so they attend
// to the C context keys written by earlier chunks plus their own causal
// prefix.  Every other segment is an independent packed document (C = 0,
// chunk-local K/V).  This replaces flash-attn's varlen `cu_seqlens` with a
// table that also carries the context offset and K/V base pointers, so one
// launch covers a Batched, Split or Hybrid chunk (paper §3, PAPER.md:180-181;
// cost model cost_model.cpp:18 charges exactly these (C+s0)^2 - C^2 pairs).
//
// bf16 (the product path): the tcgen05 kernels of attention_tc.cu, the only
// bf16 implementation.  fp32 (the parity mode checked against the fp32
// oracle at 1e-3): warp-per-row SIMT kernels below, same math:
//   fwd : grid (query blocks, H)           -> O, LSE (log2 domain)
//   dq  : grid (query blocks, H)           -> dQ (fp32), no atomics
//   dkv : grid (key blocks, Hkv)           -> dK/dV += (fp32 RMW into the
//         segment's accumulator; each key block is owned by one CTA, GQA
//         heads are looped inside the CTA, so no atomics and deterministic)
// The dK/dV accumulators of a split sequence persist across its chunks:
// later slices' backwards (which run first) add into earlier slices' keys.
#include "common.cuh"
#include "kernels.h"
#include "profile.h"

namespace eppk {

namespace {

constexpr int BM = kAttnBlock;    // query rows per CTA
constexpr int BN = kAttnBlock;    // keys per tile
constexpr float kLog2e = 1.4426950408889634f;

// delta[h, t] = sum_d dO[t,h,d] * O[t,h,d]   (one warp per (t, h))
template <typename T>
__global__ void attn_delta_kernel(const T* dout, const T* out, float* delta, int Tn, int H,
                                  int hd) {
    pdl_wait();
    pdl_trigger();
    const long long wid = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= static_cast<long long>(Tn) * H) return;
    const long long t = wid / H;
    const int h = static_cast<int>(wid % H);
    const T* a = dout + (t * H + h) * hd;
    const T* b = out + (t * H + h) * hd;
    float s = 0.f;
    for (int d = lane; d < hd; d += 32) s += to_f(a[d]) * to_f(b[d]);
    s = warp_sum(s);
    if (lane == 0) delta[static_cast<long long>(h) * Tn + t] = s;
}

// ------------------------------------------------------- F32 (parity) ----
// One warp per query row; lanes split the head dimension.
__global__ void attn_fwd_f32(const AttnArgs a) {
    pdl_wait();
    pdl_trigger();
    const AttnWork w = a.qwork[blockIdx.x];
    const AttnSeg sg = a.segs[w.seg];
    const int h = blockIdx.y, kvh = h / (a.H / a.Hkv);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int hd = a.hd;
    const long long kvs = static_cast<long long>(a.Hkv) * hd;
    const float* K = static_cast<const float*>(sg.k) + a.layer * sg.kv_layer_stride + kvh * hd;
    const float* V = static_cast<const float*>(sg.v) + a.layer * sg.kv_layer_stride + kvh * hd;
    const float c2 = a.scale * kLog2e;
    for (int r = warp; r < BM; r += blockDim.x / 32) {
        const int qi = w.block * BM + r;
        if (qi >= sg.q_len) break;
        const long long t = sg.q_start + qi;
        const float* q = static_cast<const float*>(a.q) + (t * a.H + h) * hd;
        float qv[4], ov[4] = {0.f, 0.f, 0.f, 0.f};
        for (int i = 0; i < 4; ++i) qv[i] = (lane + 32 * i < hd) ? q[lane + 32 * i] : 0.f;
        float m = -INFINITY, l = 0.f;
        const int last = sg.kv_ctx + qi;
        for (int j = 0; j <= last; ++j) {
            float d = 0.f;
            for (int i = 0; i < 4; ++i)
                if (lane + 32 * i < hd) d += qv[i] * K[j * kvs + lane + 32 * i];
            const float s = warp_sum(d) * c2;
            const float mn = fmaxf(m, s);
            const float al = exp2f(m - mn), p = exp2f(s - mn);
            l = l * al + p;
            for (int i = 0; i < 4; ++i)
                if (lane + 32 * i < hd) ov[i] = ov[i] * al + p * V[j * kvs + lane + 32 * i];
            m = mn;
        }
        float* o = static_cast<float*>(a.o) + (t * a.H + h) * hd;
        for (int i = 0; i < 4; ++i)
            if (lane + 32 * i < hd) o[lane + 32 * i] = ov[i] / l;
        if (lane == 0) a.lse[static_cast<long long>(h) * a.T + t] = m + log2f(l);
    }
}

__global__ void attn_bwd_dq_f32(const AttnArgs a) {
    pdl_wait();
    pdl_trigger();
    const AttnWork w = a.qwork[blockIdx.x];
    const AttnSeg sg = a.segs[w.seg];
    const int h = blockIdx.y, kvh = h / (a.H / a.Hkv);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int hd = a.hd;
    const long long kvs = static_cast<long long>(a.Hkv) * hd;
    const float* K = static_cast<const float*>(sg.k) + a.layer * sg.kv_layer_stride + kvh * hd;
    const float* V = static_cast<const float*>(sg.v) + a.layer * sg.kv_layer_stride + kvh * hd;
    const float c2 = a.scale * kLog2e;
    for (int r = warp; r < BM; r += blockDim.x / 32) {
        const int qi = w.block * BM + r;
        if (qi >= sg.q_len) break;
        const long long t = sg.q_start + qi;
        const float* q = static_cast<const float*>(a.q) + (t * a.H + h) * hd;
        const float* go = static_cast<const float*>(a.dout) + (t * a.H + h) * hd;
        const float lse = a.lse[static_cast<long long>(h) * a.T + t];
        const float dl = a.delta[static_cast<long long>(h) * a.T + t];
        float qv[4], gv[4], dq[4] = {0.f, 0.f, 0.f, 0.f};
        for (int i = 0; i < 4; ++i) {
            const bool ok = lane + 32 * i < hd;
            qv[i] = ok ? q[lane + 32 * i] : 0.f;
            gv[i] = ok ? go[lane + 32 * i] : 0.f;
        }
        const int last = sg.kv_ctx + qi;
        for (int j = 0; j <= last; ++j) {
            float d = 0.f, e = 0.f;
            for (int i = 0; i < 4; ++i)
                if (lane + 32 * i < hd) {
                    d += qv[i] * K[j * kvs + lane + 32 * i];
                    e += gv[i] * V[j * kvs + lane + 32 * i];
                }
            const float s = warp_sum(d), dp = warp_sum(e);
            const float p = exp2f(s * c2 - lse);
            const float ds = p * (dp - dl);
            for (int i = 0; i < 4; ++i)
                if (lane + 32 * i < hd) dq[i] += ds * K[j * kvs + lane + 32 * i];
        }
        float* out = a.dq + (t * a.H + h) * hd;
        for (int i = 0; i < 4; ++i)
            if (lane + 32 * i < hd) out[lane + 32 * i] = dq[i] * a.scale;
    }
}

__global__ void attn_bwd_dkv_f32(const AttnArgs a) {
    pdl_wait();
    pdl_trigger();
    const AttnWork w = a.kwork[blockIdx.x];
    const AttnSeg sg = a.segs[w.seg];
    const int kvh = blockIdx.y, group = a.H / a.Hkv;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int hd = a.hd;
    const long long kvs = static_cast<long long>(a.Hkv) * hd;
    const float* K = static_cast<const float*>(sg.k) + a.layer * sg.kv_layer_stride + kvh * hd;
    const float* V = static_cast<const float*>(sg.v) + a.layer * sg.kv_layer_stride + kvh * hd;
    float* DK = sg.dk + a.layer * sg.dkv_layer_stride + kvh * hd;
    float* DV = sg.dv + a.layer * sg.dkv_layer_stride + kvh * hd;
    const float c2 = a.scale * kLog2e;
    const int kv_len = sg.kv_ctx + sg.q_len;
    for (int r = warp; r < BN; r += blockDim.x / 32) {
        const int j = w.block * BN + r;
        if (j >= kv_len) break;
        float kv[4], vv[4], dk[4] = {0.f, 0.f, 0.f, 0.f}, dv[4] = {0.f, 0.f, 0.f, 0.f};
        for (int i = 0; i < 4; ++i) {
            const bool ok = lane + 32 * i < hd;
            kv[i] = ok ? K[j * kvs + lane + 32 * i] : 0.f;
            vv[i] = ok ? V[j * kvs + lane + 32 * i] : 0.f;
        }
        const int qi0 = max(0, j - sg.kv_ctx);
        for (int hq = kvh * group; hq < (kvh + 1) * group; ++hq)
            for (int qi = qi0; qi < sg.q_len; ++qi) {
                const long long t = sg.q_start + qi;
                const float* q = static_cast<const float*>(a.q) + (t * a.H + hq) * hd;
                const float* go = static_cast<const float*>(a.dout) + (t * a.H + hq) * hd;
                float d = 0.f, e = 0.f;
                for (int i = 0; i < 4; ++i)
                    if (lane + 32 * i < hd) {
                        d += q[lane + 32 * i] * kv[i];
                        e += go[lane + 32 * i] * vv[i];
                    }
                const float s = warp_sum(d), dp = warp_sum(e);
                const float p = exp2f(s * c2 - a.lse[static_cast<long long>(hq) * a.T + t]);
                const float ds = p * (dp - a.delta[static_cast<long long>(hq) * a.T + t]);
                for (int i = 0; i < 4; ++i)
                    if (lane + 32 * i < hd) {
                        dv[i] += p * go[lane + 32 * i];
                        dk[i] += ds * q[lane + 32 * i];
                    }
            }
        for (int i = 0; i < 4; ++i)
            if (lane + 32 * i < hd) {
                DK[j * kvs + lane + 32 * i] += dk[i] * a.scale;
                DV[j * kvs + lane + 32 * i] += dv[i];
            }
    }
}

}  // namespace

void attn_delta(const AttnArgs& a, cudaStream_t s) {
    if (a.T <= 0) return;
    const long long warps = static_cast<long long>(a.T) * a.H;
    const int blocks = static_cast<int>((warps * 32 + 255) / 256);
    if (a.dtype == DType::F32)
        launch_k(attn_delta_kernel<float>, blocks, 256, 0, s, static_cast<const float*>(a.dout),
                                                        static_cast<const float*>(a.o), a.delta, a.T, a.H, a.hd);
    else
        launch_k(attn_delta_kernel<bf16>, blocks, 256, 0, s, static_cast<const bf16*>(a.dout),
                                                       static_cast<const bf16*>(a.o), a.delta, a.T, a.H, a.hd);
    EPP_CHECK_LAUNCH();
}

void attn_fwd(const AttnArgs& a, cudaStream_t s) {
    EPP_REQUIRE(a.H % a.Hkv == 0, "attn: H must be a multiple of Hkv");
    if (a.nqwork == 0) return;
    if (a.dtype == DType::BF16) {
        EPP_REQUIRE(attn_fwd_tc_supported(a), "attn(bf16): needs head_dim 64/128 and the TMA maps");
        attn_fwd_tc(a, s);
        return;
    }
    ProfScope prof(kProfAttnFwd, 4.0 * a.H * a.hd * a.pairs, s);
    EPP_REQUIRE(a.hd <= 128, "attn(f32): head_dim <= 128");
    launch_k(attn_fwd_f32, dim3(a.nqwork, a.H), 128, 0, s, a);
    EPP_CHECK_LAUNCH();
}

void attn_bwd(const AttnArgs& a, cudaStream_t s) {
    EPP_REQUIRE(a.H % a.Hkv == 0, "attn: H must be a multiple of Hkv");
    // algorithmic backward = 2x forward (dQ, dK, dV, dP matmuls)
    ProfScope prof(kProfAttnBwd, 8.0 * a.H * a.hd * a.pairs, s);
    if (a.dtype == DType::BF16) {
        EPP_REQUIRE(attn_bwd_tc_supported(a), "attn(bf16): needs head_dim 64/128 and the TMA maps");
        attn_bwd_tc_main(a, s);      // the dQ kernel forms delta itself
        return;
    }
    attn_delta(a, s);
    EPP_REQUIRE(a.dqkv_out == nullptr, "attn_bwd: dqkv_out needs the tcgen05 kernels");
    if (a.nqwork > 0) {
        launch_k(attn_bwd_dq_f32, dim3(a.nqwork, a.H), 128, 0, s, a);
        EPP_CHECK_LAUNCH();
    }
    if (a.nkwork > 0) {
        launch_k(attn_bwd_dkv_f32, dim3(a.nkwork, a.Hkv), 128, 0, s, a);
        EPP_CHECK_LAUNCH();
    }
}

}  // namespace eppk
