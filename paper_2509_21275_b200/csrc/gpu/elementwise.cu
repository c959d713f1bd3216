// epp-b200: HBM-bound kernels of the stage executor — embedding, LayerNorm /
// RMSNorm (fwd, bwd with fused residual add, recompute), RoPE + QKV scatter
// into the per-segment KV rows and its inverse gather, GELU / SwiGLU, fused
// softmax cross-entropy, AdamW and initialisation.  All are vectorised
// (16-byte accesses), one CTA per row where a row reduction is needed.
#include <type_traits>

#include "common.cuh"
#include "kernels.h"
#include "profile.h"

namespace eppk {

namespace {

// ---- 8-wide vector load/store for float and bf16 -----------------------
__device__ __forceinline__ void load8(const float* p, float (&v)[8]) {
    const float4 a = *reinterpret_cast<const float4*>(p);
    const float4 b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void load8(const bf16* p, float (&v)[8]) {
    const uint4 raw = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(h[i]);
        v[2 * i] = f.x;
        v[2 * i + 1] = f.y;
    }
}
__device__ __forceinline__ void store8(float* p, const float (&v)[8]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
}
__device__ __forceinline__ void store8(bf16* p, const float (&v)[8]) {
    uint4 raw;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    *reinterpret_cast<uint4*>(p) = raw;
}

template <typename F>
void dispatch_t(DType t, F&& f) {
    if (t == DType::F32) f(float{});
    else f(bf16{});
}

int grid_for(long long n, int threads) {
    const long long b = (n + threads - 1) / threads;
    return static_cast<int>(b < 1 ? 1 : (b > 1048576 ? 1048576 : b));
}

// ------------------------------------------------------------ embedding ---
template <typename T>
__global__ void embed_fwd_k(const int32_t* ids, const T* table, T* out, int Tn, int D) {
    pdl_wait();
    pdl_trigger();
    const int t = blockIdx.x;
    const T* src = table + static_cast<long long>(ids[t]) * D;
    T* dst = out + static_cast<long long>(t) * D;
    for (int c = threadIdx.x * 8; c < D; c += blockDim.x * 8) {
        float v[8];
        load8(src + c, v);
        store8(dst + c, v);
    }
}
template <typename T>
__global__ void embed_bwd_k(const int32_t* ids, const T* dout, float* dtable, int Tn, int D) {
    pdl_wait();
    pdl_trigger();
    const int t = blockIdx.x;
    float* dst = dtable + static_cast<long long>(ids[t]) * D;
    const T* src = dout + static_cast<long long>(t) * D;
    for (int c = threadIdx.x * 8; c < D; c += blockDim.x * 8) {
        float v[8];
        load8(src + c, v);
#pragma unroll
        for (int i = 0; i < 8; ++i) atomicAdd(dst + c + i, v[i]);
    }
}

// ---------------------------------------------------------------- norms ---
// One CTA per row, two passes (mean, then centred variance), fp32 math.
template <typename T>
__global__ void norm_fwd_k(bool rms, const T* x, const T* w, const T* b, T* y, float* mean,
                           float* rstd, int D, float eps) {
    pdl_wait();
    pdl_trigger();
    __shared__ float scratch[32];
    const long long row = blockIdx.x;
    const T* xr = x + row * D;
    float s = 0.f;
    for (int c = threadIdx.x * 8; c < D; c += blockDim.x * 8) {
        float v[8];
        load8(xr + c, v);
#pragma unroll
        for (int i = 0; i < 8; ++i) s += v[i];
    }
    const float mu = rms ? 0.f : block_sum(s, scratch) / D;
    float q = 0.f;
    for (int c = threadIdx.x * 8; c < D; c += blockDim.x * 8) {
        float v[8];
        load8(xr + c, v);
#pragma unroll
        for (int i = 0; i < 8; ++i) q += (v[i] - mu) * (v[i] - mu);
    }
    const float rs = rsqrtf(block_sum(q, scratch) / D + eps);
    if (threadIdx.x == 0) {
        if (mean) mean[row] = mu;
        rstd[row] = rs;
    }
    for (int c = threadIdx.x * 8; c < D; c += blockDim.x * 8) {
        float v[8], wv[8], bv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        load8(xr + c, v);
        load8(w + c, wv);
        if (b) load8(b + c, bv);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = (v[i] - mu) * rs * wv[i] + bv[i];
        store8(y + row * D + c, v);
    }
}

// Warp-per-row variant (bf16, D = 256 * NC, the model widths): the row stays
// in registers as packed bf16 between the mean, variance and normalise passes
// (one HBM read), reductions are warp shuffles only.
template <int NC>
__global__ void __launch_bounds__(256) norm_fwd_warp_k(bool rms, const bf16* x, const bf16* w, const bf16* b,
                                                       bf16* y, float* mean, float* rstd, int Tn, float eps) {
    pdl_wait();
    pdl_trigger();
    constexpr int D = 256 * NC;
    const int lane = threadIdx.x & 31;
    const long long row = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (row >= Tn) return;
    const bf16* xr = x + row * D;
    uint4 raw[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) raw[k] = *reinterpret_cast<const uint4*>(xr + k * 256 + lane * 8);
    auto unpack = [](const uint4& r, float (&v)[8]) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = __bfloat1622float2(h[i]);
            v[2 * i] = f.x;
            v[2 * i + 1] = f.y;
        }
    };
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        float v[8];
        unpack(raw[k], v);
#pragma unroll
        for (int i = 0; i < 8; ++i) s += v[i];
    }
    // keep the row packed between passes (re-expanding is cheaper than 8 NC
    // live fp32 registers per lane)
    auto pin = [&]() {
#pragma unroll
        for (int k = 0; k < NC; ++k) asm volatile("" : "+r"(raw[k].x), "+r"(raw[k].y), "+r"(raw[k].z), "+r"(raw[k].w));
    };
    pin();
    const float mu = rms ? 0.f : warp_sum(s) / D;
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        float v[8];
        unpack(raw[k], v);
#pragma unroll
        for (int i = 0; i < 8; ++i) q += (v[i] - mu) * (v[i] - mu);
    }
    pin();
    const float rs = rsqrtf(warp_sum(q) / D + eps);
    if (lane == 0) {
        if (mean) mean[row] = mu;
        rstd[row] = rs;
    }
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        const int c = k * 256 + lane * 8;
        float v[8], wv[8], bv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        unpack(raw[k], v);
        load8(w + c, wv);
        if (b) load8(b + c, bv);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = (v[i] - mu) * rs * wv[i] + bv[i];
        store8(y + row * D + c, v);
    }
}

// CTA-per-row variants (bf16, D = 1024 * NPT): 128 threads, each holding
// NPT packed 16-byte chunks of the row in registers (one HBM read), a
// 4-warp shuffle + shared-memory reduction.  Small register footprint, so
// many rows are in flight per SM even for short chunks.
__device__ __forceinline__ void unpack8(const uint4& r, float (&v)[8]) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(h[i]);
        v[2 * i] = f.x;
        v[2 * i + 1] = f.y;
    }
}
__device__ __forceinline__ float sum128(float v, float* red) {   // 4-warp CTA sum
    v = warp_sum(v);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    return (red[0] + red[1]) + (red[2] + red[3]);
}

template <int NPT>
__global__ void __launch_bounds__(128) norm_fwd_row_k(bool rms, const bf16* x, const bf16* w, const bf16* b, bf16* y,
                                                      float* mean, float* rstd, float eps) {
    pdl_wait();
    pdl_trigger();
    constexpr int D = 1024 * NPT;
    __shared__ float red[4];
    const long long row = blockIdx.x;
    const bf16* xr = x + row * D;
    uint4 raw[NPT];
#pragma unroll
    for (int k = 0; k < NPT; ++k) raw[k] = *reinterpret_cast<const uint4*>(xr + k * 1024 + threadIdx.x * 8);
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        float v[8];
        unpack8(raw[k], v);
#pragma unroll
        for (int i = 0; i < 8; ++i) s += v[i];
    }
    const float mu = rms ? 0.f : sum128(s, red) / D;
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        float v[8];
        unpack8(raw[k], v);
#pragma unroll
        for (int i = 0; i < 8; ++i) q += (v[i] - mu) * (v[i] - mu);
    }
    const float rs = rsqrtf(sum128(q, red) / D + eps);
    if (threadIdx.x == 0) {
        if (mean) mean[row] = mu;
        rstd[row] = rs;
    }
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        const int c = k * 1024 + threadIdx.x * 8;
        float v[8], wv[8], bv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        unpack8(raw[k], v);
        load8(w + c, wv);
        if (b) load8(b + c, bv);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = (v[i] - mu) * rs * wv[i] + bv[i];
        store8(y + row * D + c, v);
    }
}

template <int NPT>
__global__ void __launch_bounds__(128) norm_bwd_dx_row_k(bool rms, const bf16* x, const bf16* w, const bf16* dy,
                                                         const float* mean, const float* rstd, const bf16* dres,
                                                         bf16* dx, const bf16* bias, bf16* xn_out) {
    pdl_wait();
    pdl_trigger();
    constexpr int D = 1024 * NPT;
    __shared__ float red[2][4];
    const long long row = blockIdx.x;
    const long long off = row * D;
    uint4 rx[NPT], rg[NPT];
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        rx[k] = *reinterpret_cast<const uint4*>(x + off + k * 1024 + threadIdx.x * 8);
        rg[k] = *reinterpret_cast<const uint4*>(dy + off + k * 1024 + threadIdx.x * 8);
    }
    const float mu = rms ? 0.f : mean[row];
    const float rs = rstd[row];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        float xv[8], gv[8], wv[8];
        unpack8(rx[k], xv);
        unpack8(rg[k], gv);
        load8(w + k * 1024 + threadIdx.x * 8, wv);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float dxh = gv[i] * wv[i];
            s1 += dxh;
            s2 += dxh * (xv[i] - mu) * rs;
        }
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = s1;
        red[1][threadIdx.x >> 5] = s2;
    }
    __syncthreads();
    const float m1 = rms ? 0.f : ((red[0][0] + red[0][1]) + (red[0][2] + red[0][3])) / D;
    const float m2 = ((red[1][0] + red[1][1]) + (red[1][2] + red[1][3])) / D;
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        const int c = k * 1024 + threadIdx.x * 8;
        float xv[8], gv[8], wv[8], out[8], rv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        unpack8(rx[k], xv);
        unpack8(rg[k], gv);
        load8(w + c, wv);
        if (dres) load8(dres + off + c, rv);
#pragma unroll
        for (int i = 0; i < 8; ++i) out[i] = rv[i] + rs * (gv[i] * wv[i] - m1 - (xv[i] - mu) * rs * m2);
        store8(dx + off + c, out);
        if (xn_out) {   // y = norm(x) from the registers already holding x
            float bv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            if (bias) load8(bias + c, bv);
#pragma unroll
            for (int i = 0; i < 8; ++i) out[i] = (xv[i] - mu) * rs * wv[i] + bv[i];
            store8(xn_out + off + c, out);
        }
    }
}

template <typename T>
__global__ void norm_apply_k(bool rms, const T* x, const T* w, const T* b, const float* mean,
                             const float* rstd, T* y, int D) {
    pdl_wait();
    pdl_trigger();
    const long long row = blockIdx.x;
    const float mu = rms ? 0.f : mean[row];
    const float rs = rstd[row];
    for (int c = threadIdx.x * 8; c < D; c += blockDim.x * 8) {
        float v[8], wv[8], bv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        load8(x + row * D + c, v);
        load8(w + c, wv);
        if (b) load8(b + c, bv);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = (v[i] - mu) * rs * wv[i] + bv[i];
        store8(y + row * D + c, v);
    }
}

constexpr int kNormMaxG = 8;         // D <= 8192 (checked by the launcher)

// dx = dres + rstd * (dy*w - mean(dy*w) - xhat * mean(dy*w*xhat)): one warp per
// row, two sweeps over the row (the second re-reads from L1/L2), warp
// shuffles only — no shared memory, no block barriers.
template <typename T>
__global__ void __launch_bounds__(256) norm_bwd_dx_k(bool rms, const T* x, const T* w, const T* dy,
                                                     const float* mean, const float* rstd,
                                                     const T* dres, T* dx, int Tn, int D) {
    pdl_wait();
    pdl_trigger();
    const int lane = threadIdx.x & 31;
    const long long row = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (row >= Tn) return;
    const long long off = row * D;
    const float mu = rms ? 0.f : mean[row];
    const float rs = rstd[row];
    float s1 = 0.f, s2 = 0.f;
    for (int c = lane * 8; c < D; c += 256) {
        float xv[8], wv[8], gv[8];
        load8(x + off + c, xv);
        load8(w + c, wv);
        load8(dy + off + c, gv);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float dxh = gv[i] * wv[i];
            s1 += dxh;
            s2 += dxh * (xv[i] - mu) * rs;
        }
    }
    const float m1 = rms ? 0.f : warp_sum(s1) / D;
    const float m2 = warp_sum(s2) / D;
    for (int c = lane * 8; c < D; c += 256) {
        float xv[8], wv[8], gv[8], out[8], rv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        load8(x + off + c, xv);
        load8(w + c, wv);
        load8(dy + off + c, gv);
        if (dres) load8(dres + off + c, rv);
#pragma unroll
        for (int i = 0; i < 8; ++i) out[i] = rv[i] + rs * (gv[i] * wv[i] - m1 - (xv[i] - mu) * rs * m2);
        store8(dx + off + c, out);
    }
}

// Partial dγ/dβ, one partial row per CTA: 32 column groups (8 columns each)
// x 8 row groups; the row groups are combined in shared memory.
template <typename T>
__global__ void __launch_bounds__(256) norm_bwd_dw2_k(bool rms, const T* x, const T* dy, const float* mean,
                                                      const float* rstd, float* pw, float* pb, int Tn, int D,
                                                      int rows_per) {
    pdl_wait();
    pdl_trigger();
    __shared__ float red[2][8][256 + 8];
    const int cx = threadIdx.x & 31, ry = threadIdx.x >> 5;
    const int c = blockIdx.x * 256 + cx * 8;
    const int r0 = blockIdx.y * rows_per, r1 = min(Tn, r0 + rows_per);
    float aw[8] = {0, 0, 0, 0, 0, 0, 0, 0}, ab[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (c < D) {
        for (int r = r0 + ry; r < r1; r += 8) {
            const long long o = static_cast<long long>(r) * D + c;
            const float mu = rms ? 0.f : mean[r];
            const float rs = rstd[r];
            float xv[8], gv[8];
            load8(x + o, xv);
            load8(dy + o, gv);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                aw[i] += gv[i] * (xv[i] - mu) * rs;
                ab[i] += gv[i];
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        red[0][ry][cx * 8 + i] = aw[i];
        red[1][ry][cx * 8 + i] = ab[i];
    }
    __syncthreads();
    // 256 threads: thread t reduces column t of the CTA's 256 columns
    const int col = blockIdx.x * 256 + threadIdx.x;
    if (col < D) {
        float sw = 0.f, sb = 0.f;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            sw += red[0][g][threadIdx.x];
            sb += red[1][g][threadIdx.x];
        }
        pw[static_cast<long long>(blockIdx.y) * D + col] = sw;
        if (pb) pb[static_cast<long long>(blockIdx.y) * D + col] = sb;
    }
}

// dst[c] += sum_g part[g, c]  (deterministic column reduction).  A CTA owns
// 32 columns; its 8 warps stride over g with coalesced 128-byte row reads,
// then combine in shared memory in a fixed order.
__global__ void __launch_bounds__(256) col_reduce_add(const float* part, int G, int D, float* dst) {
    pdl_wait();
    pdl_trigger();
    __shared__ float red[8][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int c = blockIdx.x * 32 + tx;
    float s = 0.f;
    if (c < D) {
#pragma unroll 4
        for (int g = ty; g < G; g += 8) s += part[static_cast<long long>(g) * D + c];
    }
    red[ty][tx] = s;
    __syncthreads();
    if (ty == 0 && c < D) {
        float t = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) t += red[i][tx];
        dst[c] += t;
    }
}

// ----------------------------------------------------------------- RoPE ---
// Rotate-half RoPE.  cos/sin come from a per-position table built in double
// precision (positions reach ~2e5, where float angle products lose accuracy).
struct RopeTable {
    float2* cs = nullptr;   // [max_pos, hd/2] (cos, sin)
    int max_pos = 0;
    int half = 0;
    float theta = 0.f;
};

__global__ void rope_table_k(float2* cs, int max_pos, int half, double theta) {
    pdl_wait();
    pdl_trigger();
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<long long>(max_pos) * half) return;
    const int pos = static_cast<int>(i / half), j = static_cast<int>(i % half);
    const double inv = pow(theta, -2.0 * j / (2.0 * half));
    double s, c;
    sincos(pos * inv, &s, &c);
    cs[i] = make_float2(static_cast<float>(c), static_cast<float>(s));
}

// One thread = 8 consecutive rotation pairs (j .. j+7) of one head slot of
// one token: two 16-byte loads (x1, x2 halves), 8 table entries, two
// 16-byte stores.  Requires hd % 16 == 0.
template <typename T>
__global__ void rope_scatter_k(const T* qkv, T* q_out, const AttnSeg* segs, const int* tok_seg,
                               const int* tok_pos, const float2* cs, int Tn, int H, int Hkv,
                               int hd, int layer) {
    pdl_wait();
    pdl_trigger();
    const int half = hd / 2;
    const int per_slot = half / 8;
    const int slots = H + 2 * Hkv;
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<long long>(Tn) * slots * per_slot) return;
    const int j = static_cast<int>(idx % per_slot) * 8;
    const int slot = static_cast<int>((idx / per_slot) % slots);
    const long long t = idx / (static_cast<long long>(per_slot) * slots);
    const T* src = qkv + t * slots * hd + static_cast<long long>(slot) * hd;
    const int pos = tok_pos[t];
    float x1[8], x2[8];
    load8(src + j, x1);
    load8(src + j + half, x2);
    if (slot < H + Hkv) {
        const float4* c4 = reinterpret_cast<const float4*>(cs + static_cast<long long>(pos) * half + j);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float4 cc = c4[k];     // (cos, sin) of pairs 2k, 2k+1
            const float a1 = x1[2 * k] * cc.x - x2[2 * k] * cc.y;
            const float a2 = x2[2 * k] * cc.x + x1[2 * k] * cc.y;
            const float b1 = x1[2 * k + 1] * cc.z - x2[2 * k + 1] * cc.w;
            const float b2 = x2[2 * k + 1] * cc.z + x1[2 * k + 1] * cc.w;
            x1[2 * k] = a1; x2[2 * k] = a2; x1[2 * k + 1] = b1; x2[2 * k + 1] = b2;
        }
    }
    T* dst;
    if (slot < H) {
        dst = q_out + (t * H + slot) * hd;
    } else {
        const AttnSeg& sg = segs[tok_seg[t]];
        const long long kvrow = static_cast<long long>(pos) * Hkv * hd;
        const bool is_k = slot < H + Hkv;
        const void* base = is_k ? sg.k : sg.v;
        dst = const_cast<T*>(static_cast<const T*>(base)) + layer * sg.kv_layer_stride + kvrow +
              static_cast<long long>(slot - H - (is_k ? 0 : Hkv)) * hd;
    }
    store8(dst + j, x1);
    store8(dst + j + half, x2);
}

template <typename T>
__global__ void rope_gather_grad_k(const float* dq, const AttnSeg* segs, const int* tok_seg,
                                   const int* tok_pos, const float2* cs, T* dqkv, int Tn, int H,
                                   int Hkv, int hd, int layer) {
    pdl_wait();
    pdl_trigger();
    const int half = hd / 2;
    const int per_slot = half / 8;
    const int slots = H + 2 * Hkv;
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<long long>(Tn) * slots * per_slot) return;
    const int j = static_cast<int>(idx % per_slot) * 8;
    const int slot = static_cast<int>((idx / per_slot) % slots);
    const long long t = idx / (static_cast<long long>(per_slot) * slots);
    const int pos = tok_pos[t];
    const float* src;
    if (slot < H) {
        src = dq + (t * H + slot) * hd;
    } else {
        const AttnSeg& sg = segs[tok_seg[t]];
        const long long kvrow = static_cast<long long>(pos) * Hkv * hd;
        src = (slot < H + Hkv ? sg.dk + static_cast<long long>(slot - H) * hd
                              : sg.dv + static_cast<long long>(slot - H - Hkv) * hd) +
              layer * sg.dkv_layer_stride + kvrow;
    }
    float g1[8], g2[8];
    load8(src + j, g1);
    load8(src + j + half, g2);
    if (slot < H + Hkv) {
        const float4* c4 = reinterpret_cast<const float4*>(cs + static_cast<long long>(pos) * half + j);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float4 cc = c4[k];
            const float a1 = g1[2 * k] * cc.x + g2[2 * k] * cc.y;
            const float a2 = g2[2 * k] * cc.x - g1[2 * k] * cc.y;
            const float b1 = g1[2 * k + 1] * cc.z + g2[2 * k + 1] * cc.w;
            const float b2 = g2[2 * k + 1] * cc.z - g1[2 * k + 1] * cc.w;
            g1[2 * k] = a1; g2[2 * k] = a2; g1[2 * k + 1] = b1; g2[2 * k + 1] = b2;
        }
    }
    T* dst = dqkv + t * slots * hd + static_cast<long long>(slot) * hd;
    store8(dst + j, g1);
    store8(dst + j + half, g2);
}

// ------------------------------------------------------------ activation ---
// fp32 (parity) path: exact tanhf / division; bf16 path: MUFU forms.
template <typename T>
__device__ __forceinline__ float gelu_tanh(float x) {
    if constexpr (std::is_same<T, float>::value) return gelu_tanh_f(x);
    else return gelu_tanh_fast_f(x);
}
template <typename T>
__device__ __forceinline__ float gelu_tanh_grad(float x) {
    if constexpr (std::is_same<T, float>::value) return gelu_tanh_grad_f(x);
    else return gelu_tanh_grad_fast_f(x);
}
template <typename T>
__device__ __forceinline__ float sigmoidf_(float x) {
    if constexpr (std::is_same<T, float>::value) return 1.f / (1.f + expf(-x));
    else return __fdividef(1.f, 1.f + __expf(-x));
}

template <typename T>
__global__ void act_fwd_k(int act, const T* h, T* out, long long Tn, int F) {
    pdl_wait();
    pdl_trigger();
    const long long n8 = Tn * F / 8;
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n8;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long e = i * 8;
        float v[8];
        if (act == 0) {
            load8(h + e, v);
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = gelu_tanh<T>(v[k]);
        } else {
            const long long t = e / F;
            const int c = static_cast<int>(e % F);
            float g[8], u[8];
            load8(h + t * 2 * F + c, g);
            load8(h + t * 2 * F + F + c, u);
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = g[k] * sigmoidf_<T>(g[k]) * u[k];
        }
        store8(out + e, v);
    }
}

template <typename T>
__global__ void act_bwd_k(int act, const T* h, const T* da, T* dh, long long Tn, int F) {
    pdl_wait();
    pdl_trigger();
    const long long n8 = Tn * F / 8;
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n8;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long e = i * 8;
        float d[8];
        load8(da + e, d);
        if (act == 0) {
            float x[8];
            load8(h + e, x);
#pragma unroll
            for (int k = 0; k < 8; ++k) d[k] *= gelu_tanh_grad<T>(x[k]);
            store8(dh + e, d);
        } else {
            const long long t = e / F;
            const int c = static_cast<int>(e % F);
            float g[8], u[8], dg[8], du[8];
            load8(h + t * 2 * F + c, g);
            load8(h + t * 2 * F + F + c, u);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const float sg = sigmoidf_<T>(g[k]);
                const float si = g[k] * sg;
                du[k] = d[k] * si;
                dg[k] = d[k] * u[k] * sg * (1.f + g[k] * (1.f - sg));
            }
            store8(dh + t * 2 * F + c, dg);
            store8(dh + t * 2 * F + F + c, du);
        }
    }
}

// -------------------------------------------------------- cross entropy ---
// One CTA per row; logits overwritten with grad_scale * (softmax - onehot);
// row_loss[row] = lse - logit[target] (0 for rows without a target).
template <typename T>
__global__ void ce_k(T* logits, const int32_t* targets, float* row_loss, int V, float gscale) {
    pdl_wait();
    pdl_trigger();
    __shared__ float scratch[32];
    __shared__ float red_m[32], red_s[32];
    const long long row = blockIdx.x;
    T* lr = logits + row * V;
    const int tgt = targets[row];
    float m = -INFINITY, s = 0.f;
    // online (max, sum) per 8-element vector: one rescale per vector instead
    // of per element (9 exponentials per 8 logits instead of 16; the MUFU
    // pipe and HBM otherwise co-limit this kernel)
    for (int c = threadIdx.x * 8; c < V; c += blockDim.x * 8) {
        float v[8];
        load8(lr + c, v);
        float mv = fmaxf(fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3])), fmaxf(fmaxf(v[4], v[5]), fmaxf(v[6], v[7])));
        const float mn = fmaxf(m, mv);
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) acc += __expf(v[i] - mn);
        s = (m == -INFINITY ? 0.f : s * __expf(m - mn)) + acc;
        m = mn;
    }
    // combine (m, s) across the block
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
        const float s2 = __shfl_xor_sync(0xffffffffu, s, o);
        const float mn = fmaxf(m, m2);
        s = (m == -INFINITY ? 0.f : s * __expf(m - mn)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mn));
        m = mn;
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        red_m[wid] = m;
        red_s[wid] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float M = -INFINITY, S = 0.f;
        for (int i = 0; i < (blockDim.x + 31) / 32; ++i) {
            const float mn = fmaxf(M, red_m[i]);
            S = (M == -INFINITY ? 0.f : S * __expf(M - mn)) +
                (red_m[i] == -INFINITY ? 0.f : red_s[i] * __expf(red_m[i] - mn));
            M = mn;
        }
        scratch[0] = M;
        scratch[1] = S;
    }
    __syncthreads();
    const float M = scratch[0];
    const float lse = M + logf(scratch[1]);
    const bool valid = tgt >= 0;
    if (threadIdx.x == 0) row_loss[row] = valid ? lse - to_f(lr[tgt]) : 0.f;
    __syncthreads();   // target logit read before overwrite
    for (int c = threadIdx.x * 8; c < V; c += blockDim.x * 8) {
        float v[8];
        load8(lr + c, v);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float p = valid ? __expf(v[i] - lse) : 0.f;
            if (valid && c + i == tgt) p -= 1.f;
            v[i] = p * gscale;
        }
        store8(lr + c, v);
    }
}

// Per-chunk loss: (sum of row losses, #rows with a target) in fp64, one CTA,
// fixed reduction order (deterministic); written to slot[0..1] and added to
// the stage accumulator acc[0..1] (stream-ordered, so no atomics).
__global__ void __launch_bounds__(1024) chunk_loss_k(const float* row_loss, const int32_t* targets, int Tn,
                                                     double* slot, double* acc) {
    pdl_wait();
    pdl_trigger();
    __shared__ double red_s[32], red_c[32];
    double s = 0.0, c = 0.0;
    for (int i = threadIdx.x; i < Tn; i += blockDim.x) {
        s += static_cast<double>(row_loss[i]);
        c += targets[i] >= 0 ? 1.0 : 0.0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        red_s[wid] = s;
        red_c[wid] = c;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double S = 0.0, C = 0.0;
        for (int i = 0; i < (blockDim.x + 31) / 32; ++i) {
            S += red_s[i];
            C += red_c[i];
        }
        slot[0] = S;
        slot[1] = C;
        acc[0] += S;
        acc[1] += C;
    }
}

// ---------------------------------------------------------------- misc ----
template <typename T>
__global__ void cast_k(const float* src, T* dst, long long n) {
    pdl_wait();
    pdl_trigger();
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        dst[i] = from_f<T>(src[i]);
}

template <typename T>
__global__ void add_k(T* y, const T* x, long long n) {
    pdl_wait();
    pdl_trigger();
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        y[i] = from_f<T>(to_f(y[i]) + to_f(x[i]));
}

// Multi-tensor AdamW: a block owns kAdamPer * blockDim consecutive float4
// groups of the concatenated segments; each thread finds its first group's
// segment by binary search over the start4 prefix (a few hundred entries,
// L1-resident) and then only walks forward, so the whole stage updates in one
// launch with independent, coalesced 16-byte accesses.
constexpr int kAdamPer = 4;
template <typename T>
__global__ void adamw_multi_k(const AdamSeg* __restrict__ segs, int nseg, long long total4,
                              float* __restrict__ master, T* __restrict__ work, float* __restrict__ grad,
                              float* __restrict__ m, float* __restrict__ v, float lr, float b1, float b2, float eps,
                              float wd, float bc1, float bc2) {
    pdl_wait();
    pdl_trigger();
    const float ib1 = 1.f / bc1, ib2 = 1.f / bc2;
    auto one = [&](float& p, float& mi, float& vi, float g, float w) {
        mi = b1 * mi + (1.f - b1) * g;
        vi = b2 * vi + (1.f - b2) * g * g;
        p -= lr * (w * p + (mi * ib1) / (sqrtf(vi * ib2) + eps));
    };
    const long long first = static_cast<long long>(blockIdx.x) * kAdamPer * blockDim.x + threadIdx.x;
    if (first >= total4) return;
    int lo = 0, hi = nseg - 1;     // last segment with start4 <= first
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(&segs[mid].start4) <= first) lo = mid;
        else hi = mid - 1;
    }
    int seg = lo;
#pragma unroll
    for (int u = 0; u < kAdamPer; ++u) {
        const long long i = first + static_cast<long long>(u) * blockDim.x;
        if (i >= total4) break;
        while (seg + 1 < nseg && __ldg(&segs[seg + 1].start4) <= i) ++seg;
        const long long local = i - __ldg(&segs[seg].start4);
        const long long e = __ldg(&segs[seg].off) / 4 + local;      // float4 index in the arenas
        const long long q = __ldg(&segs[seg].mv) / 4 + local;       // float4 index in the state
        const float w = __ldg(&segs[seg].decay) ? wd : 0.f;
        float4 g = reinterpret_cast<const float4*>(grad)[e];
        float4 mm = reinterpret_cast<const float4*>(m)[q];
        float4 vv = reinterpret_cast<const float4*>(v)[q];
        float4 p = reinterpret_cast<const float4*>(master)[e];
        one(p.x, mm.x, vv.x, g.x, w);
        one(p.y, mm.y, vv.y, g.y, w);
        one(p.z, mm.z, vv.z, g.z, w);
        one(p.w, mm.w, vv.w, g.w, w);
        reinterpret_cast<float4*>(m)[q] = mm;
        reinterpret_cast<float4*>(v)[q] = vv;
        reinterpret_cast<float4*>(master)[e] = p;
        reinterpret_cast<float4*>(grad)[e] = make_float4(0.f, 0.f, 0.f, 0.f);
        if constexpr (std::is_same<T, float>::value) {
            reinterpret_cast<float4*>(work)[e] = p;
        } else {
            __nv_bfloat162 lo2 = __floats2bfloat162_rn(p.x, p.y), hi2 = __floats2bfloat162_rn(p.z, p.w);
            uint2 raw;
            raw.x = *reinterpret_cast<uint32_t*>(&lo2);
            raw.y = *reinterpret_cast<uint32_t*>(&hi2);
            reinterpret_cast<uint2*>(work)[e] = raw;
        }
    }
}

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

__global__ void init_normal_k(float* dst, long long n, float std, unsigned long long seed) {
    pdl_wait();
    pdl_trigger();
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const unsigned long long r = mix64(seed ^ mix64(static_cast<unsigned long long>(i)));
        const float u1 = (static_cast<float>(r >> 40) + 0.5f) * (1.f / 16777216.f);
        const float u2 = (static_cast<float>((r >> 16) & 0xFFFFFF) + 0.5f) * (1.f / 16777216.f);
        dst[i] = std * sqrtf(-2.f * logf(u1)) * cospif(2.f * u2);
    }
}

__global__ void init_const_k(float* dst, long long n, float v) {
    pdl_wait();
    pdl_trigger();
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        dst[i] = v;
}

// Lazily grown RoPE table (one per process; positions only ever grow).
RopeTable g_rope;

const float2* rope_table(int max_pos, int hd, float theta, cudaStream_t s) {
    const int half = hd / 2;
    if (g_rope.cs && g_rope.max_pos >= max_pos && g_rope.half == half && g_rope.theta == theta)
        return g_rope.cs;
    if (max_pos <= 0) throw CudaError("rope table used before rope_reserve()");
    int want = 4096;
    while (want < max_pos) want *= 2;
    if (g_rope.cs) {
        EPP_CUDA(cudaStreamSynchronize(s));
        EPP_CUDA(cudaFree(g_rope.cs));
    }
    EPP_CUDA(cudaMalloc(&g_rope.cs, sizeof(float2) * want * half));
    const long long n = static_cast<long long>(want) * half;
    launch_k(rope_table_k, grid_for(n, 256), 256, 0, s, g_rope.cs, want, half, theta);
    EPP_CHECK_LAUNCH();
    g_rope.max_pos = want;
    g_rope.half = half;
    g_rope.theta = theta;
    return g_rope.cs;
}

int norm_threads(int D) {
    int t = D / 8;
    if (t > 128) t = 128;
    if (t < 32) t = 32;
    return t;
}

}  // namespace

// =========================================================================
void embed_fwd(DType t, const int32_t* ids, const void* table, void* out, int T, int D,
               cudaStream_t s) {
    ProfScope prof_(kProfEmbed, 0, s);
    if (T == 0) return;
    dispatch_t(t, [&](auto z) {
        using E = decltype(z);
        launch_k(embed_fwd_k<E>, T, norm_threads(D), 0, s, ids, static_cast<const E*>(table),
                                                     static_cast<E*>(out), T, D);
    });
    EPP_CHECK_LAUNCH();
}

void embed_bwd(DType t, const int32_t* ids, const void* dout, float* dtable, int T, int D,
               cudaStream_t s) {
    ProfScope prof_(kProfEmbed, 0, s);
    if (T == 0) return;
    dispatch_t(t, [&](auto z) {
        using E = decltype(z);
        launch_k(embed_bwd_k<E>, T, norm_threads(D), 0, s, ids, static_cast<const E*>(dout), dtable, T, D);
    });
    EPP_CHECK_LAUNCH();
}

void norm_fwd(DType t, bool rms, const void* x, const void* w, const void* b, void* y, float* mean,
              float* rstd, int T, int D, float eps, cudaStream_t s) {
    ProfScope prof_(kProfNormFwd, double(T) * D * 2 * dtype_size(t), s);
    EPP_REQUIRE(D % 8 == 0, "norm: D must be a multiple of 8");
    if (T == 0) return;
    dispatch_t(t, [&](auto z) {
        using E = decltype(z);
        const int blocks = ceil_div(static_cast<long long>(T) * 32, 256);
        auto warp_kernel = [&](auto nc) {
            constexpr int NC = decltype(nc)::value;
            launch_k(norm_fwd_warp_k<NC>, blocks, 256, 0, s, rms, static_cast<const bf16*>(x), static_cast<const bf16*>(w),
                                                       static_cast<const bf16*>(b), static_cast<bf16*>(y), mean, rstd,
                                                       T, eps);
        };
        if constexpr (std::is_same<E, bf16>::value) {
            auto row_kernel = [&](auto npt) {
                constexpr int NPT = decltype(npt)::value;
                launch_k(norm_fwd_row_k<NPT>, T, 128, 0, s, rms, static_cast<const bf16*>(x), static_cast<const bf16*>(w),
                                                      static_cast<const bf16*>(b), static_cast<bf16*>(y), mean, rstd,
                                                      eps);
            };
            if (D == 256) return warp_kernel(std::integral_constant<int, 1>{});
            if (D == 512) return warp_kernel(std::integral_constant<int, 2>{});
            if (D == 1024) return row_kernel(std::integral_constant<int, 1>{});
            if (D == 2048) return row_kernel(std::integral_constant<int, 2>{});
            if (D == 4096) return row_kernel(std::integral_constant<int, 4>{});
            if (D == 8192) return row_kernel(std::integral_constant<int, 8>{});
        }
        launch_k(norm_fwd_k<E>, T, norm_threads(D), 0, s, rms, static_cast<const E*>(x),
                                                    static_cast<const E*>(w),
                                                    static_cast<const E*>(b), static_cast<E*>(y),
                                                    mean, rstd, D, eps);
    });
    EPP_CHECK_LAUNCH();
}

void norm_apply(DType t, bool rms, const void* x, const void* w, const void* b, const float* mean,
                const float* rstd, void* y, int T, int D, cudaStream_t s) {
    ProfScope prof_(kProfNormFwd, double(T) * D * 2 * dtype_size(t), s);
    if (T == 0) return;
    dispatch_t(t, [&](auto z) {
        using E = decltype(z);
        launch_k(norm_apply_k<E>, T, norm_threads(D), 0, s, rms, static_cast<const E*>(x),
                                                      static_cast<const E*>(w),
                                                      static_cast<const E*>(b), mean, rstd,
                                                      static_cast<E*>(y), D);
    });
    EPP_CHECK_LAUNCH();
}

void norm_bwd(DType t, bool rms, const void* x, const void* w, const void* dy, const float* mean,
              const float* rstd, const void* dres, void* dx, float* dw, float* db, int T, int D,
              cudaStream_t s, const void* bias, void* xn_out) {
    ProfScope prof_(kProfNormBwd, double(T) * D * (xn_out ? 7 : 6) * dtype_size(t), s);
    EPP_REQUIRE(D % 8 == 0 && D <= 8 * 256 * kNormMaxG, "norm_bwd: unsupported D");
    if (T == 0) return;
    // ~4 waves of 148 SMs for the partial-sum kernel (256 columns per CTA)
    const int col_blocks = ceil_div(D, 256);
    const int G = std::max(1, std::min(ceil_div(T, 8), 592 / col_blocks));
    const int rows_per = ceil_div(T, G);
    float* part = nullptr;
    EPP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&part), sizeof(float) * 2 * G * D, s));
    float* pw = part;
    float* pb = db ? part + static_cast<long long>(G) * D : nullptr;
    dispatch_t(t, [&](auto z) {
        using E = decltype(z);
        bool done = false;
        if constexpr (std::is_same<E, bf16>::value) {
            auto row_kernel = [&](auto npt) {
                constexpr int NPT = decltype(npt)::value;
                launch_k(norm_bwd_dx_row_k<NPT>, T, 128, 0, s, rms, static_cast<const bf16*>(x), static_cast<const bf16*>(w),
                                                         static_cast<const bf16*>(dy), mean, rstd,
                                                         static_cast<const bf16*>(dres), static_cast<bf16*>(dx),
                                                         static_cast<const bf16*>(bias), static_cast<bf16*>(xn_out));
                done = true;
            };
            if (D == 1024) row_kernel(std::integral_constant<int, 1>{});
            else if (D == 2048) row_kernel(std::integral_constant<int, 2>{});
            else if (D == 4096) row_kernel(std::integral_constant<int, 4>{});
            else if (D == 8192) row_kernel(std::integral_constant<int, 8>{});
        }
        if (!done && xn_out) norm_apply(t, rms, x, w, bias, mean, rstd, xn_out, T, D, s);
        if (!done)
            launch_k(norm_bwd_dx_k<E>, ceil_div(static_cast<long long>(T) * 32, 256), 256, 0, s, 
                rms, static_cast<const E*>(x), static_cast<const E*>(w), static_cast<const E*>(dy), mean,
                rstd, static_cast<const E*>(dres), static_cast<E*>(dx), T, D);
        EPP_CHECK_LAUNCH();
        launch_k(norm_bwd_dw2_k<E>, dim3(col_blocks, G), 256, 0, s, 
            rms, static_cast<const E*>(x), static_cast<const E*>(dy), mean, rstd, pw, pb, T, D, rows_per);
        EPP_CHECK_LAUNCH();
    });
    launch_k(col_reduce_add, ceil_div(D, 32), 256, 0, s, pw, G, D, dw);
    if (db) launch_k(col_reduce_add, ceil_div(D, 32), 256, 0, s, pb, G, D, db);
    EPP_CHECK_LAUNCH();
    EPP_CUDA(cudaFreeAsync(part, s));
}

void rope_qkv_scatter(DType t, const void* qkv, void* q_out, const AttnSeg* segs_dev, int nseg,
                      const int* tok_seg, const int* tok_pos, int T, int H, int Hkv, int hd,
                      int layer, float theta, cudaStream_t s) {
    ProfScope prof_(kProfRope, double(T) * (H + 2 * Hkv) * hd * 2 * dtype_size(t), s);
    (void)nseg;
    if (T == 0) return;
    EPP_REQUIRE(hd % 16 == 0, "rope: head_dim must be a multiple of 16");
    const float2* cs = rope_table(0, hd, theta, s);
    const long long n = static_cast<long long>(T) * (H + 2 * Hkv) * (hd / 16);
    dispatch_t(t, [&](auto z) {
        using E = decltype(z);
        launch_k(rope_scatter_k<E>, grid_for(n, 256), 256, 0, s, static_cast<const E*>(qkv),
                                                           static_cast<E*>(q_out), segs_dev,
                                                           tok_seg, tok_pos, cs, T, H, Hkv, hd,
                                                           layer);
    });
    EPP_CHECK_LAUNCH();
}

void rope_qkv_gather_grad(DType t, const float* dq, const AttnSeg* segs_dev, const int* tok_seg,
                          const int* tok_pos, void* dqkv, int T, int H, int Hkv, int hd, int layer,
                          float theta, cudaStream_t s) {
    ProfScope prof_(kProfRope, double(T) * (H + 2 * Hkv) * hd * (4 + dtype_size(t)), s);
    if (T == 0) return;
    const float2* cs = rope_table(0, hd, theta, s);
    const long long n = static_cast<long long>(T) * (H + 2 * Hkv) * (hd / 16);
    dispatch_t(t, [&](auto z) {
        using E = decltype(z);
        launch_k(rope_gather_grad_k<E>, grid_for(n, 256), 256, 0, s, dq, segs_dev, tok_seg, tok_pos, cs,
                                                               static_cast<E*>(dqkv), T, H, Hkv,
                                                               hd, layer);
    });
    EPP_CHECK_LAUNCH();
}

void act_fwd(DType t, int act, const void* h, void* a, int T, int F, cudaStream_t s) {
    ProfScope prof_(kProfAct, double(T) * F * (act ? 3 : 2) * dtype_size(t), s);
    EPP_REQUIRE(F % 8 == 0, "act: F must be a multiple of 8");
    if (T == 0) return;
    const long long n8 = static_cast<long long>(T) * F / 8;
    dispatch_t(t, [&](auto z) {
        using E = decltype(z);
        launch_k(act_fwd_k<E>, grid_for(n8, 256), 256, 0, s, act, static_cast<const E*>(h),
                                                       static_cast<E*>(a), T, F);
    });
    EPP_CHECK_LAUNCH();
}

void act_bwd(DType t, int act, const void* h, const void* da, void* dh, int T, int F,
             cudaStream_t s) {
    ProfScope prof_(kProfAct, double(T) * F * (act ? 5 : 3) * dtype_size(t), s);
    if (T == 0) return;
    const long long n8 = static_cast<long long>(T) * F / 8;
    dispatch_t(t, [&](auto z) {
        using E = decltype(z);
        launch_k(act_bwd_k<E>, grid_for(n8, 256), 256, 0, s, act, static_cast<const E*>(h),
                                                       static_cast<const E*>(da),
                                                       static_cast<E*>(dh), T, F);
    });
    EPP_CHECK_LAUNCH();
}

void cross_entropy(DType t, void* logits, const int32_t* targets, float* row_loss, int T, int V,
                   float grad_scale, cudaStream_t s) {
    ProfScope prof_(kProfCe, double(T) * V * 2 * dtype_size(t), s);
    EPP_REQUIRE(V % 8 == 0, "ce: V must be a multiple of 8");
    if (T == 0) return;
    dispatch_t(t, [&](auto z) {
        using E = decltype(z);
        launch_k(ce_k<E>, T, 256, 0, s, static_cast<E*>(logits), targets, row_loss, V, grad_scale);
    });
    EPP_CHECK_LAUNCH();
}

void chunk_loss(const float* row_loss, const int32_t* targets, int T, double* slot, double* acc, cudaStream_t s) {
    ProfScope prof_(kProfCe, double(T) * 8, s);
    launch_k(chunk_loss_k, 1, 1024, 0, s, row_loss, targets, T, slot, acc);
    EPP_CHECK_LAUNCH();
}

void fill_zero(void* p, size_t bytes, cudaStream_t s) {
    ProfScope prof_(kProfCopy, double(bytes), s);
    if (bytes) EPP_CUDA(cudaMemsetAsync(p, 0, bytes, s));
}

void cast_f32_to(DType t, const float* src, void* dst, long long n, cudaStream_t s) {
    ProfScope prof_(kProfCopy, 0, s);
    if (n == 0) return;
    dispatch_t(t, [&](auto z) {
        using E = decltype(z);
        launch_k(cast_k<E>, grid_for(n, 256), 256, 0, s, src, static_cast<E*>(dst), n);
    });
    EPP_CHECK_LAUNCH();
}

void add_inplace(DType t, void* y, const void* x, long long n, cudaStream_t s) {
    ProfScope prof_(kProfCopy, 0, s);
    if (n == 0) return;
    dispatch_t(t, [&](auto z) {
        using E = decltype(z);
        launch_k(add_k<E>, grid_for(n, 256), 256, 0, s, static_cast<E*>(y), static_cast<const E*>(x), n);
    });
    EPP_CHECK_LAUNCH();
}

void adamw_multi(const AdamSeg* segs, int nseg, long long total4, float* master, void* work, DType t, float* grad,
                 float* m, float* v, float lr, float b1, float b2, float eps, float wd, float bc1, float bc2,
                 cudaStream_t s) {
    ProfScope prof_(kProfAdam, double(total4) * 4 * (26 + dtype_size(t)), s);
    if (total4 == 0 || nseg == 0) return;
    dispatch_t(t, [&](auto z) {
        using E = decltype(z);
        const long long blocks = (total4 + kAdamPer * 256 - 1) / (kAdamPer * 256);
        launch_k(adamw_multi_k<E>, dim3(static_cast<unsigned>(blocks)), 256, 0, s, segs, nseg, total4, master,
                 static_cast<E*>(work), grad, m, v, lr, b1, b2, eps, wd, bc1, bc2);
    });
    EPP_CHECK_LAUNCH();
}

void init_normal(float* dst, long long n, float std, unsigned long long seed, cudaStream_t s) {
    if (n == 0) return;
    launch_k(init_normal_k, grid_for(n, 256), 256, 0, s, dst, n, std, seed);
    EPP_CHECK_LAUNCH();
}

void init_const(float* dst, long long n, float v, cudaStream_t s) {
    if (n == 0) return;
    launch_k(init_const_k, grid_for(n, 256), 256, 0, s, dst, n, v);
    EPP_CHECK_LAUNCH();
}

const float2* rope_table_ptr(int hd, float theta, cudaStream_t s) { return rope_table(0, hd, theta, s); }

void rope_reserve(int max_pos, int hd, float theta, cudaStream_t s) {
    rope_table(max_pos, hd, theta, s);
}

}  // namespace eppk
