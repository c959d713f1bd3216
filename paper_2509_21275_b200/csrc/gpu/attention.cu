// epp-b200: slice-causal flash attention for heterogeneous EPP chunks.
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
// BF16 kernels: FA2-style mma.sync.m16n8k16 (fp32 accumulate), 64-row query
// and key blocks, cp.async double-buffered K/V tiles in XOR-swizzled smem.
//   fwd : grid (query blocks, H)           -> O, LSE (log2 domain)
//   dq  : grid (query blocks, H)           -> dQ (fp32), no atomics
//   dkv : grid (key blocks, Hkv)           -> dK/dV += (fp32 RMW into the
//         segment's accumulator; each key block is owned by one CTA, GQA
//         heads are looped inside the CTA, so no atomics and deterministic)
// The dK/dV accumulators of a split sequence persist across its chunks:
// later slices' backwards (which run first) add into earlier slices' keys.
// F32 kernels (parity mode): warp-per-row SIMT versions of the same math.
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "kernels.h"
#include "profile.h"

namespace eppk {

namespace {

constexpr int BM = kAttnBlock;    // query rows per CTA
constexpr int BN = kAttnBlock;    // keys per tile
constexpr float kLog2e = 1.4426950408889634f;

// ------------------------------------------------------------ primitives --
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int HD>
__device__ __forceinline__ int swz(int row, int chunk) {   // element offset
    return row * HD + ((chunk ^ (row & 7)) << 3);
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
    const int n = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)),
                 "l"(valid ? src : nullptr), "r"(n)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_addr(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_addr(p)));
}

__device__ __forceinline__ void mma(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                    uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}

// A fragment (16x16) of a row-major swizzled tile at (row0, col0).
template <int HD>
__device__ __forceinline__ void lda_frag(uint32_t (&r)[4], const bf16* tile, int row0, int col0,
                                         int lane) {
    const int row = row0 + (lane & 15);
    const int chunk = (col0 >> 3) + (lane >> 4);
    ldsm_x4(r, tile + swz<HD>(row, chunk));
}
// Two B fragments (n-blocks n0, n0+8; k16 at k0) from a tile stored n-major
// (rows = n, cols = k): r0,r1 -> n-block n0, r2,r3 -> n-block n0+8.
template <int HD>
__device__ __forceinline__ void ldb_nmajor(uint32_t (&r)[4], const bf16* tile, int n0, int k0,
                                           int lane) {
    const int row = n0 + (lane & 7) + ((lane >> 4) << 3);
    const int chunk = (k0 >> 3) + ((lane >> 3) & 1);
    ldsm_x4(r, tile + swz<HD>(row, chunk));
}
// Two B fragments from a tile stored k-major (rows = k, cols = n).
template <int HD>
__device__ __forceinline__ void ldb_kmajor(uint32_t (&r)[4], const bf16* tile, int k0, int n0,
                                           int lane) {
    const int row = k0 + (lane & 7) + (((lane >> 3) & 1) << 3);
    const int chunk = (n0 >> 3) + (lane >> 4);
    ldsm_x4_t(r, tile + swz<HD>(row, chunk));
}

// Async copy of `nrows` valid rows (rest zero) of a [64, HD] tile.
template <int HD>
__device__ __forceinline__ void load_tile(bf16* tile, const bf16* base, long long row_stride,
                                          int nrows) {
    constexpr int kChunks = HD / 8;
    for (int i = threadIdx.x; i < BM * kChunks; i += blockDim.x) {
        const int r = i / kChunks, c = i % kChunks;
        const bool ok = r < nrows;
        cp_async16(tile + swz<HD>(r, c), ok ? base + r * row_stride + c * 8 : base, ok);
    }
}

// ------------------------------------------------------------ forward ----
template <int HD>
__global__ void __launch_bounds__(128) attn_fwd_bf16(const AttnArgs a) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(128) uint8_t smem_raw[];
    bf16* sQ = reinterpret_cast<bf16*>(smem_raw);
    bf16* sK = sQ + BM * HD;          // 2 buffers
    bf16* sV = sK + 2 * BN * HD;      // 2 buffers
    const AttnWork w = a.qwork[blockIdx.x];
    const AttnSeg sg = a.segs[w.seg];
    const int h = blockIdx.y;
    const int kvh = h / (a.H / a.Hkv);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q0 = w.block * BM;
    const int rows = min(BM, sg.q_len - q0);
    const int kv_end = sg.kv_ctx + q0 + rows;
    const int nkb = (kv_end + BN - 1) / BN;
    const long long kvs = static_cast<long long>(a.Hkv) * HD;
    const bf16* kbase = static_cast<const bf16*>(sg.k) + a.layer * sg.kv_layer_stride + kvh * HD;
    const bf16* vbase = static_cast<const bf16*>(sg.v) + a.layer * sg.kv_layer_stride + kvh * HD;
    const bf16* qbase = static_cast<const bf16*>(a.q) +
                        (static_cast<long long>(sg.q_start + q0) * a.H + h) * HD;

    load_tile<HD>(sQ, qbase, static_cast<long long>(a.H) * HD, rows);
    load_tile<HD>(sK, kbase, kvs, min(BN, kv_end));
    load_tile<HD>(sV, vbase, kvs, min(BN, kv_end));
    cp_commit();

    const int r_lo = warp * 16 + (lane >> 2);     // tile row of c[0..1]; +8 for c[2..3]
    const int qpos_lo = (r_lo < rows) ? sg.kv_ctx + q0 + r_lo : -1;
    const int qpos_hi = (r_lo + 8 < rows) ? sg.kv_ctx + q0 + r_lo + 8 : -1;
    const float c2 = a.scale * kLog2e;

    uint32_t qf[HD / 16][4];
    float o[HD / 8][4];
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};

    for (int kb = 0; kb < nkb; ++kb) {
        const int buf = kb & 1;
        if (kb + 1 < nkb) {
            const int k1 = (kb + 1) * BN;
            load_tile<HD>(sK + (buf ^ 1) * BN * HD, kbase + k1 * kvs, kvs, min(BN, kv_end - k1));
            load_tile<HD>(sV + (buf ^ 1) * BN * HD, vbase + k1 * kvs, kvs, min(BN, kv_end - k1));
            cp_commit();
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        if (kb == 0) {
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk) lda_frag<HD>(qf[kk], sQ, warp * 16, kk * 16, lane);
        }
        const bf16* tK = sK + buf * BN * HD;
        const bf16* tV = sV + buf * BN * HD;

        float s[BN / 8][4];
#pragma unroll
        for (int i = 0; i < BN / 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
#pragma unroll
            for (int nb = 0; nb < BN / 16; ++nb) {
                uint32_t b[4];
                ldb_nmajor<HD>(b, tK, nb * 16, kk * 16, lane);
                mma(s[2 * nb], qf[kk], b[0], b[1]);
                mma(s[2 * nb + 1], qf[kk], b[2], b[3]);
            }

        const int kfirst = kb * BN;
        const bool need_mask = (kfirst + BN - 1 > sg.kv_ctx + q0) || rows < BM;
        float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int nb = 0; nb < BN / 8; ++nb)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int key = kfirst + nb * 8 + 2 * (lane & 3) + (j & 1);
                const int qp = (j < 2) ? qpos_lo : qpos_hi;
                float v = s[nb][j] * c2;
                if (need_mask && key > qp) v = -INFINITY;
                s[nb][j] = v;
                mx[j >> 1] = fmaxf(mx[j >> 1], v);
            }
        float alpha[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
            mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
            const float mnew = fmaxf(m[r], mx[r]);
            const float muse = (mnew == -INFINITY) ? 0.f : mnew;
            alpha[r] = exp2f(m[r] - muse);
            m[r] = mnew;
            mx[r] = muse;
        }
        float rs[2] = {0.f, 0.f};
#pragma unroll
        for (int nb = 0; nb < BN / 8; ++nb)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float p = exp2f(s[nb][j] - mx[j >> 1]);
                s[nb][j] = p;
                rs[j >> 1] += p;
            }
#pragma unroll
        for (int r = 0; r < 2; ++r) l[r] = l[r] * alpha[r] + rs[r];
#pragma unroll
        for (int i = 0; i < HD / 8; ++i) {
            o[i][0] *= alpha[0]; o[i][1] *= alpha[0];
            o[i][2] *= alpha[1]; o[i][3] *= alpha[1];
        }
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk) {
            uint32_t pa[4];
            pa[0] = pack_bf16(s[2 * kk][0], s[2 * kk][1]);
            pa[1] = pack_bf16(s[2 * kk][2], s[2 * kk][3]);
            pa[2] = pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]);
            pa[3] = pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
            for (int nd = 0; nd < HD / 16; ++nd) {
                uint32_t b[4];
                ldb_kmajor<HD>(b, tV, kk * 16, nd * 16, lane);
                mma(o[2 * nd], pa, b[0], b[1]);
                mma(o[2 * nd + 1], pa, b[2], b[3]);
            }
        }
        __syncthreads();
    }

#pragma unroll
    for (int r = 0; r < 2; ++r) {
        l[r] += __shfl_xor_sync(0xffffffffu, l[r], 1);
        l[r] += __shfl_xor_sync(0xffffffffu, l[r], 2);
    }
    const float inv[2] = {l[0] > 0.f ? 1.f / l[0] : 0.f, l[1] > 0.f ? 1.f / l[1] : 0.f};
    bf16* obase = static_cast<bf16*>(a.o);
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int tr = r_lo + 8 * r;
        if (tr >= rows) continue;
        const long long t = sg.q_start + q0 + tr;
        bf16* orow = obase + (t * a.H + h) * HD;
#pragma unroll
        for (int nd = 0; nd < HD / 8; ++nd) {
            const int col = nd * 8 + 2 * (lane & 3);
            *reinterpret_cast<__nv_bfloat162*>(orow + col) =
                __floats2bfloat162_rn(o[nd][2 * r] * inv[r], o[nd][2 * r + 1] * inv[r]);
        }
        if ((lane & 3) == 0)
            a.lse[static_cast<long long>(h) * a.T + t] =
                l[r] > 0.f ? m[r] + log2f(l[r]) : INFINITY;
    }
}

// ------------------------------------------------------- backward: dQ ----
template <int HD>
__global__ void __launch_bounds__(128) attn_bwd_dq_bf16(const AttnArgs a) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(128) uint8_t smem_raw[];
    bf16* sQ = reinterpret_cast<bf16*>(smem_raw);
    bf16* sO = sQ + BM * HD;           // dO
    bf16* sK = sO + BM * HD;           // 2 buffers
    bf16* sV = sK + 2 * BN * HD;       // 2 buffers
    const AttnWork w = a.qwork[blockIdx.x];
    const AttnSeg sg = a.segs[w.seg];
    const int h = blockIdx.y;
    const int kvh = h / (a.H / a.Hkv);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q0 = w.block * BM;
    const int rows = min(BM, sg.q_len - q0);
    const int kv_end = sg.kv_ctx + q0 + rows;
    const int nkb = (kv_end + BN - 1) / BN;
    const long long kvs = static_cast<long long>(a.Hkv) * HD;
    const long long qs = static_cast<long long>(a.H) * HD;
    const bf16* kbase = static_cast<const bf16*>(sg.k) + a.layer * sg.kv_layer_stride + kvh * HD;
    const bf16* vbase = static_cast<const bf16*>(sg.v) + a.layer * sg.kv_layer_stride + kvh * HD;
    const long long row0 = static_cast<long long>(sg.q_start + q0);

    load_tile<HD>(sQ, static_cast<const bf16*>(a.q) + (row0 * a.H + h) * HD, qs, rows);
    load_tile<HD>(sO, static_cast<const bf16*>(a.dout) + (row0 * a.H + h) * HD, qs, rows);
    load_tile<HD>(sK, kbase, kvs, min(BN, kv_end));
    load_tile<HD>(sV, vbase, kvs, min(BN, kv_end));
    cp_commit();

    const int r_lo = warp * 16 + (lane >> 2);
    const int qpos[2] = {(r_lo < rows) ? sg.kv_ctx + q0 + r_lo : -1,
                         (r_lo + 8 < rows) ? sg.kv_ctx + q0 + r_lo + 8 : -1};
    float lse[2], dlt[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int tr = min(r_lo + 8 * r, rows - 1);
        const long long t = row0 + tr;
        lse[r] = a.lse[static_cast<long long>(h) * a.T + t];
        dlt[r] = a.delta[static_cast<long long>(h) * a.T + t];
    }
    const float c2 = a.scale * kLog2e;

    uint32_t qf[HD / 16][4], of[HD / 16][4];
    float dq[HD / 8][4];
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;

    for (int kb = 0; kb < nkb; ++kb) {
        const int buf = kb & 1;
        if (kb + 1 < nkb) {
            const int k1 = (kb + 1) * BN;
            load_tile<HD>(sK + (buf ^ 1) * BN * HD, kbase + k1 * kvs, kvs, min(BN, kv_end - k1));
            load_tile<HD>(sV + (buf ^ 1) * BN * HD, vbase + k1 * kvs, kvs, min(BN, kv_end - k1));
            cp_commit();
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        if (kb == 0) {
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk) {
                lda_frag<HD>(qf[kk], sQ, warp * 16, kk * 16, lane);
                lda_frag<HD>(of[kk], sO, warp * 16, kk * 16, lane);
            }
        }
        const bf16* tK = sK + buf * BN * HD;
        const bf16* tV = sV + buf * BN * HD;
        float s[BN / 8][4], dp[BN / 8][4];
#pragma unroll
        for (int i = 0; i < BN / 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) s[i][j] = dp[i][j] = 0.f;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
#pragma unroll
            for (int nb = 0; nb < BN / 16; ++nb) {
                uint32_t b[4];
                ldb_nmajor<HD>(b, tK, nb * 16, kk * 16, lane);
                mma(s[2 * nb], qf[kk], b[0], b[1]);
                mma(s[2 * nb + 1], qf[kk], b[2], b[3]);
                ldb_nmajor<HD>(b, tV, nb * 16, kk * 16, lane);
                mma(dp[2 * nb], of[kk], b[0], b[1]);
                mma(dp[2 * nb + 1], of[kk], b[2], b[3]);
            }
        const int kfirst = kb * BN;
#pragma unroll
        for (int nb = 0; nb < BN / 8; ++nb)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int key = kfirst + nb * 8 + 2 * (lane & 3) + (j & 1);
                const int r = j >> 1;
                const float p = (key > qpos[r]) ? 0.f : exp2f(s[nb][j] * c2 - lse[r]);
                s[nb][j] = p * (dp[nb][j] - dlt[r]);     // dS
            }
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk) {
            uint32_t pa[4];
            pa[0] = pack_bf16(s[2 * kk][0], s[2 * kk][1]);
            pa[1] = pack_bf16(s[2 * kk][2], s[2 * kk][3]);
            pa[2] = pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]);
            pa[3] = pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
            for (int nd = 0; nd < HD / 16; ++nd) {
                uint32_t b[4];
                ldb_kmajor<HD>(b, tK, kk * 16, nd * 16, lane);
                mma(dq[2 * nd], pa, b[0], b[1]);
                mma(dq[2 * nd + 1], pa, b[2], b[3]);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int tr = r_lo + 8 * r;
        if (tr >= rows) continue;
        float* drow = a.dq + ((row0 + tr) * a.H + h) * HD;
#pragma unroll
        for (int nd = 0; nd < HD / 8; ++nd) {
            const int col = nd * 8 + 2 * (lane & 3);
            *reinterpret_cast<float2*>(drow + col) =
                make_float2(dq[nd][2 * r] * a.scale, dq[nd][2 * r + 1] * a.scale);
        }
    }
}

// --------------------------------------------------- backward: dK, dV ----
template <int HD>
__global__ void __launch_bounds__(128) attn_bwd_dkv_bf16(const AttnArgs a) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(128) uint8_t smem_raw[];
    bf16* sK = reinterpret_cast<bf16*>(smem_raw);
    bf16* sV = sK + BN * HD;
    bf16* sQ = sV + BN * HD;           // 2 buffers
    bf16* sO = sQ + 2 * BM * HD;       // 2 buffers (dO)
    float* sL = reinterpret_cast<float*>(sO + 2 * BM * HD);   // [2][BM] lse
    float* sD = sL + 2 * BM;                                  // [2][BM] delta
    const AttnWork w = a.kwork[blockIdx.x];
    const AttnSeg sg = a.segs[w.seg];
    const int kvh = blockIdx.y;
    const int group = a.H / a.Hkv;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int k0 = w.block * BN;
    const int kv_len = sg.kv_ctx + sg.q_len;
    const int nkeys = min(BN, kv_len - k0);
    const long long kvs = static_cast<long long>(a.Hkv) * HD;
    const long long qs = static_cast<long long>(a.H) * HD;
    const bf16* kbase = static_cast<const bf16*>(sg.k) + a.layer * sg.kv_layer_stride + kvh * HD;
    const bf16* vbase = static_cast<const bf16*>(sg.v) + a.layer * sg.kv_layer_stride + kvh * HD;

    // Query blocks whose rows can see a key of this block.
    const int qb_first = max(0, k0 - sg.kv_ctx) / BM;
    const int nqb = (sg.q_len + BM - 1) / BM;
    const int per_head = nqb - qb_first;
    const int iters = per_head * group;

    auto issue = [&](int it, int buf) {
        const int hq = kvh * group + it / per_head;
        const int qb = qb_first + it % per_head;
        const int q0 = qb * BM;
        const int rows = min(BM, sg.q_len - q0);
        const long long row0 = sg.q_start + q0;
        load_tile<HD>(sQ + buf * BM * HD, static_cast<const bf16*>(a.q) + (row0 * a.H + hq) * HD,
                      qs, rows);
        load_tile<HD>(sO + buf * BM * HD,
                      static_cast<const bf16*>(a.dout) + (row0 * a.H + hq) * HD, qs, rows);
        for (int i = threadIdx.x; i < BM; i += blockDim.x) {
            const bool ok = i < rows;
            sL[buf * BM + i] = ok ? a.lse[static_cast<long long>(hq) * a.T + row0 + i] : INFINITY;
            sD[buf * BM + i] = ok ? a.delta[static_cast<long long>(hq) * a.T + row0 + i] : 0.f;
        }
    };

    load_tile<HD>(sK, kbase + k0 * kvs, kvs, nkeys);
    load_tile<HD>(sV, vbase + k0 * kvs, kvs, nkeys);
    if (iters > 0) issue(0, 0);
    cp_commit();

    const int kr_lo = warp * 16 + (lane >> 2);
    const int kpos[2] = {k0 + kr_lo, k0 + kr_lo + 8};
    const float c2 = a.scale * kLog2e;
    float dk[HD / 8][4], dv[HD / 8][4];
#pragma unroll
    for (int i = 0; i < HD / 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dk[i][j] = dv[i][j] = 0.f;

    for (int it = 0; it < iters; ++it) {
        const int buf = it & 1;
        if (it + 1 < iters) {
            issue(it + 1, buf ^ 1);
            cp_commit();
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        const int qb = qb_first + it % per_head;
        const int q0 = qb * BM;
        const int rows = min(BM, sg.q_len - q0);
        const bf16* tQ = sQ + buf * BM * HD;
        const bf16* tO = sO + buf * BM * HD;
        const float* tL = sL + buf * BM;
        const float* tD = sD + buf * BM;

        float st[BM / 8][4], dpt[BM / 8][4];
#pragma unroll
        for (int i = 0; i < BM / 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) st[i][j] = dpt[i][j] = 0.f;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
            uint32_t ka[4], va[4];
            lda_frag<HD>(ka, sK, warp * 16, kk * 16, lane);
            lda_frag<HD>(va, sV, warp * 16, kk * 16, lane);
#pragma unroll
            for (int nb = 0; nb < BM / 16; ++nb) {
                uint32_t b[4];
                ldb_nmajor<HD>(b, tQ, nb * 16, kk * 16, lane);
                mma(st[2 * nb], ka, b[0], b[1]);
                mma(st[2 * nb + 1], ka, b[2], b[3]);
                ldb_nmajor<HD>(b, tO, nb * 16, kk * 16, lane);
                mma(dpt[2 * nb], va, b[0], b[1]);
                mma(dpt[2 * nb + 1], va, b[2], b[3]);
            }
        }
        // P^T and dS^T (rows = keys, cols = queries)
#pragma unroll
        for (int nb = 0; nb < BM / 8; ++nb)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int qi = nb * 8 + 2 * (lane & 3) + (j & 1);
                const int qp = (qi < rows) ? sg.kv_ctx + q0 + qi : -1;
                const float p = (kpos[j >> 1] > qp) ? 0.f : exp2f(st[nb][j] * c2 - tL[qi]);
                st[nb][j] = p;
                dpt[nb][j] = p * (dpt[nb][j] - tD[qi]);
            }
#pragma unroll
        for (int kk = 0; kk < BM / 16; ++kk) {
            uint32_t pa[4], sa[4];
            pa[0] = pack_bf16(st[2 * kk][0], st[2 * kk][1]);
            pa[1] = pack_bf16(st[2 * kk][2], st[2 * kk][3]);
            pa[2] = pack_bf16(st[2 * kk + 1][0], st[2 * kk + 1][1]);
            pa[3] = pack_bf16(st[2 * kk + 1][2], st[2 * kk + 1][3]);
            sa[0] = pack_bf16(dpt[2 * kk][0], dpt[2 * kk][1]);
            sa[1] = pack_bf16(dpt[2 * kk][2], dpt[2 * kk][3]);
            sa[2] = pack_bf16(dpt[2 * kk + 1][0], dpt[2 * kk + 1][1]);
            sa[3] = pack_bf16(dpt[2 * kk + 1][2], dpt[2 * kk + 1][3]);
#pragma unroll
            for (int nd = 0; nd < HD / 16; ++nd) {
                uint32_t b[4];
                ldb_kmajor<HD>(b, tO, kk * 16, nd * 16, lane);
                mma(dv[2 * nd], pa, b[0], b[1]);
                mma(dv[2 * nd + 1], pa, b[2], b[3]);
                ldb_kmajor<HD>(b, tQ, kk * 16, nd * 16, lane);
                mma(dk[2 * nd], sa, b[0], b[1]);
                mma(dk[2 * nd + 1], sa, b[2], b[3]);
            }
        }
        __syncthreads();
    }

    float* dkb = sg.dk + a.layer * sg.dkv_layer_stride + kvh * HD;
    float* dvb = sg.dv + a.layer * sg.dkv_layer_stride + kvh * HD;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int kr = kr_lo + 8 * r;
        if (kr >= nkeys) continue;
        float* dkr = dkb + (k0 + kr) * kvs;
        float* dvr = dvb + (k0 + kr) * kvs;
#pragma unroll
        for (int nd = 0; nd < HD / 8; ++nd) {
            const int col = nd * 8 + 2 * (lane & 3);
            float2 x = *reinterpret_cast<float2*>(dkr + col);
            x.x += dk[nd][2 * r] * a.scale;
            x.y += dk[nd][2 * r + 1] * a.scale;
            *reinterpret_cast<float2*>(dkr + col) = x;
            float2 y = *reinterpret_cast<float2*>(dvr + col);
            y.x += dv[nd][2 * r];
            y.y += dv[nd][2 * r + 1];
            *reinterpret_cast<float2*>(dvr + col) = y;
        }
    }
}

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

template <int HD>
constexpr int fwd_smem() { return (BM + 4 * BN) * HD * 2; }
template <int HD>
constexpr int dq_smem() { return (2 * BM + 4 * BN) * HD * 2; }
template <int HD>
constexpr int dkv_smem() { return (2 * BN + 4 * BM) * HD * 2 + 4 * BM * 4; }

template <int HD>
void launch_bf16_fwd(const AttnArgs& a, cudaStream_t s) {
    static bool cfg = false;
    if (!cfg) {
        EPP_CUDA(cudaFuncSetAttribute(attn_fwd_bf16<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      fwd_smem<HD>()));
        cfg = true;
    }
    launch_k(attn_fwd_bf16<HD>, dim3(a.nqwork, a.H), 128, fwd_smem<HD>(), s, a);
    EPP_CHECK_LAUNCH();
}

template <int HD>
void launch_bf16_bwd(const AttnArgs& a, cudaStream_t s) {
    static bool cfg = false;
    if (!cfg) {
        EPP_CUDA(cudaFuncSetAttribute(attn_bwd_dq_bf16<HD>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, dq_smem<HD>()));
        EPP_CUDA(cudaFuncSetAttribute(attn_bwd_dkv_bf16<HD>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, dkv_smem<HD>()));
        cfg = true;
    }
    if (a.nqwork > 0) {
        launch_k(attn_bwd_dq_bf16<HD>, dim3(a.nqwork, a.H), 128, dq_smem<HD>(), s, a);
        EPP_CHECK_LAUNCH();
    }
    if (a.nkwork > 0) {
        launch_k(attn_bwd_dkv_bf16<HD>, dim3(a.nkwork, a.Hkv), 128, dkv_smem<HD>(), s, a);
        EPP_CHECK_LAUNCH();
    }
}

}  // namespace

// 1 = tcgen05 kernels (default), 2 = tcgen05 with the fused dK/dV/dQ
// backward, 0 = FA2-style mma.sync kernels.  Initial value from
// EPP_ATTN_IMPL ("fa2", "fused"); switchable at run time through
// epp_gpu_set_attention_impl for A/B tests.
int& attention_impl() {
    static int impl = [] {
        const char* e = getenv("EPP_ATTN_IMPL");
        if (e && std::string(e) == "fa2") return 0;
        if (e && std::string(e) == "fused") return 2;
        return 1;
    }();
    return impl;
}

bool use_tc_attention() { return attention_impl() >= 1; }

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
    if (use_tc_attention() && attn_fwd_tc_supported(a)) {
        attn_fwd_tc(a, s);
        return;
    }
    ProfScope prof(kProfAttnFwd, 4.0 * a.H * a.hd * a.pairs, s);
    if (a.dtype == DType::F32) {
        EPP_REQUIRE(a.hd <= 128, "attn(f32): head_dim <= 128");
        launch_k(attn_fwd_f32, dim3(a.nqwork, a.H), 128, 0, s, a);
        EPP_CHECK_LAUNCH();
        return;
    }
    if (a.hd == 64) launch_bf16_fwd<64>(a, s);
    else if (a.hd == 128) launch_bf16_fwd<128>(a, s);
    else EPP_REQUIRE(false, "attn(bf16): head_dim must be 64 or 128");
}

void attn_bwd(const AttnArgs& a, cudaStream_t s) {
    EPP_REQUIRE(a.H % a.Hkv == 0, "attn: H must be a multiple of Hkv");
    // algorithmic backward = 2x forward (dQ, dK, dV, dP matmuls)
    ProfScope prof(kProfAttnBwd, 8.0 * a.H * a.hd * a.pairs, s);
    if (use_tc_attention() && attn_bwd_tc_supported(a)) {
        attn_bwd_tc_main(a, s);      // the dQ kernel (or the fused path) forms delta
        return;
    }
    attn_delta(a, s);
    EPP_REQUIRE(a.dqkv_out == nullptr, "attn_bwd: dqkv_out needs the tcgen05 kernels");
    if (a.dtype == DType::F32) {
        if (a.nqwork > 0) {
            launch_k(attn_bwd_dq_f32, dim3(a.nqwork, a.H), 128, 0, s, a);
            EPP_CHECK_LAUNCH();
        }
        if (a.nkwork > 0) {
            launch_k(attn_bwd_dkv_f32, dim3(a.nkwork, a.Hkv), 128, 0, s, a);
            EPP_CHECK_LAUNCH();
        }
        return;
    }
    if (a.hd == 64) launch_bf16_bwd<64>(a, s);
    else if (a.hd == 128) launch_bf16_bwd<128>(a, s);
    else EPP_REQUIRE(false, "attn(bf16): head_dim must be 64 or 128");
}

}  // namespace eppk
