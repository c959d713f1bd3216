// epp-b200: GEMMs for the stage executor.
//
// BF16 path: tcgen05.mma (kind::f16, cta_group::1, M=128, N=BN) with the fp32
// accumulator in TMEM, operands staged by TMA (cp.async.bulk.tensor, 128-byte
// swizzle) through a STAGES-deep mbarrier ring.  Warp roles per CTA:
//   warp 0  TMA producer (one elected lane)
//   warp 1  TMEM allocator + MMA issuer (one elected lane)
//   warps 2-5  epilogue: tcgen05.ld -> registers -> fused epilogue -> global
// Both operands may be K-major or MN-major (transposed) in global memory, so
// forward (X W^T), data-gradient (dY W) and weight-gradient (dY^T X) GEMMs all
// run without materialised transposes.
//
// F32 path (parity mode): a register-tiled SIMT kernel with the same operand
// conventions.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <mutex>

#include "common.cuh"
#include "kernels.h"
#include "profile.h"
#include "tc.cuh"

namespace eppk {

static std::atomic<long long> g_gemm_launches{0};
long long gemm_launch_count() { return g_gemm_launches.load(); }



// =========================================================================
// tcgen05 kernel
// =========================================================================
constexpr int kBM = 128;
constexpr int kBK = 64;              // one 128-byte swizzle atom of bf16
constexpr int kThreads = 192;

template <int BN, int STAGES>
struct TcSmem {
    static constexpr int kABytes = kBM * kBK * 2;     // 16 KB
    static constexpr int kBBytes = BN * kBK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kBarOffset = STAGES * kStageBytes;
    static constexpr int kTotal = kBarOffset + (2 * STAGES + 4) * 8 + 16 + 1024;  // + align slack
};

struct TcParams {
    int M, N, K;
    void* C;
    long long ldc;
    const bf16* R;
    long long ldr;
    bf16* C2;
    long long ldc2;
    RopeScatterArgs rope;
    int defer;   // GemmArgs::defer_wait
};

// Persistent CTAs (one per SM) walk the output tiles in a grouped raster
// order; the TMA ring and the two TMEM accumulator buffers persist across
// tiles, so the epilogue of tile i overlaps the mainloop of tile i+1.
struct TileSched {
    int tiles_m, tiles_n;
    __device__ __forceinline__ void coords(int t, int& mb, int& nb) const {
        // groups of 8 M-blocks: consecutive tiles share the same B column
        // panel while sweeping a small set of A row panels (L2 reuse).
        // 8 measured best in the step (profiles/r02_raster_group_ab.json):
        // 16 re-reads B panels half as often and is +2.5 % on isolated
        // forward GEMMs, but neutral-to-worse in the power-capped step; 32
        // overflows L2 with A panels (-4 %)
#ifndef EPP_RASTER_G
#define EPP_RASTER_G 8
#endif
        constexpr int G = EPP_RASTER_G;
        const int per_group = G * tiles_n;
        const int g = t / per_group;
        const int first_m = g * G;
        const int gm = min(G, tiles_m - first_m);
        const int r = t % per_group;
        mb = first_m + r % gm;
        nb = r / gm;
    }
};

// Epilogue of one accumulator row slice: this thread's output row `row`,
// columns [n0, n0 + BN), read 32 columns at a time from TMEM (taddr = the
// warp's lane quarter), fused epilogue, 16-byte stores.  The tcgen05.ld is
// warp-collective, so every lane runs the loop even past the matrix edge.
// Fused QKV epilogue (Epi::RopeScatter): rotate-half RoPE on the q and k
// heads of the tile (column d pairs with d + hd/2 of the same head, so the
// two 32-column chunks are read together), one bf16 rounding, and direct
// stores to q [T, H, hd] and to the segment's K / V rows of this layer —
// the separate rope_qkv_scatter pass and the [T, (H+2Hkv) hd] round trip
// through HBM disappear.
template <int BN>
__device__ __forceinline__ void epilogue_rope(const TcParams& p, uint32_t taddr, int row, int n0) {
    const RopeScatterArgs& rp = p.rope;
    const int hd = rp.hd, half = hd / 2;
    const bool valid = row < p.M;
    const int pos = valid ? rp.tok_pos[row] : 0;
    const AttnSeg* sg = valid ? rp.segs + rp.tok_seg[row] : nullptr;
#pragma unroll 1
    for (int hs = 0; hs < BN; hs += hd) {
        const int slot = (n0 + hs) / hd;
#pragma unroll 1
        for (int cc = 0; cc < half; cc += 32) {
            float a[32], b[32];
            tc::tmem_ld32(taddr + hs + cc, a);          // warp-collective: every lane
            tc::tmem_ld32(taddr + hs + half + cc, b);
            if (!valid || n0 + hs >= p.N) continue;
            if (slot < rp.H + rp.Hkv) {
                const float4* c4 = reinterpret_cast<const float4*>(rp.cs + static_cast<long long>(pos) * half + cc);
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const float4 cs2 = c4[k];          // (cos, sin) of d = cc + 2k, cc + 2k + 1
                    const float a0 = a[2 * k] * cs2.x - b[2 * k] * cs2.y;
                    const float b0 = b[2 * k] * cs2.x + a[2 * k] * cs2.y;
                    const float a1 = a[2 * k + 1] * cs2.z - b[2 * k + 1] * cs2.w;
                    const float b1 = b[2 * k + 1] * cs2.z + a[2 * k + 1] * cs2.w;
                    a[2 * k] = a0; b[2 * k] = b0; a[2 * k + 1] = a1; b[2 * k + 1] = b1;
                }
            }
            bf16* dst;
            if (slot < rp.H) {
                dst = static_cast<bf16*>(rp.q_out) + (static_cast<long long>(row) * rp.H + slot) * hd;
            } else {
                const bool is_k = slot < rp.H + rp.Hkv;
                const int kvh = slot - rp.H - (is_k ? 0 : rp.Hkv);
                dst = static_cast<bf16*>(const_cast<void*>(is_k ? sg->k : sg->v)) + rp.layer * sg->kv_layer_stride +
                      static_cast<long long>(pos) * rp.Hkv * hd + static_cast<long long>(kvh) * hd;
            }
#pragma unroll
            for (int i = 0; i < 32; i += 8) {
                uint4 ra, rb;
                __nv_bfloat162* ha = reinterpret_cast<__nv_bfloat162*>(&ra);
                __nv_bfloat162* hb = reinterpret_cast<__nv_bfloat162*>(&rb);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    ha[j] = __floats2bfloat162_rn(a[i + 2 * j], a[i + 2 * j + 1]);
                    hb[j] = __floats2bfloat162_rn(b[i + 2 * j], b[i + 2 * j + 1]);
                }
                *reinterpret_cast<uint4*>(dst + cc + i) = ra;
                *reinterpret_cast<uint4*>(dst + half + cc + i) = rb;
            }
        }
    }
}

template <int BN, int EPI>
__device__ __forceinline__ void epilogue_plain(const TcParams& p, uint32_t taddr, int row, int n0, bool have_acc);

__device__ __forceinline__ float silu_sig(float g, float& sg) {
    sg = __fdividef(1.f, 1.f + __expf(-g));
    return g * sg;
}
__device__ __forceinline__ void store32_bf16(bf16* dst, const float (&v)[32]) {
#pragma unroll
    for (int i = 0; i < 32; i += 8) {
        uint4 raw;
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw);
#pragma unroll
        for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(v[i + 2 * j], v[i + 2 * j + 1]);
        *reinterpret_cast<uint4*>(dst + i) = raw;
    }
}

// Epi::SwiGlu: the tile's accumulator columns [0, BN/2) are gate features
// j0.., [BN/2, BN) the up features j0.. (the producer loaded w13 rows j0..
// and F+j0.. for the two CTAs' B halves).  h keeps the [gate | up] layout.
template <int BN>
__device__ __forceinline__ void epilogue_swiglu(const TcParams& p, uint32_t taddr, int row, int j0) {
    const int F = p.N / 2;
#pragma unroll 1
    for (int c = 0; c < BN / 2; c += 32) {
        float g[32], u[32];
        tc::tmem_ld32(taddr + c, g);
        tc::tmem_ld32(taddr + BN / 2 + c, u);
        const int col = j0 + c;
        if (row >= p.M || col >= F) continue;
        bf16* h = static_cast<bf16*>(p.C) + static_cast<long long>(row) * p.ldc + col;
        store32_bf16(h, g);
        store32_bf16(h + F, u);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            float sg;
            g[i] = silu_sig(g[i], sg) * u[i];
        }
        store32_bf16(p.C2 + static_cast<long long>(row) * p.ldc2 + col, g);
    }
}

// Epi::SwiGluBwd: acc = dA [., F]; R = h = [g | u].
template <int BN>
__device__ __forceinline__ void epilogue_swiglu_bwd(const TcParams& p, uint32_t taddr, int row, int n0) {
    const int F = p.N;
    // h of chunk c+1 is loaded before chunk c is processed (the row-strided
    // loads are latency-bound; one chunk of lookahead doubles the bytes in
    // flight per thread)
    const bf16* hrow = p.R + static_cast<long long>(min(row, p.M - 1)) * p.ldr + n0;
    uint4 ng[4], nu[4];
    auto load_h = [&](int c) {
        if (row < p.M && n0 + c < F) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                ng[i] = *reinterpret_cast<const uint4*>(hrow + c + 8 * i);
                nu[i] = *reinterpret_cast<const uint4*>(hrow + F + c + 8 * i);
            }
        }
    };
    load_h(0);
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
        uint4 cg[4], cu[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            cg[i] = ng[i];
            cu[i] = nu[i];
        }
        if (c + 32 < BN) load_h(c + 32);
        float d[32];
        tc::tmem_ld32(taddr + c, d);
        const int col = n0 + c;
        if (row >= p.M || col >= F) continue;
        float dg[32], du[32], a[32];
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
            const uint4 rg = cg[i / 8];
            const uint4 ru = cu[i / 8];
            const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&rg);
            const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&ru);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2 gf = __bfloat1622float2(g2[j]), uf = __bfloat1622float2(u2[j]);
                const float gv[2] = {gf.x, gf.y}, uv[2] = {uf.x, uf.y};
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const int e = i + 2 * j + k;
                    float sg;
                    const float si = silu_sig(gv[k], sg);
                    a[e] = si * uv[k];
                    du[e] = d[e] * si;
                    dg[e] = d[e] * uv[k] * sg * (1.f + gv[k] * (1.f - sg));
                }
            }
        }
        bf16* dh = static_cast<bf16*>(p.C) + static_cast<long long>(row) * p.ldc + col;
        store32_bf16(dh, dg);
        store32_bf16(dh + F, du);
        store32_bf16(p.C2 + static_cast<long long>(row) * p.ldc2 + col, a);
    }
}

template <int BN, int EPI>
__device__ __forceinline__ void epilogue_rows(const TcParams& p, uint32_t taddr, int row, int n0, bool have_acc) {
    if constexpr (EPI == static_cast<int>(Epi::RopeScatter)) {
        epilogue_rope<BN>(p, taddr, row, n0);
    } else if constexpr (EPI == static_cast<int>(Epi::SwiGlu)) {
        epilogue_swiglu<BN>(p, taddr, row, n0);
    } else if constexpr (EPI == static_cast<int>(Epi::SwiGluBwd)) {
        epilogue_swiglu_bwd<BN>(p, taddr, row, n0);
    } else {
        epilogue_plain<BN, EPI>(p, taddr, row, n0, have_acc);
    }
}

template <int BN, int EPI>
__device__ __forceinline__ void epilogue_plain(const TcParams& p, uint32_t taddr, int row, int n0, bool have_acc) {
    // AddRes / GeluBwd read R: chunk c+1's R is loaded before chunk c is
    // processed (one chunk of lookahead for the row-strided loads)
    constexpr bool kR = EPI == static_cast<int>(Epi::AddRes) || EPI == static_cast<int>(Epi::GeluBwd);
    const bf16* rrow = kR ? p.R + static_cast<long long>(min(row, p.M - 1)) * p.ldr + n0 : nullptr;
    uint4 nr[4];
    auto load_r = [&](int c) {
        if (kR && row < p.M && n0 + c < p.N) {
#pragma unroll
            for (int i = 0; i < 4; ++i) nr[i] = *reinterpret_cast<const uint4*>(rrow + c + 8 * i);
        }
    };
    load_r(0);
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
        uint4 cr[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) cr[i] = nr[i];
        if (c + 32 < BN) load_r(c + 32);
        float v[32];
        if (have_acc) {
            tc::tmem_ld32(taddr + c, v);
        } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.f;
        }
        const int col = n0 + c;
        if (row >= p.M || col >= p.N) continue;
        if (EPI == static_cast<int>(Epi::AccumF32) || EPI == static_cast<int>(Epi::StoreF32)) {
            float* dst = static_cast<float*>(p.C) + static_cast<long long>(row) * p.ldc + col;
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
                float4 o = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                if (EPI == static_cast<int>(Epi::AccumF32)) {
                    const float4 old = *reinterpret_cast<const float4*>(dst + i);
                    o.x += old.x; o.y += old.y; o.z += old.z; o.w += old.w;
                }
                *reinterpret_cast<float4*>(dst + i) = o;
            }
        } else {
            if (kR) {
                // GeluBwd with C2: also emit gelu(R) (the MLP activation that
                // dW2 needs), re-created here from the h already being read
                bf16* dst2 = (EPI == static_cast<int>(Epi::GeluBwd) && p.C2)
                                 ? p.C2 + static_cast<long long>(row) * p.ldc2 + col : nullptr;
#pragma unroll
                for (int i = 0; i < 32; i += 8) {
                    const uint4 raw = cr[i / 8];
                    const bf16* rb = reinterpret_cast<const bf16*>(&raw);
                    float a[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const float rv = __bfloat162float(rb[j]);
                        if (EPI == static_cast<int>(Epi::AddRes)) {
                            v[i + j] += rv;
                        } else {
                            float dg;
                            a[j] = gelu_tanh_and_grad_fast_f(rv, dg);
                            v[i + j] *= dg;
                        }
                    }
                    if (EPI == static_cast<int>(Epi::GeluBwd) && dst2) {
                        uint4 out;
                        __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&out);
#pragma unroll
                        for (int j = 0; j < 4; ++j) h2[j] = __floats2bfloat162_rn(a[2 * j], a[2 * j + 1]);
                        *reinterpret_cast<uint4*>(dst2 + i) = out;
                    }
                }
            }
            if (EPI == static_cast<int>(Epi::StoreGelu)) {
                bf16* dst2 = p.C2 + static_cast<long long>(row) * p.ldc2 + col;
#pragma unroll
                for (int i = 0; i < 32; i += 8) {
                    uint4 raw;
                    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw);
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        h[j] = __floats2bfloat162_rn(gelu_tanh_fast_f(v[i + 2 * j]), gelu_tanh_fast_f(v[i + 2 * j + 1]));
                    *reinterpret_cast<uint4*>(dst2 + i) = raw;
                }
            }
            bf16* dst = static_cast<bf16*>(p.C) + static_cast<long long>(row) * p.ldc + col;
#pragma unroll
            for (int i = 0; i < 32; i += 8) {
                uint4 raw;
                __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw);
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    h[j] = __floats2bfloat162_rn(v[i + 2 * j], v[i + 2 * j + 1]);
                *reinterpret_cast<uint4*>(dst + i) = raw;
            }
        }
    }
}

template <int BN, int STAGES, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap map_a,
                   const __grid_constant__ CUtensorMap map_b, const TcParams p) {
    if (!p.defer) pdl_wait();
    pdl_trigger();
    using L = TcSmem<BN, STAGES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const uint32_t sbase = (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) + 1023u) & ~1023u;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
    uint64_t* empty = full + STAGES;
    uint64_t* acc_full = empty + STAGES;     // [2]
    uint64_t* acc_empty = acc_full + 2;      // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);   // warp-uniform for the compiler
    const int lane = threadIdx.x & 31;
    const int nk = (p.K + kBK - 1) / kBK;
    const TileSched sched{(p.M + kBM - 1) / kBM, (p.N + BN - 1) / BN};
    const int ntiles = sched.tiles_m * sched.tiles_n;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&acc_full[b], 1);
            tc::mbar_init(&acc_empty[b], 4);     // one arrive per epilogue warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
    }
    constexpr uint32_t kTmemCols = 2 * BN;     // double-buffered accumulator
    if (warp == 1) tc::tmem_alloc(tmem_slot, kTmemCols);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                int mb, nb;
                sched.coords(t, mb, nb);
                const int m0 = mb * kBM, n0 = nb * BN;
                for (int kb = 0; kb < nk; ++kb) {
                    tc::mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* sa = smem + stage * L::kStageBytes;
                    uint8_t* sb = sa + L::kABytes;
                    tc::mbar_expect_tx(&full[stage], L::kStageBytes);
                    const int k0 = kb * kBK;
                    if (A_MN) {
#pragma unroll
                        for (int i = 0; i < kBM / 64; ++i)
                            tc::tma_load_2d(sa + i * 8192, &map_a, &full[stage], m0 + 64 * i, k0);
                    } else {
                        tc::tma_load_2d(sa, &map_a, &full[stage], k0, m0);
                    }
                    if (B_MN) {
#pragma unroll
                        for (int i = 0; i < BN / 64; ++i)
                            tc::tma_load_2d(sb + i * 8192, &map_b, &full[stage], n0 + 64 * i, k0);
                    } else {
                        tc::tma_load_2d(sb, &map_b, &full[stage], k0, n0);
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        constexpr uint32_t idesc = tc::instr_desc(BN, A_MN, B_MN);
        int stage = 0;
        uint32_t phase = 0;
        int local = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++local) {
            const int acc = local & 1;
            const uint32_t acc_phase = (local >> 1) & 1;
            tc::mbar_wait(&acc_empty[acc], acc_phase ^ 1);     // epilogue drained this buffer
            tc::fence_after();
            const uint32_t d = tmem + acc * BN;
            for (int kb = 0; kb < nk; ++kb) {
                tc::mbar_wait(&full[stage], phase);
                tc::fence_after();
                // whole warp, one elected lane issues the 4 K16 steps of the
                // stage (K-major: +32 B per step; MN-major: +2 KB per step)
                const uint32_t sa = sbase + stage * L::kStageBytes;
                const uint32_t sb = sa + L::kABytes;
                const uint64_t ad = A_MN ? tc::smem_desc(sa, 8192, 1024) : tc::smem_desc(sa, 16, 1024);
                const uint64_t bd = B_MN ? tc::smem_desc(sb, 8192, 1024) : tc::smem_desc(sb, 16, 1024);
                static_assert(kBK == 64, "one 4-step batch per stage");
                tc::mma4_ss<A_MN ? 128 : 2, B_MN ? 128 : 2>(d, ad, bd, idesc, kb != 0);
                tc::commit_w(&empty[stage]);
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            tc::commit_w(&acc_full[acc]);
        }
    } else {
        // ---------------- epilogue (warps 2..5) ----------------
        const int quarter = warp & 3;                  // TMEM lane quarter
        int local = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++local) {
            int mb, nb;
            sched.coords(t, mb, nb);
            const int row = mb * kBM + quarter * 32 + lane;
            const int n0 = nb * BN;
            const int acc = local & 1;
            if (nk > 0) {
                tc::mbar_wait(&acc_full[acc], (local >> 1) & 1);
                tc::fence_after();
            }
            epilogue_rows<BN, EPI>(p, tmem + acc * BN + (static_cast<uint32_t>(quarter * 32) << 16), row, n0, nk > 0);
            // release the accumulator buffer to the MMA warp
            tc::fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&acc_empty[acc]);
        }
    }
    if (p.defer) pdl_wait();   // completion of this grid implies the previous one's
    __syncthreads();
    if (warp == 1) {
        tc::fence_after();
        tc::tmem_dealloc(tmem, kTmemCols);
    }
}


// =========================================================================
// CTA-pair kernel (cta_group::2): a cluster of two CTAs on one TPC computes
// a 256 x BN tile with M=256 MMAs issued by the leader CTA.  Each CTA stages
// its own 128 rows of A and BN/2 rows of B (the MMA reads the peer's halves
// through the pair's shared-memory path), so per SM the TMA and tensor-core
// shared-memory traffic per FLOP is 2/3 of the single-CTA 128 x 256 tile and
// the issuing warp runs at half the rate.  Barriers:
//   full[s]      leader only: its producer arms 2 x stage bytes, both CTAs'
//                TMA loads complete_tx on it (peer bit cleared in the address)
//   empty[s]     both CTAs: the leader's MMA commit multicasts to the pair
//   acc_full[b]  both CTAs: multicast commit after a tile's last MMA
//   acc_empty[b] leader only: 4 epilogue warps x 2 CTAs arrive (peer: remote)
// =========================================================================
// TMA-staged bf16 epilogues of the pair kernel (Store, AddRes, StoreGelu,
// GeluBwd, SwiGlu, SwiGluBwd).  An epilogue thread owns one accumulator row
// (the tcgen05.ld 32x32b shape), so direct global stores / residual loads are
// one 16-byte access per row and lane: 32 L1 wavefronts per warp instruction,
// and every extra row-strided stream cost ~10 % of the GEMM at K = 2048
// (tools/gemm_bench.py: store 1462, + residual load 1311, GELU' with h load
// and gelu(h) store 1075 TFLOP/s) because those wavefronts share the SM's
// L1 / shared-memory data path with the TMA writes and MMA reads of the main
// loop.  Here each warp moves 32 x 32 bf16 boxes (64-byte swizzle) through
// shared memory: residual / h boxes arrive by TMA (two slots, one group of
// lookahead), outputs leave by TMA bulk stores; the warp's shared-memory
// accesses are 4 wavefronts per instruction.
template <int EPI>
struct EpiTma {
    static constexpr bool kOn = EPI == static_cast<int>(Epi::Store) || EPI == static_cast<int>(Epi::AddRes) ||
                                EPI == static_cast<int>(Epi::StoreGelu) || EPI == static_cast<int>(Epi::GeluBwd) ||
                                EPI == static_cast<int>(Epi::SwiGlu) || EPI == static_cast<int>(Epi::SwiGluBwd);
    // R streams per 32-column group: residual, h, or SwiGLU's gate and up halves of h
    static constexpr int kR = EPI == static_cast<int>(Epi::AddRes) || EPI == static_cast<int>(Epi::GeluBwd) ? 1
                              : EPI == static_cast<int>(Epi::SwiGluBwd)                                   ? 2
                                                                                                          : 0;
    // output boxes per group: C (SwiGLU: both halves of h / dh) and C2
    static constexpr int kOut = EPI == static_cast<int>(Epi::Store) || EPI == static_cast<int>(Epi::AddRes) ? 1
                                : EPI == static_cast<int>(Epi::StoreGelu) || EPI == static_cast<int>(Epi::GeluBwd) ? 2
                                : kOn ? 3 : 0;
    static constexpr int kBox = 32 * 64;            // 32 rows x 32 bf16
    static constexpr int kRSlots = kR ? 2 : 0;
    // one output buffer set when there are several outputs: keeps the main
    // loop's six TMA stages (GELU': 1212 -> 1222, SwiGLU' 1025 -> 1075 TFLOP/s
    // at K = 2048) at the price of a wait for the previous group's stores
    static constexpr int kOutBufs = kOut >= 2 ? 1 : 2;
    static constexpr int kWarpBytes = (kRSlots * kR + kOutBufs * kOut) * kBox;
};

// 64-byte swizzle: 16-byte chunk j of a 64-byte row r sits at j ^ ((r >> 1) & 3)
__device__ __forceinline__ uint32_t sw64(int r, int j) { return r * 64 + ((j ^ ((r >> 1) & 3)) << 4); }

__device__ __forceinline__ void box_store_row(uint8_t* box, int r, const float (&v)[32]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        uint4 raw;
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw);
#pragma unroll
        for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(v[8 * j + 2 * k], v[8 * j + 2 * k + 1]);
        *reinterpret_cast<uint4*>(box + sw64(r, j)) = raw;
    }
}
__device__ __forceinline__ void box_load_row(const uint8_t* box, int r, float (&v)[32]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint4 raw = *reinterpret_cast<const uint4*>(box + sw64(r, j));
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float2 f = __bfloat1622float2(h[k]);
            v[8 * j + 2 * k] = f.x;
            v[8 * j + 2 * k + 1] = f.y;
        }
    }
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const uint8_t* box, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(tc::smem_u32(box))
                 : "memory");
}

// Per-warp state of the TMA epilogue across tiles.
struct EpiTmaState {
    uint32_t r_used = 0;     // R groups consumed (slot = r_used & 1)
    uint32_t stored = 0;     // output groups committed (buffer = stored & 1)
};

// One tile's epilogue for one warp: rows row0 .. row0 + 31 (this thread:
// row0 + lane), accumulator columns [0, kCols) at taddr; output column of
// accumulator column 0 = n0 (SwiGlu: gate feature j0 = n0).
template <int BN, int EPI>
__device__ __forceinline__ void epilogue_tma(const TcParams& p, const CUtensorMap* map_r, const CUtensorMap* map_c,
                                             const CUtensorMap* map_c2, uint32_t taddr, uint8_t* ebuf,
                                             uint64_t* rbar, int row0, int n0, int lane, EpiTmaState& st) {
    using E = EpiTma<EPI>;
    constexpr bool kSwi = EPI == static_cast<int>(Epi::SwiGlu);
    constexpr bool kSwiB = EPI == static_cast<int>(Epi::SwiGluBwd);
    constexpr int kCols = kSwi ? BN / 2 : BN;            // accumulator columns walked (SwiGlu: gate half)
    const int nlog = kSwi ? p.N / 2 : p.N;                // columns of the logical output
    const int F = kSwi ? p.N / 2 : p.N;                   // SwiGLU halves
    const int groups = max(0, min(kCols, nlog - n0)) / 32;
    const bool rows_live = row0 < p.M;
    const bool has_c2 = p.C2 != nullptr;
    uint8_t* rbase = ebuf;
    uint8_t* obase = ebuf + E::kRSlots * E::kR * E::kBox;
    auto issue_r = [&](int gi, uint32_t k) {   // lane 0: R boxes of group gi, the warp's k-th R group
        const int slot = k & 1;
        uint64_t* bar = rbar + slot;
        tc::mbar_expect_tx(bar, E::kR * E::kBox);
        const int col = n0 + 32 * gi;
        tc::tma_load_2d(rbase + (slot * E::kR) * E::kBox, map_r, bar, col, row0);
        if constexpr (E::kR == 2) tc::tma_load_2d(rbase + (slot * E::kR + 1) * E::kBox, map_r, bar, F + col, row0);
    };
    if constexpr (E::kR > 0) {
        if (lane == 0 && rows_live) {
            if (groups > 0) issue_r(0, st.r_used);
            if (groups > 1) issue_r(1, st.r_used + 1);
        }
    }
#pragma unroll 1
    for (int gi = 0; gi < groups; ++gi) {
        const int col = n0 + 32 * gi;
        float v[32], w[32];
        tc::tmem_ld32(taddr + 32 * gi, v);
        if constexpr (kSwi) tc::tmem_ld32(taddr + BN / 2 + 32 * gi, w);
        if (!rows_live) continue;       // warp-uniform: the whole 32-row box lies past M
        float r0[32], r1[32];
        if constexpr (E::kR > 0) {
            const int slot = st.r_used & 1;
            tc::mbar_wait(rbar + slot, (st.r_used >> 1) & 1);
            box_load_row(rbase + (slot * E::kR) * E::kBox, lane, r0);
            if constexpr (E::kR == 2) box_load_row(rbase + (slot * E::kR + 1) * E::kBox, lane, r1);
            tc::fence_proxy_async();
            __syncwarp();
            ++st.r_used;
            // the slot just read takes group gi + 2
            if (lane == 0 && gi + 2 < groups) issue_r(gi + 2, st.r_used + 1);
        }
        // outputs: o0 -> C (col), o1 -> C (F + col) for SwiGLU / C2 otherwise, o2 -> C2 (SwiGLU)
        float o1[32], o2[32];
        if constexpr (EPI == static_cast<int>(Epi::AddRes)) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] += r0[i];
        } else if constexpr (EPI == static_cast<int>(Epi::StoreGelu)) {
#pragma unroll
            for (int i = 0; i < 32; ++i) o1[i] = gelu_tanh_fast_f(v[i]);
        } else if constexpr (EPI == static_cast<int>(Epi::GeluBwd)) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                float dg;
                o1[i] = gelu_tanh_and_grad_fast_f(r0[i], dg);
                v[i] *= dg;
            }
        } else if constexpr (kSwi) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                float sg;
                o1[i] = w[i];
                o2[i] = silu_sig(v[i], sg) * w[i];
            }
        } else if constexpr (kSwiB) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                float sg;
                const float g = r0[i], u = r1[i], d = v[i];
                const float si = silu_sig(g, sg);
                o2[i] = si * u;
                o1[i] = d * si;
                v[i] = d * u * sg * (1.f + g * (1.f - sg));
            }
        }
        const int buf = E::kOutBufs == 2 ? (st.stored & 1) : 0;
        if (st.stored >= E::kOutBufs) {   // this buffer's stores (kOutBufs groups ago) must have been read
            if (lane == 0) {
                if constexpr (E::kOutBufs == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
            __syncwarp();
        }
        uint8_t* ob = obase + buf * E::kOut * E::kBox;
        box_store_row(ob, lane, v);
        if constexpr (E::kOut >= 2) box_store_row(ob + E::kBox, lane, o1);
        if constexpr (E::kOut >= 3) box_store_row(ob + 2 * E::kBox, lane, o2);
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
            tma_store_2d(map_c, ob, col, row0);
            if constexpr (kSwi || kSwiB) {
                tma_store_2d(map_c, ob + E::kBox, F + col, row0);
                tma_store_2d(map_c2, ob + 2 * E::kBox, col, row0);
            } else if constexpr (E::kOut >= 2) {
                if (has_c2) tma_store_2d(map_c2, ob + E::kBox, col, row0);
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        ++st.stored;
    }
}

template <int BN, int STAGES, int EPI = 0>
struct Tc2Smem {
    static constexpr int kABytes = kBM * kBK * 2;            // this CTA's 128 rows of A
    static constexpr int kBBytes = (BN / 2) * kBK * 2;       // this CTA's BN/2 rows of B
    static constexpr int kStageBytes = kABytes + kBBytes;
    // AccumF32: per epilogue warp two [32 rows x 32 fp32] staging boxes for
    // the TMA reduce-add into C
    static constexpr int kEpiOffset = STAGES * kStageBytes;
    static constexpr int kEpiBytes = EPI == static_cast<int>(Epi::AccumF32) ? 4 * 2 * 4096
                                     : EpiTma<EPI>::kOn                    ? 4 * EpiTma<EPI>::kWarpBytes
                                                                           : 0;
    static constexpr int kBarOffset = kEpiOffset + kEpiBytes;
    static constexpr int kTotal = kBarOffset + (2 * STAGES + 4 + 8) * 8 + 16 + 1024;   // + 2 R barriers per epilogue warp
};

// Weight-gradient epilogue (Epi::AccumF32) of the pair kernel: C(fp32) +=
// acc without reading C into the SM.  Each epilogue warp moves its 32 rows x
// 32 columns of the accumulator to a swizzled shared-memory box and one lane
// issues a TMA reduce-add of the box into C (the L2 performs the
// read-modify-write; the tensor map clips rows / columns past M / N).  Two
// boxes per warp alternate, so the bulk reduction of one overlaps the TMEM
// load of the next.  The per-row float4 read-modify-write this replaces kept
// every epilogue warp waiting on uncoalesced HBM reads, and for short chunks
// (K = a 2K-token chunk) the epilogue outlasted the next tile's main loop:
// 0.85-0.88 PFLOP/s against 1.29-1.31 for the bf16-store GEMMs.
template <int BN>
__device__ __forceinline__ void epilogue_accum_tma(const CUtensorMap* map_c, uint32_t taddr, uint8_t* ebuf,
                                                   int row0, int n0, int lane, int& issued) {
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
        float v[32];
        tc::tmem_ld32(taddr + c, v);
        const int buf = issued & 1;
        if (issued >= 2) {   // the box we are about to overwrite was issued two reductions ago
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncwarp();
        }
        uint8_t* box = ebuf + buf * 4096 + lane * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j)   // 128-byte swizzle: 16-byte chunk j of row r at j ^ (r & 7)
            *reinterpret_cast<float4*>(box + ((j ^ (lane & 7)) << 4)) =
                make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
            asm volatile(
                "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                    reinterpret_cast<uint64_t>(map_c)),
                "r"(n0 + c), "r"(row0), "r"(tc::smem_u32(ebuf + buf * 4096))
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        ++issued;
    }
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA 2-D load whose completion is counted on the LEADER CTA's barrier.
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, uint32_t leader_bar, int c0,
                                                 int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1)
        : "memory");
}
// Four K16 MMAs, cta_group::2 (see tc::mma4_ss).
template <int A_STEP, int B_STEP>
__device__ __forceinline__ void mma4_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t acc0) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 a, b;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "mov.b64 a, %1;\n\tmov.b64 b, %2;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, p;\n\t"
        "add.s64 a, a, %5;\n\tadd.s64 b, b, %6;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, 1;\n\t"
        "add.s64 a, a, %5;\n\tadd.s64 b, b, %6;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, 1;\n\t"
        "add.s64 a, a, %5;\n\tadd.s64 b, b, %6;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, 1;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc0), "n"(A_STEP), "n"(B_STEP)
        : "memory");
}
__device__ __forceinline__ void commit_pair(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
            tc::smem_u32(bar)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
}

template <int BN, int STAGES, bool A_MN, bool B_MN, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap map_a,
                    const __grid_constant__ CUtensorMap map_b, const __grid_constant__ CUtensorMap map_c,
                    const __grid_constant__ CUtensorMap map_r, const __grid_constant__ CUtensorMap map_c2,
                    const TcParams p) {
    if (!p.defer) pdl_wait();   // deferred: see GemmArgs::defer_wait
    pdl_trigger();
    using L = Tc2Smem<BN, STAGES, EPI>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const uint32_t sbase = (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) + 1023u) & ~1023u;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
    uint64_t* empty = full + STAGES;
    uint64_t* acc_full = empty + STAGES;     // [2]
    uint64_t* acc_empty = acc_full + 2;      // [2]
    uint64_t* rbar = acc_empty + 2;          // [4 epilogue warps][2 R slots] (TMA epilogues)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + 8);

    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);   // warp-uniform for the compiler
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int nk = (p.K + kBK - 1) / kBK;
    // SwiGlu: a tile covers BN/2 gate and the same BN/2 up features
    constexpr bool kSwi = EPI == static_cast<int>(Epi::SwiGlu);
    static_assert(!kSwi || !B_MN, "SwiGlu: K-major w13");
    constexpr int kTileN = kSwi ? BN / 2 : BN;
    const int n_logical = kSwi ? p.N / 2 : p.N;
    const TileSched sched{(p.M + 2 * kBM - 1) / (2 * kBM), (n_logical + kTileN - 1) / kTileN};
    const int ntiles = sched.tiles_m * sched.tiles_n;
    const int cluster_id = blockIdx.x >> 1, nclusters = gridDim.x >> 1;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&acc_full[b], 1);
            tc::mbar_init(&acc_empty[b], 8);     // 4 epilogue warps x 2 CTAs (leader's copy)
        }
        for (int b = 0; b < 8; ++b) tc::mbar_init(&rbar[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
    }
    constexpr uint32_t kTmemCols = 2 * BN;     // double-buffered accumulator (this CTA's 128 rows)
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(tmem_slot)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc::fence_before();
    cluster_sync_all();      // barrier inits and the TMEM allocation visible to the pair
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer (both CTAs) ----------------
        if (lane == 0) {
            const uint32_t leader_full0 = tc::smem_u32(full) & 0xFEFFFFFFu;   // peer bit cleared
            int stage = 0;
            uint32_t phase = 0;
            for (int t = cluster_id; t < ntiles; t += nclusters) {
                int mb, nb;
                sched.coords(t, mb, nb);
                const int m0 = mb * 2 * kBM + rank * kBM;
                const int n0 = kSwi ? nb * kTileN + rank * (p.N / 2) : nb * BN + rank * (BN / 2);
                for (int kb = 0; kb < nk; ++kb) {
                    tc::mbar_wait(&empty[stage], phase ^ 1);
                    if (leader) tc::mbar_expect_tx(&full[stage], 2 * L::kStageBytes);
                    const uint32_t sa = sbase + stage * L::kStageBytes;
                    const uint32_t sb = sa + L::kABytes;
                    const uint32_t fb = leader_full0 + stage * 8;
                    const int k0 = kb * kBK;
                    if (A_MN) {
#pragma unroll
                        for (int i = 0; i < kBM / 64; ++i) tma_load_2d_pair(sa + i * 8192, &map_a, fb, m0 + 64 * i, k0);
                    } else {
                        tma_load_2d_pair(sa, &map_a, fb, k0, m0);
                    }
                    if (B_MN) {
#pragma unroll
                        for (int i = 0; i < BN / 128; ++i) tma_load_2d_pair(sb + i * 8192, &map_b, fb, n0 + 64 * i, k0);
                    } else {
                        tma_load_2d_pair(sb, &map_b, fb, k0, n0);
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (leader CTA only) ----------------
        if (leader) {
            constexpr uint32_t idesc = tc::instr_desc_mn(2 * kBM, BN, A_MN, B_MN);
            int stage = 0;
            uint32_t phase = 0;
            int local = 0;
            for (int t = cluster_id; t < ntiles; t += nclusters, ++local) {
                const int acc = local & 1;
                tc::mbar_wait(&acc_empty[acc], ((local >> 1) & 1) ^ 1);   // both CTAs drained this buffer
                tc::fence_after();
                const uint32_t d = tmem + acc * BN;
                for (int kb = 0; kb < nk; ++kb) {
                    tc::mbar_wait(&full[stage], phase);
                    tc::fence_after();
                    const uint32_t sa = sbase + stage * L::kStageBytes;
                    const uint32_t sb = sa + L::kABytes;
                    const uint64_t ad = A_MN ? tc::smem_desc(sa, 8192, 1024) : tc::smem_desc(sa, 16, 1024);
                    const uint64_t bd = B_MN ? tc::smem_desc(sb, 8192, 1024) : tc::smem_desc(sb, 16, 1024);
                    mma4_pair<A_MN ? 128 : 2, B_MN ? 128 : 2>(d, ad, bd, idesc, kb != 0);
                    commit_pair(&empty[stage]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                commit_pair(&acc_full[acc]);
            }
        }
    } else {
        // ---------------- epilogue (warps 2..5, both CTAs) ----------------
        const int quarter = warp & 3;
        uint32_t leader_acc_empty0;
        asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(leader_acc_empty0) : "r"(tc::smem_u32(acc_empty)));
        int local = 0, issued = 0;
        constexpr bool kTma = EpiTma<EPI>::kOn;
        uint8_t* ebuf = smem + L::kEpiOffset + quarter * (kTma ? EpiTma<EPI>::kWarpBytes : 8192);
        EpiTmaState est;
        for (int t = cluster_id; t < ntiles; t += nclusters, ++local) {
            int mb, nb;
            sched.coords(t, mb, nb);
            const int row = mb * 2 * kBM + rank * kBM + quarter * 32 + lane;
            const int n0 = nb * kTileN;
            const int acc = local & 1;
            tc::mbar_wait(&acc_full[acc], (local >> 1) & 1);
            tc::fence_after();
            const uint32_t taddr = tmem + acc * BN + (static_cast<uint32_t>(quarter * 32) << 16);
            if constexpr (EPI == static_cast<int>(Epi::AccumF32))
                epilogue_accum_tma<BN>(&map_c, taddr, ebuf, row - lane, n0, lane, issued);
            else if constexpr (kTma)
                epilogue_tma<BN, EPI>(p, &map_r, &map_c, &map_c2, taddr, ebuf, rbar + 2 * quarter, row - lane, n0, lane,
                                      est);
            else
                epilogue_rows<BN, EPI>(p, taddr, row, n0, true);
            tc::fence_before();
            __syncwarp();
            if (lane == 0)
                asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                                 leader_acc_empty0 + acc * 8)
                             : "memory");
        }
        if ((EPI == static_cast<int>(Epi::AccumF32) || kTma) && lane == 0)
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // staging boxes read, C updated
    }
    if (p.defer) pdl_wait();   // completion of this grid implies the previous one's
    tc::fence_before();
    cluster_sync_all();
    if (warp == 1) {
        tc::fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
    }
}

// =========================================================================
// Host side: tensor maps + dispatch
// =========================================================================
namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        EPP_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p)
            throw CudaError("cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// 2-D bf16 tensor [rows, cols] (cols contiguous, row pitch ld elements),
// box = [box_cols (inner), box_rows].
CUtensorMap make_map(const void* base, long long rows, long long cols, long long ld,
                     int box_cols, int box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base),
                                   dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
    return m;
}

// 2-D fp32 tensor [rows, cols], 128-byte swizzle, box = [box_cols, box_rows].
CUtensorMap make_map_f32(const void* base, long long rows, long long cols, long long ld, int box_cols,
                         int box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 4};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw CudaError("cuTensorMapEncodeTiled (f32) failed (" + std::to_string(static_cast<int>(r)) + ")");
    return m;
}

// 2-D bf16 tensor [rows, cols], 64-byte swizzle, 32 x 32 boxes (the TMA epilogues).
CUtensorMap make_map_sw64(const void* base, long long rows, long long cols, long long ld) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
    const cuuint32_t box[2] = {32, 32};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw CudaError("cuTensorMapEncodeTiled (sw64) failed (" + std::to_string(static_cast<int>(r)) + ")");
    return m;
}

// Deepest TMA ring (<= MAX stages) whose shared memory fits next to the
// epilogue staging of EPI.
template <int BN, int MAX, int EPI>
constexpr int pair_stages() {
    int st = MAX;
    while (st > 2 && Tc2Smem<BN, 0, EPI>::kEpiBytes + st * Tc2Smem<BN, 0, EPI>::kStageBytes + (2 * st + 12) * 8 + 16 +
                             1024 > 227 * 1024)
        --st;
    return st;
}

}  // namespace

// bf16 tensor map with 128-byte swizzle: dims[0] is the contiguous one,
// strides_b[i] = byte stride of dims[i+1].
CUtensorMap make_tma_map(const void* base, int rank, const unsigned long long* dims,
                         const unsigned long long* strides_b, const unsigned* box) {
    CUtensorMap m;
    cuuint64_t d[5], st[4];
    cuuint32_t b[5], es[5];
    for (int i = 0; i < rank; ++i) {
        d[i] = dims[i];
        b[i] = box[i];
        es[i] = 1;
        if (i + 1 < rank) st[i] = strides_b[i];
    }
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), d, st,
                                   b, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
    return m;
}

namespace {

template <int BN, int STAGES, bool A_MN, bool B_MN, int EPI>
void launch_tc(const GemmArgs& g, cudaStream_t s) {
    using L = TcSmem<BN, STAGES>;
    auto kern = gemm_tc_kernel<BN, STAGES, A_MN, B_MN, EPI>;
    static bool configured = false;   // per instantiation
    if (!configured) {
        EPP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kTotal));
        configured = true;
    }
    // A: K-major -> tensor [M, K]; MN-major -> tensor [K, M].
    const CUtensorMap ma = A_MN ? make_map(g.A, g.K, g.M, g.lda, 64, kBK)
                                : make_map(g.A, g.M, g.K, g.lda, kBK, kBM);
    const CUtensorMap mb = B_MN ? make_map(g.B, g.K, g.N, g.ldb, 64, kBK)
                                : make_map(g.B, g.N, g.K, g.ldb, kBK, BN);
    TcParams p{g.M, g.N, g.K, g.C, g.ldc, static_cast<const bf16*>(g.R), g.ldr,
               static_cast<bf16*>(g.C2), g.ldc2, g.rope ? *g.rope : RopeScatterArgs{}, g.defer_wait ? 1 : 0};
    static int num_sms = 0;
    if (!num_sms) {
        int dev = 0;
        EPP_CUDA(cudaGetDevice(&dev));
        EPP_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    const int tiles = ceil_div(g.N, BN) * ceil_div(g.M, kBM);
    launch_k(kern, std::min(tiles, num_sms), kThreads, L::kTotal, s, ma, mb, p);
    EPP_CHECK_LAUNCH();
    g_gemm_launches.fetch_add(1);
}


template <int BN, int STAGES, int EPI>
void dispatch_major(const GemmArgs& g, cudaStream_t s) {
    const bool a_mn = !g.a_kmajor, b_mn = !g.b_kmajor;
    if (!a_mn && !b_mn) launch_tc<BN, STAGES, false, false, EPI>(g, s);
    else if (!a_mn && b_mn) launch_tc<BN, STAGES, false, true, EPI>(g, s);
    else if (a_mn && !b_mn) launch_tc<BN, STAGES, true, false, EPI>(g, s);
    else launch_tc<BN, STAGES, true, true, EPI>(g, s);
}

template <int BN, int STAGES>
void dispatch_epi(const GemmArgs& g, cudaStream_t s) {
    switch (g.epi) {
        case Epi::Store: dispatch_major<BN, STAGES, 0>(g, s); break;
        case Epi::AccumF32: dispatch_major<BN, STAGES, 1>(g, s); break;
        case Epi::AddRes: dispatch_major<BN, STAGES, 2>(g, s); break;
        case Epi::StoreF32: dispatch_major<BN, STAGES, 3>(g, s); break;
        case Epi::StoreGelu: dispatch_major<BN, STAGES, 4>(g, s); break;
        case Epi::GeluBwd: dispatch_major<BN, STAGES, 5>(g, s); break;
        case Epi::RopeScatter:
            EPP_REQUIRE(g.a_kmajor && g.b_kmajor && g.rope, "RopeScatter: K-major operands and rope args");
            launch_tc<BN, STAGES, false, false, 6>(g, s);
            break;
        case Epi::SwiGlu:
        case Epi::SwiGluBwd:
            EPP_REQUIRE(false, "SwiGlu epilogues run on the CTA-pair kernel only (gemm_swiglu_fusable)");
            break;
    }
}

template <int BN, int STAGES, bool A_MN, bool B_MN, int EPI>
void launch_tc2(const GemmArgs& g, cudaStream_t s) {
    constexpr int S = pair_stages<BN, STAGES, EPI>();   // the TMA epilogues' staging can cost a ring stage
    using L = Tc2Smem<BN, S, EPI>;
    auto kern = gemm_tc2_kernel<BN, S, A_MN, B_MN, EPI>;
    static bool configured = false;   // per instantiation
    if (!configured) {
        EPP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kTotal));
        configured = true;
    }
    // per CTA: A box = 128 rows (or 64-col MN boxes), B box = BN/2 rows
    const CUtensorMap ma = A_MN ? make_map(g.A, g.K, g.M, g.lda, 64, kBK)
                                : make_map(g.A, g.M, g.K, g.lda, kBK, kBM);
    const CUtensorMap mb = B_MN ? make_map(g.B, g.K, g.N, g.ldb, 64, kBK)
                                : make_map(g.B, g.N, g.K, g.ldb, kBK, BN / 2);
    TcParams p{g.M, g.N, g.K, g.C, g.ldc, static_cast<const bf16*>(g.R), g.ldr,
               static_cast<bf16*>(g.C2), g.ldc2, g.rope ? *g.rope : RopeScatterArgs{}, g.defer_wait ? 1 : 0};
    static int num_sms = 0;
    if (!num_sms) {
        int dev = 0;
        EPP_CUDA(cudaGetDevice(&dev));
        EPP_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    const int tiles = ceil_div(g.N, BN) * ceil_div(g.M, 2 * kBM);
    const int clusters = std::min(tiles, num_sms / 2);
    // C as an fp32 [M, N] tensor, 32 x 32 boxes (the AccumF32 reduce-add);
    // the TMA epilogues' bf16 C / R / C2 tensors in 32 x 32 boxes
    CUtensorMap mc{}, mr{}, mc2{};
    if (EPI == static_cast<int>(Epi::AccumF32)) mc = make_map_f32(g.C, g.M, g.N, g.ldc, 32, 32);
    if constexpr (EpiTma<EPI>::kOn) {
        constexpr bool kSwi = EPI == static_cast<int>(Epi::SwiGlu), kSwiB = EPI == static_cast<int>(Epi::SwiGluBwd);
        auto aligned = [](const void* q, long long ld) {
            return (reinterpret_cast<uintptr_t>(q) & 15) == 0 && ld % 8 == 0;
        };
        // C: [M, N] (SwiGluBwd: dh = [M, 2N]); R: [M, N] (SwiGluBwd: h = [M, 2N]);
        // C2: [M, N] (SwiGlu: [M, N/2])
        mc = make_map_sw64(g.C, g.M, kSwiB ? 2LL * g.N : g.N, g.ldc);
        if (EpiTma<EPI>::kR) {
            EPP_REQUIRE(g.R && aligned(g.R, g.ldr), "gemm: R must be 16-byte aligned with ldr % 8 == 0");
            mr = make_map_sw64(g.R, g.M, kSwiB ? 2LL * g.N : g.N, g.ldr);
        }
        if (EpiTma<EPI>::kOut >= 2 && g.C2) {
            EPP_REQUIRE(aligned(g.C2, g.ldc2), "gemm: C2 must be 16-byte aligned with ldc2 % 8 == 0");
            mc2 = make_map_sw64(g.C2, g.M, kSwi ? g.N / 2 : g.N, g.ldc2);
        }
    }
    launch_k(kern, 2 * clusters, kThreads, L::kTotal, s, ma, mb, mc, mr, mc2, p);
    EPP_CHECK_LAUNCH();
    g_gemm_launches.fetch_add(1);
}

template <int BN, int STAGES, int EPI>
void dispatch_major2(const GemmArgs& g, cudaStream_t s) {
    const bool a_mn = !g.a_kmajor, b_mn = !g.b_kmajor;
    if (!a_mn && !b_mn) launch_tc2<BN, STAGES, false, false, EPI>(g, s);
    else if (!a_mn && b_mn) launch_tc2<BN, STAGES, false, true, EPI>(g, s);
    else if (a_mn && !b_mn) launch_tc2<BN, STAGES, true, false, EPI>(g, s);
    else launch_tc2<BN, STAGES, true, true, EPI>(g, s);
}

template <int BN, int STAGES>
void dispatch_epi2(const GemmArgs& g, cudaStream_t s) {
    switch (g.epi) {
        case Epi::Store: dispatch_major2<BN, STAGES, 0>(g, s); break;
        case Epi::AccumF32: dispatch_major2<BN, STAGES, 1>(g, s); break;
        case Epi::AddRes: dispatch_major2<BN, STAGES, 2>(g, s); break;
        case Epi::StoreF32: dispatch_major2<BN, STAGES, 3>(g, s); break;
        case Epi::StoreGelu: dispatch_major2<BN, STAGES, 4>(g, s); break;
        case Epi::GeluBwd: dispatch_major2<BN, STAGES, 5>(g, s); break;
        case Epi::RopeScatter:
            EPP_REQUIRE(g.a_kmajor && g.b_kmajor && g.rope, "RopeScatter: K-major operands and rope args");
            launch_tc2<BN, STAGES, false, false, 6>(g, s);
            break;
        case Epi::SwiGlu:
            launch_tc2<BN, STAGES, false, false, 7>(g, s);
            break;
        case Epi::SwiGluBwd:
            dispatch_major2<BN, STAGES, 8>(g, s);
            break;
    }
}

// ---------------------------------------------------------------- SIMT f32
template <typename T>
__global__ void __launch_bounds__(256) gemm_simt_kernel(GemmArgs g) {
    pdl_wait();
    pdl_trigger();
    constexpr int TM = 64, TN = 64, TK = 16;
    __shared__ float As[TK][TM + 1];
    __shared__ float Bs[TK][TN + 1];
    const T* A = static_cast<const T*>(g.A);
    const T* B = static_cast<const T*>(g.B);
    const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < g.K; k0 += TK) {
        for (int i = threadIdx.x; i < TK * TM; i += 256) {
            const int kk = g.a_kmajor ? i % TK : i / TM;
            const int mm = g.a_kmajor ? i / TK : i % TM;
            const int m = m0 + mm, k = k0 + kk;
            float v = 0.f;
            if (m < g.M && k < g.K)
                v = to_f(g.a_kmajor ? A[static_cast<long long>(m) * g.lda + k]
                                    : A[static_cast<long long>(k) * g.lda + m]);
            As[kk][mm] = v;
        }
        for (int i = threadIdx.x; i < TK * TN; i += 256) {
            const int kk = g.b_kmajor ? i % TK : i / TN;
            const int nn = g.b_kmajor ? i / TK : i % TN;
            const int n = n0 + nn, k = k0 + kk;
            float v = 0.f;
            if (n < g.N && k < g.K)
                v = to_f(g.b_kmajor ? B[static_cast<long long>(n) * g.ldb + k]
                                    : B[static_cast<long long>(k) * g.ldb + n]);
            Bs[kk][nn] = v;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < TK; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = m0 + ty + 16 * i;
        if (m >= g.M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + tx + 16 * j;
            if (n >= g.N) continue;
            const long long off = static_cast<long long>(m) * g.ldc + n;
            float v = acc[i][j];
            if (g.epi == Epi::AccumF32) {
                static_cast<float*>(g.C)[off] += v;
            } else if (g.epi == Epi::StoreF32) {
                static_cast<float*>(g.C)[off] = v;
            } else {
                if (g.epi == Epi::AddRes)
                    v += to_f(static_cast<const T*>(g.R)[static_cast<long long>(m) * g.ldr + n]);
                if (g.epi == Epi::GeluBwd) {
                    const float rv = to_f(static_cast<const T*>(g.R)[static_cast<long long>(m) * g.ldr + n]);
                    v *= gelu_tanh_grad_f(rv);
                    if (g.C2) static_cast<T*>(g.C2)[static_cast<long long>(m) * g.ldc2 + n] = from_f<T>(gelu_tanh_f(rv));
                }
                if (g.epi == Epi::StoreGelu)
                    static_cast<T*>(g.C2)[static_cast<long long>(m) * g.ldc2 + n] = from_f<T>(gelu_tanh_f(v));
                static_cast<T*>(g.C)[off] = from_f<T>(v);
            }
        }
    }
}

}  // namespace

bool gemm_swiglu_fusable(const GemmArgs& g) {
    if (g.dtype != DType::BF16 || g.K <= 0 || g.M <= 0 || !g.C2) return false;
    const long long mt = ceil_div(g.M, 2 * kBM);
    if (g.epi == Epi::SwiGlu)   // gate / up tiles must not straddle the F boundary
        return g.a_kmajor && g.b_kmajor && g.N % 256 == 0 && mt * (g.N / 256) >= 60;
    if (g.epi == Epi::SwiGluBwd)
        return g.a_kmajor && g.R && g.N % 32 == 0 && g.ldc >= 2LL * g.N && mt * ceil_div(g.N, 256) >= 60;
    return false;
}

void gemm(const GemmArgs& g, cudaStream_t s) {
    EPP_REQUIRE(g.M >= 0 && g.N >= 0 && g.K >= 0, "gemm: negative extent");
    if (g.M == 0 || g.N == 0) return;
    ProfScope prof(kProfGemm, 2.0 * g.M * g.N * g.K, s);
    ProfScope prof_epi(kProfGemmEpi0 + static_cast<int>(g.epi), 2.0 * g.M * g.N * g.K, s);
    if (g.dtype == DType::F32) {
        dim3 grid(ceil_div(g.N, 64), ceil_div(g.M, 64));
        launch_k(gemm_simt_kernel<float>, grid, 256, 0, s, g);
        EPP_CHECK_LAUNCH();
        g_gemm_launches.fetch_add(1);
        return;
    }
    EPP_REQUIRE(g.N % 32 == 0, "gemm(bf16): N must be a multiple of 32");
    EPP_REQUIRE(g.lda % 8 == 0 && g.ldb % 8 == 0, "gemm(bf16): lda/ldb must be multiples of 8");
    EPP_REQUIRE(g.ldc % 8 == 0, "gemm(bf16): ldc must be a multiple of 8");
    EPP_REQUIRE((reinterpret_cast<uintptr_t>(g.A) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(g.B) & 15) == 0,
                "gemm(bf16): operands must be 16-byte aligned");
    EPP_REQUIRE((reinterpret_cast<uintptr_t>(g.C) & 15) == 0, "gemm(bf16): C must be 16-byte aligned");
    if (g.K == 0) {
        // Empty reduction: Store/StoreF32 write zeros, AddRes copies R, AccumF32 no-op.
        if (g.epi == Epi::AccumF32) return;
    }
    // Wide tiles keep the tensor pipe fed (128x256 per MMA); narrow problems
    // use 128-wide tiles to expose more CTAs.
    if (g.epi == Epi::SwiGlu || g.epi == Epi::SwiGluBwd) {
        EPP_REQUIRE(gemm_swiglu_fusable(g), "gemm: SwiGlu epilogue on a problem the pair kernel does not take");
        dispatch_epi2<256, 6>(g, s);
        return;
    }
    const long long tiles256 = static_cast<long long>(ceil_div(g.N, 256)) * ceil_div(g.M, kBM);
    const long long pair_tiles = static_cast<long long>(ceil_div(g.N, 256)) * ceil_div(g.M, 2 * kBM);
    // A ragged last column tile (N % 256 != 0, e.g. the LM head's V = 50304)
    // is fine: TMA zero-fills the B rows past N (the box still completes its
    // full byte count) and the epilogue stores only columns < N.
    if (g.K > 0 && pair_tiles >= 60)
        dispatch_epi2<256, 6>(g, s);      // CTA pairs: 256 x 256 tiles
    else if (tiles256 >= 120)
        dispatch_epi<256, 4>(g, s);
    else
        dispatch_epi<128, 6>(g, s);
}

}  // namespace eppk
