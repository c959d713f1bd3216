// epp-b200: slice-causal flash attention on tcgen05 (sm_100a).
//
// Same segment semantics as attention.cu (query rows of a segment sit at key
// positions [C, C+len) of the segment's K/V rows; key j visible iff j <= pos),
// with every matmul on the 5th-gen tensor cores (tcgen05.mma, accumulators in
// TMEM, operands staged by TMA in the UMMA 128-byte-swizzled layout).  The
// forward runs two 128-row query tiles per CTA with one softmax warpgroup
// each (see attn_fwd_tc); the backward is split into a query-parallel dQ
// kernel and a key-parallel dK/dV kernel (see the backward section).
#include "common.cuh"
#include "kernels.h"
#include "profile.h"
#include "tc.cuh"

namespace eppk {

namespace {

constexpr int TQ = 128;            // query rows per CTA (= TMEM lanes)
constexpr int TK = 128;            // keys per tile
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleSlack = 8.f;   // log2 units: p <= 2^8 before a rescale

// MUFU.EX2 without the denormal fix-up sequence of exp2f (inputs are
// <= ~8 and results below 2^-126 flush to zero, which softmax tolerates).
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// TMA tile loads: a [ROWS x HD] tile = HD/64 boxes of 64 columns, each
// landing as ROWS x 128 B with the 128-byte swizzle (the UMMA K-major
// SWIZZLE_128B layout).  Q/dO maps are {hd, H, T}; K/V maps {hd, Hkv, rows, L}.
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%3, %4, %5}], [%2];" ::"r"(tc::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(tc::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void tma4(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2,
                                     int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(tc::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(tc::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
template <int HD, int ROWS>
__device__ __forceinline__ void load_q_tile(uint8_t* dst, const CUtensorMap* m, uint64_t* bar, int head, int row) {
#pragma unroll
    for (int c = 0; c < HD / 64; ++c) tma3(dst + c * ROWS * 128, m, bar, c * 64, head, row);
}
template <int HD, int ROWS>
__device__ __forceinline__ void load_kv_tile(uint8_t* dst, const CUtensorMap* m, uint64_t* bar, int head, int row,
                                             int layer) {
#pragma unroll
    for (int c = 0; c < HD / 64; ++c) tma4(dst + c * ROWS * 128, m, bar, c * 64, head, row, layer);
}

// Packed fp32x2 arithmetic (FFMA2 / FADD2 on sm_100: two lanes of work per
// issue slot).
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void f2unpack(uint64_t v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

// Share of exponentials (in eighths of the pairs) computed on the FMA pipe
// instead of MUFU.EX2; tuned with tools/attn_bench.py.
#ifndef EPP_DKV_PAIR
#define EPP_DKV_PAIR 0
#endif
#ifndef EPP_FWD_EMU
#define EPP_FWD_EMU 3
#endif
// Backward: the dQ kernel gains from 2/8 (+2-4 %, its softmax loads the XU
// pipe with the exponentials and the dS packing), the dK/dV kernel (bound by
// the shared-memory port of its SS score MMAs) loses 2 % with any.
#ifndef EPP_DQ_EMU
#define EPP_DQ_EMU 2
#endif
#ifndef EPP_DKV_EMU
#define EPP_DKV_EMU 0
#endif
constexpr int kEmuFwd = EPP_FWD_EMU, kEmuDq = EPP_DQ_EMU, kEmuDkv = EPP_DKV_EMU;
template <int E>
__device__ __forceinline__ constexpr bool emu_pair(int q) {   // q: pair index within a 32-column chunk
    return (q & 7) >= 8 - E;
}

// 2^x for a pair on the FMA pipe (Cody-Waite split + degree-3 minimax, rel.
// err 7.5e-5, far below the bf16 rounding of P): offloads part of the
// exponentials from the MUFU unit, which 128-wide softmax rows saturate.
__device__ __forceinline__ void ex2_fma2(uint64_t x, float& p0, float& p1) {
    float x0, x1;
    f2unpack(x, x0, x1);
    x = f2pack(fmaxf(x0, -126.f), fmaxf(x1, -126.f));
    const uint64_t magic = f2pack(12582912.f, 12582912.f);     // 1.5 * 2^23: round to integer
    const uint64_t t = fadd2(x, magic);
    const uint64_t f = fsub2(x, fsub2(t, magic));              // f in [-0.5, 0.5]
    uint64_t p = ffma2(f2pack(0.05517025f, 0.05517025f), f, f2pack(0.2426079f, 0.2426079f));
    p = ffma2(p, f, f2pack(0.6932609f, 0.6932609f));
    p = ffma2(p, f, f2pack(0.9999283f, 0.9999283f));
    float t0, t1, q0, q1;
    f2unpack(t, t0, t1);
    f2unpack(p, q0, q1);
    p0 = __int_as_float(__float_as_int(t0) * (1 << 23) + __float_as_int(q0));
    p1 = __int_as_float(__float_as_int(t1) * (1 << 23) + __float_as_int(q1));
}

// bf16 pair (a in the low half) for a tcgen05 operand, F2FP.BF16.PACK_AB.
// (Packing on the integer pipes instead, IADD + PRMT with round half away
// from zero, measured 2-3 % slower in every attention kernel.)
__device__ __forceinline__ uint32_t pack_bf2(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ float max3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

// Row maximum of a 128-wide score row (FMNMX3, 4 independent chains).
__device__ __forceinline__ float row_max(const float (&sv)[TK / 32][32]) {
    float m[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        m[c] = sv[c][0];
#pragma unroll
        for (int i = 1; i < 31; i += 2) m[c] = max3(m[c], sv[c][i], sv[c][i + 1]);
        m[c] = fmaxf(m[c], sv[c][31]);
    }
    return fmaxf(fmaxf(m[0], m[1]), fmaxf(m[2], m[3]));
}

// P = 2^(s*c2 - mu) -> bf16 pairs written over the first 64 columns of the
// row's S buffer in TMEM (the A operand of the PV MMA); returns the fp32 row
// sum.  One pair in four takes the FMA-pipe exp2.
__device__ __forceinline__ float exp_pack_tmem(const float (&sv)[TK / 32][32], float c2, float mu, uint32_t taddr) {
    const uint64_t c2x = f2pack(c2, c2), nmu = f2pack(-mu, -mu);
    uint64_t l4[4] = {0, 0, 0, 0};
#pragma unroll
    for (int c = 0; c < TK / 32; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
            const uint64_t x = ffma2(f2pack(sv[c][i], sv[c][i + 1]), c2x, nmu);
            float p0, p1;
            if (emu_pair<kEmuFwd>(i >> 1)) {
                ex2_fma2(x, p0, p1);
            } else {
                float x0, x1;
                f2unpack(x, x0, x1);
                p0 = ex2(x0);
                p1 = ex2(x1);
            }
            l4[(i >> 1) & 3] = fadd2(l4[(i >> 1) & 3], f2pack(p0, p1));
            pk[i >> 1] = pack_bf2(p0, p1);
        }
        tc::tmem_st16u(taddr + c * 16, pk);
    }
    tc::tmem_wait_st();
    const uint64_t s2 = fadd2(fadd2(l4[0], l4[1]), fadd2(l4[2], l4[3]));
    float a, b;
    f2unpack(s2, a, b);
    return a + b;
}

// Launch order.  The block scheduler dispatches in linear block order and
// the work lists are sorted longest-first.  Large launches run head-major
// (grid (work, head)): a wave covers one or two heads, whose K/V (16 MB per
// head at 32K) then stays in L2.  Launches of a few waves run head-fastest
// (grid (head, work)), so every head's most expensive item starts in the
// first wave instead of forming the tail.  The kernels read the order from
// AttnArgs::hfast, set by the launcher.
constexpr int kAttnFewWaves = 4 * 148;
inline bool attn_hfast(int heads, int nwork) { return static_cast<long long>(heads) * nwork <= kAttnFewWaves; }
inline dim3 attn_grid(int heads, int nwork) {
    return attn_hfast(heads, nwork) ? dim3(heads, nwork) : dim3(nwork, heads);
}
#define EPP_WORK_INDEX (a.hfast ? blockIdx.y : blockIdx.x)
#define EPP_HEAD_INDEX (a.hfast ? blockIdx.x : blockIdx.y)

// Forward: one CTA = 256 query rows (two 128-row tiles Q0, Q1) of one head,
// so each K/V tile fetched into shared memory feeds two score MMAs and two PV
// MMAs, and the two softmax warpgroups ping-pong on the tensor core:
//   tensor queue  ... PV0(j) S0(j+1) PV1(j) S1(j+1) PV0(j+1) ...
// while softmax group 0 works on S0(j+1) the tensor core runs PV1(j) and
// S1(j+1), and vice versa.  S_i(j+1) is issued after PV_i(j), so the commit
// that publishes S_i(j+1) also proves that PV_i(j) has finished reading P_i
// and updating O_i: no separate "PV done" barrier is needed.
// TMEM columns: S0 [0,128) S1 [128,256) O0 [256,256+HD) O1 [384,384+HD);
// P_i (bf16 pairs) overwrites the first 64 columns of S_i and feeds the PV
// MMA straight from TMEM (A operand), so P costs no shared memory traffic.
// Shared memory: Q0, Q1 and a 4-slot ring holding K(0) V(0) K(1) V(1) ...
// (a slot is released by the commit after its last reader).
// Warps 0-3 softmax Q0, 4-7 softmax Q1, 8 MMA, 9 TMA, 10-11 idle: three
// whole warpgroups, so setmaxnreg can move registers from the issue
// warpgroup (56) to the softmax warpgroups (224; a row of S is 128 fp32).
constexpr int kThreadsFwd = 384;
constexpr int kFwdSlots = 4;

template <int HD>
struct FwdSmem {
    static constexpr int kTile = TQ * HD * 2;       // one 128-row Q / K / V tile
    static constexpr int kQ = 0;                     // Q0, Q1
    static constexpr int kRing = kQ + 2 * kTile;
    static constexpr int kBar = kRing + kFwdSlots * kTile;
    static constexpr int kBytes = kBar + 16 * 8 + 16;
    static constexpr int kAlloc = kBytes + 1024;
};

template <int HD>
__global__ void __launch_bounds__(kThreadsFwd, 1) attn_fwd_tc(const AttnArgs a,
                                                              const __grid_constant__ AttnMaps mp) {
    pdl_wait();
    pdl_trigger();
    using L = FwdSmem<HD>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    // 32-bit shared-window address of the same (aligned) base: computed from
    // the symbol directly so descriptor math stays on the uniform datapath
    const uint32_t sbase = (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) + 1023u) & ~1023u;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kBar);
    uint64_t* q_full = bar + 0;
    uint64_t* full = bar + 1;                 // [kFwdSlots]
    uint64_t* empty = full + kFwdSlots;       // [kFwdSlots]
    uint64_t* s_full = empty + kFwdSlots;     // [2]
    uint64_t* p_full = s_full + 2;            // [2]
    uint64_t* o_full = p_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 1);

    const AttnWork w = a.qwork256[EPP_WORK_INDEX];
    const AttnSeg sg = a.segs[w.seg];
    const int h = EPP_HEAD_INDEX;
    const int kvh = h / (a.H / a.Hkv);
    // warp index broadcast from lane 0: the compiler then knows it is warp-uniform
    // and keeps the role branches and the MMA warp's loop state on the uniform
    // datapath (no R2UR before every tcgen05.mma)
    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    const int q0 = w.block * 2 * TQ;
    const int rows0 = min(TQ, sg.q_len - q0);
    const int rows1 = max(0, min(TQ, sg.q_len - q0 - TQ));
    const int nkb0 = (sg.kv_ctx + q0 + rows0 + TK - 1) / TK;
    const int nkb1 = rows1 > 0 ? (sg.kv_ctx + q0 + TQ + rows1 + TK - 1) / TK : 0;
    const int nkb = max(nkb0, nkb1);

    if (threadIdx.x == 0) {
        tc::mbar_init(q_full, 1);
        for (int s = 0; s < kFwdSlots; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&s_full[i], 1);
            tc::mbar_init(&p_full[i], TQ);
        }
        tc::mbar_init(o_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 8) tc::tmem_alloc(tmem_slot, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp >= 8) tc::setmaxnreg_dec<56>();
    if (warp == 9) {
        // --------------------------------------------------------- TMA loads
        if (lane == 0) {
            const CUtensorMap* mk = &mp.kv128[2 * sg.tma_map];
            const CUtensorMap* mv = &mp.kv128[2 * sg.tma_map + 1];
            tc::mbar_expect_tx(q_full, (rows1 > 0 ? 2 : 1) * L::kTile);
            load_q_tile<HD, TQ>(smem + L::kQ, &mp.q128, q_full, h, sg.q_start + q0);
            if (rows1 > 0) load_q_tile<HD, TQ>(smem + L::kQ + L::kTile, &mp.q128, q_full, h, sg.q_start + q0 + TQ);
            for (int t = 0; t < 2 * nkb; ++t) {     // t = 2j: K(j), t = 2j+1: V(j)
                const int s = t % kFwdSlots;
                tc::mbar_wait(&empty[s], ((t / kFwdSlots) & 1) ^ 1);
                tc::mbar_expect_tx(&full[s], L::kTile);
                load_kv_tile<HD, TK>(smem + L::kRing + s * L::kTile, (t & 1) ? mv : mk, &full[s], kvh,
                                     sg.kv_row0 + (t >> 1) * TK, a.layer);
            }
        }
        __syncwarp();
    } else if (warp == 8) {
        // This CTA holds all 512 TMEM columns (one CTA per SM), so the
        // allocation starts at lane 0, column 0: a compile-time base keeps the
        // MMA operands in uniform registers.
        if (tmem != 0) __trap();
        constexpr uint32_t tmem_u = 0;
        // ------------------------------------------------------- MMA issuer
        constexpr uint32_t idS = tc::instr_desc_mn(TQ, TK, false, false);
        constexpr uint32_t idO = tc::instr_desc_mn(TQ, HD, false, true);
        auto slot_addr = [&](int t) { return (sbase + L::kRing + (t % kFwdSlots) * L::kTile); };
        auto wait_full = [&](int t) {
            tc::mbar_wait(&full[t % kFwdSlots], (t / kFwdSlots) & 1);
            tc::fence_after();
        };
        auto issue_s = [&](int i, int j) {       // S_i = Q_i K(j)^T
            const uint32_t sQ = (sbase + L::kQ + i * L::kTile);
            const uint32_t sK = slot_addr(2 * j);
            const uint64_t dq = tc::smem_desc(sQ, 16, 1024), dk = tc::smem_desc(sK, 16, 1024);
#pragma unroll
            for (int cb = 0; cb < HD / 64; ++cb)   // 64-column blocks: +16 KB; K16 steps: +32 B
                tc::mma4_ss<2, 2>(tmem_u + i * TK, dq + cb * 1024, dk + cb * 1024, idS, cb != 0);
            tc::commit_w(&s_full[i]);
        };
        auto issue_pv = [&](int i, int j) {      // O_i += P_i V(j)
            tc::mbar_wait(&p_full[i], j & 1);
            tc::fence_after();
            const uint32_t sV = slot_addr(2 * j + 1);
            // P from TMEM (bf16 pairs over S_i: 8 columns per K16 step); V: MN-major (+2 KB per K16 step)
            const uint64_t dv = tc::smem_desc(sV, 16384, 1024);
#pragma unroll
            for (int cb = 0; cb < TK / 64; ++cb)
                tc::mma4_ts<8, 128>(tmem_u + 256 + i * 128, tmem_u + i * TK + cb * 32, dv + cb * 512, idO,
                                    (j | cb) != 0);
        };
        tc::mbar_wait(q_full, 0);
        tc::fence_after();
        wait_full(0);
        issue_s(0, 0);
        if (nkb1 > 0) issue_s(1, 0);
        tc::commit_w(&empty[0]);
        for (int j = 0; j < nkb; ++j) {
            wait_full(2 * j + 1);
            if (j < nkb0) issue_pv(0, j);
            if (j + 1 < nkb) wait_full(2 * j + 2);
            if (j + 1 < nkb0) issue_s(0, j + 1);
            if (j < nkb1) issue_pv(1, j);
            tc::commit_w(&empty[(2 * j + 1) % kFwdSlots]);
            if (j + 1 < nkb1) issue_s(1, j + 1);
            if (j + 1 < nkb) tc::commit_w(&empty[(2 * j + 2) % kFwdSlots]);
        }
        tc::commit_w(o_full);
        __syncwarp();
    } else if (warp < 8) {
        // ---------------------------------------------------------- softmax
        tc::setmaxnreg_inc<224>();
        const int grp = warp >> 2;             // Q tile of this warpgroup
        const int r = threadIdx.x & 127;       // query row == TMEM lane
        const int rows = grp ? rows1 : rows0;
        const int my_nkb = grp ? nkb1 : nkb0;
        const int qt0 = q0 + grp * TQ;          // first query of the tile (segment-relative)
        const uint32_t lane_base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
        const uint32_t colS = grp * TK, colO = 256 + grp * 128;
        const int qp = (r < rows) ? sg.kv_ctx + qt0 + r : -1;
        const float c2 = a.scale * kLog2e;
        const int first_q = sg.kv_ctx + qt0;
        float m_run = -INFINITY, l = 0.f;
        for (int j = 0; j < my_nkb; ++j) {
            tc::mbar_wait(&s_full[grp], j & 1);
            tc::fence_after();
#ifdef EPP_FWD_MMA_ONLY   // pipeline experiment: no softmax work at all (wrong results)
            tc::fence_before();
            tc::mbar_arrive(&p_full[grp]);
            continue;
#endif
            const int key0 = j * TK;
            const bool need_mask = (key0 + TK - 1 > first_q) || rows < TQ;
            float sv[TK / 32][32];
#pragma unroll
            for (int c = 0; c < TK / 32; ++c) tc::tmem_ld32_async(lane_base + colS + c * 32, sv[c]);
            tc::tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < TK / 32; ++c) tc::reg_fence(sv[c]);
            // Causal / ragged tiles (at most two per query tile) mask in
            // place; interior tiles skip every compare and select.
            if (need_mask) {
#pragma unroll
                for (int c = 0; c < TK / 32; ++c) {
                    const int lim = qp - (key0 + c * 32);   // keys i <= lim visible
#pragma unroll
                    for (int i = 0; i < 32; ++i) sv[c][i] = i > lim ? -INFINITY : sv[c][i];
                }
            }
#ifdef EPP_FWD_FAKE_SOFTMAX   // pipeline-bound experiment: no max, no exp (wrong results)
            {
                uint32_t pk[16];
#pragma unroll
                for (int c = 0; c < TK / 32; ++c) {
#pragma unroll
                    for (int i = 0; i < 16; ++i) pk[i] = __float_as_uint(sv[c][2 * i]);
                    tc::tmem_st16u(lane_base + colS + c * 16, pk);
                }
                tc::tmem_wait_st();
                tc::fence_before();
                tc::mbar_arrive(&p_full[grp]);
                continue;
            }
#endif
            const float mraw = row_max(sv);
            const float mt = mraw * c2;
            const bool grow = mt > m_run + kRescaleSlack || (m_run == -INFINITY && mt > -INFINITY);
            // O_i is final through tile j-1 here (S_i(j) was issued after PV_i(j-1))
            if (__any_sync(0xffffffffu, grow) && j > 0) {
                const float alpha = grow ? ex2(m_run - mt) : 1.f;
#pragma unroll 1
                for (int c = 0; c < HD / 32; ++c) {
                    float o[32];
                    tc::tmem_ld32(lane_base + colO + c * 32, o);
#pragma unroll
                    for (int i = 0; i < 32; ++i) o[i] *= alpha;
                    tc::tmem_st32(lane_base + colO + c * 32, o);
                }
                if (grow) l *= alpha;
            }
            if (grow) m_run = mt;
            const float mu = (m_run == -INFINITY) ? 0.f : m_run;
            l += exp_pack_tmem(sv, c2, mu, lane_base + colS);
            tc::fence_before();
            tc::mbar_arrive(&p_full[grp]);
        }
        if (rows > 0) {
            tc::mbar_wait(o_full, 0);
            tc::fence_after();
            const float inv = l > 0.f ? 1.f / l : 0.f;
            bf16* orow = static_cast<bf16*>(a.o) + (static_cast<long long>(sg.q_start + qt0 + r) * a.H + h) * HD;
#pragma unroll 1
            for (int c = 0; c < HD / 32; ++c) {
                float o[32];
                tc::tmem_ld32(lane_base + colO + c * 32, o);
                if (r < rows) {
#pragma unroll
                    for (int i = 0; i < 32; i += 8) {
                        uint4 raw;
                        __nv_bfloat162* hh = reinterpret_cast<__nv_bfloat162*>(&raw);
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            hh[k] = __floats2bfloat162_rn(o[i + 2 * k] * inv, o[i + 2 * k + 1] * inv);
                        *reinterpret_cast<uint4*>(orow + c * 32 + i) = raw;
                    }
                }
            }
            if (r < rows)
                a.lse[static_cast<long long>(h) * a.T + sg.q_start + qt0 + r] =
                    l > 0.f ? m_run + log2f(l) : INFINITY;
        }
        tc::fence_before();
    }
    __syncthreads();
    if (warp == 8) {
        tc::fence_after();
        tc::tmem_dealloc(tmem, 512);
    }
}

template <int HD>
void launch_fwd_tc(const AttnArgs& a, cudaStream_t s) {
    using L = FwdSmem<HD>;
    static bool cfg = false;
    if (!cfg) {
        EPP_CUDA(cudaFuncSetAttribute(attn_fwd_tc<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kAlloc));
        cfg = true;
    }
    AttnArgs b = a;
    b.hfast = attn_hfast(a.H, a.nqwork256);
    launch_k(attn_fwd_tc<HD>, attn_grid(a.H, a.nqwork256), kThreadsFwd, L::kAlloc, s, b, *a.maps);
    EPP_CHECK_LAUNCH();
}

// ===========================================================================
// Backward.  Two kernels, no atomics, deterministic:
//   dq  (grid: 128-row query blocks x H), 64-key tiles, 4-stage K/V ring:
//        S = Q K^T, dP = dO V^T -> TMEM (double-buffered);
//        dS = P (dP - delta) -> TMEM over S (bf16), the A operand of
//        dQ += dS K -> TMEM; dQ * scale -> fp32 global.
//   dkv (grid: 128-key blocks x Hkv, GQA heads looped in the CTA), 64-row
//        query tiles, 3-stage Q/dO ring:
//        S^T = K Q^T, dP^T = V dO^T -> TMEM (double-buffered);
//        P^T, dS^T -> TMEM over S^T / dP^T (bf16), the A operands of
//        dV += P^T dO, dK += dS^T Q -> TMEM; then RMW into the fp32 dK/dV
//        accumulators of the segment (persist across a sequence's chunks).
// In both, the MMA warp issues the score MMAs of step i before the gradient
// MMAs of step i-1, and two softmax warpgroups take alternate steps (step i
// -> group i & 1, which owns TMEM buffer i & 1 and smem buffer i & 1), so
// one group's elementwise work overlaps the other's and the tensor core.
// The same swizzled [rows x hd] smem tile is a K-major operand in one MMA and
// (descriptor LBO = column-block stride, +2 KB per K16 step) an MN-major
// operand in another, so each tile is loaded once.
// ===========================================================================

// Warps 0-3 / 4-7 softmax groups, 8 MMA, 9 loads, 10-11 idle (whole
// warpgroups, for setmaxnreg).
constexpr int kThreadsBwd = 384;


__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

constexpr int TB = 64;    // secondary tile (keys in dq, queries in dkv)
constexpr int kDqStages = 7;    // K/V ring depth of the dq kernel
constexpr int kDkvStages = 4;   // Q/dO ring depth of the dk/dv kernel

// Two phases of dS for one 64-key tile of a query row, so the exponentials
// run while the dP MMA is still in flight: dq_p_tile turns the scores into
// P = 2^(s*c2 - lse) in place (MASK: keys k > lim are invisible, P = 0),
// dq_ds_tile forms dS = P * (dP - delta) as bf16 pairs.
template <bool MASK>
__device__ __forceinline__ void dq_p_tile(float (&s)[TB / 32][32], float c2, float lse, int lim0) {
    const uint64_t c2x = f2pack(c2, c2), nl = f2pack(-lse, -lse);
#pragma unroll
    for (int c = 0; c < TB / 32; ++c) {
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
            const uint64_t x = ffma2(f2pack(s[c][i], s[c][i + 1]), c2x, nl);
            float p0, p1;
            if (emu_pair<kEmuDq>(i >> 1)) {
                ex2_fma2(x, p0, p1);
            } else {
                float x0, x1;
                f2unpack(x, x0, x1);
                p0 = ex2(x0);
                p1 = ex2(x1);
            }
            if (MASK) {
                const int lim = lim0 - c * 32;
                p0 = i <= lim ? p0 : 0.f;
                p1 = i + 1 <= lim ? p1 : 0.f;
            }
            s[c][i] = p0;
            s[c][i + 1] = p1;
        }
    }
}
__device__ __forceinline__ void dq_ds_tile(const float (&p)[TB / 32][32], const float (&dp)[TB / 32][32],
                                           float dlt, uint32_t (&pk)[32]) {
    const uint64_t dl = f2pack(dlt, dlt);
#pragma unroll
    for (int c = 0; c < TB / 32; ++c) {
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
            float d0, d1;
            f2unpack(fmul2(f2pack(p[c][i], p[c][i + 1]), fsub2(f2pack(dp[c][i], dp[c][i + 1]), dl)), d0, d1);
            pk[c * 16 + (i >> 1)] = pack_bf2(d0, d1);
        }
    }
}

template <int HD>
struct DqSmem {
    static constexpr int kSmall = TB * HD * 2;      // K / V tiles
    static constexpr int kK = 0;                            // kDqStages stages
    static constexpr int kV = kK + kDqStages * kSmall;
    static constexpr int kDelta = kV + kDqStages * kSmall;  // [128] fp32 per-row delta
    static constexpr int kBar = kDelta + 128 * 4;
    static constexpr int kBytes = kBar + 24 * 8 + 16;
    static constexpr int kAlloc = kBytes + 1024;
};

template <int HD>
__global__ void __launch_bounds__(kThreadsBwd, 1) attn_bwd_dq_tc(const AttnArgs a,
                                                                 const __grid_constant__ AttnMaps mp) {
    pdl_wait();
    pdl_trigger();
    using L = DqSmem<HD>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    // 32-bit shared-window address of the same (aligned) base: computed from
    // the symbol directly so descriptor math stays on the uniform datapath
    const uint32_t sbase = (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) + 1023u) & ~1023u;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kBar);
    uint64_t* q_full = bar + 0;
    uint64_t* kv_full = bar + 1;                      // [kDqStages]
    uint64_t* kv_empty = kv_full + kDqStages;         // [kDqStages]
    uint64_t* s_full = kv_empty + kDqStages;          // [2]
    uint64_t* p_full = s_full + 2;                    // [2]
    uint64_t* acc_full = p_full + 2;                  // all MMAs retired (epilogue)
    uint64_t* d_full = acc_full + 1;                  // per-row delta in shared memory
    uint64_t* dp_full = d_full + 1;                   // [2] dP of the step (s_full: S)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dp_full + 2);

    const AttnWork w = a.qwork128[EPP_WORK_INDEX];
    const AttnSeg sg = a.segs[w.seg];
    const int h = EPP_HEAD_INDEX;
    const int kvh = h / (a.H / a.Hkv);
    // warp index broadcast from lane 0: the compiler then knows it is warp-uniform
    // and keeps the role branches and the MMA warp's loop state on the uniform
    // datapath (no R2UR before every tcgen05.mma)
    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    const int q0 = w.block * TQ;
    const int rows = min(TQ, sg.q_len - q0);
    const int kv_end = sg.kv_ctx + q0 + rows;
    const int nkb = (kv_end + TB - 1) / TB;
    const long long row0 = sg.q_start + q0;

    if (threadIdx.x == 0) {
        tc::mbar_init(q_full, 2 * TQ);      // both softmax groups stage Q / dO rows into TMEM
        tc::mbar_init(d_full, TQ);          // group 1 publishes delta
        for (int s = 0; s < kDqStages; ++s) {
            tc::mbar_init(&kv_full[s], 1);
            tc::mbar_init(&kv_empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&s_full[b], 1);
            tc::mbar_init(&dp_full[b], 1);
            tc::mbar_init(&p_full[b], TQ);
        }
        tc::mbar_init(acc_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 8) tc::tmem_alloc(tmem_slot, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;
    // TMEM: Q and dO (bf16 pairs, the A operands of the score MMAs: the
    // CTA's fixed operands cost no shared-memory bandwidth), S and dP
    // (double-buffered), the dQ accumulator.
    constexpr uint32_t kColQin = 0, kColOin = HD / 2, kColS = HD, kColP = HD + 2 * TB, kColQ = HD + 4 * TB;
    static_assert(HD + 4 * TB + HD <= 512, "TMEM budget");

    if (warp >= 8) tc::setmaxnreg_dec<56>();
    if (warp == 9) {
        if (lane == 0) {
            const CUtensorMap* mk = &mp.kv64[2 * sg.tma_map];
            const CUtensorMap* mv = &mp.kv64[2 * sg.tma_map + 1];
            for (int j = 0; j < nkb; ++j) {
                const int st = j % kDqStages;
                tc::mbar_wait(&kv_empty[st], ((j / kDqStages) & 1) ^ 1);
                tc::mbar_expect_tx(&kv_full[st], 2 * L::kSmall);
                const int row = sg.kv_row0 + j * TB;
                load_kv_tile<HD, TB>(smem + L::kK + st * L::kSmall, mk, &kv_full[st], kvh, row, a.layer);
                load_kv_tile<HD, TB>(smem + L::kV + st * L::kSmall, mv, &kv_full[st], kvh, row, a.layer);
            }
        }
        __syncwarp();
    } else if (warp == 8) {
        // This CTA holds all 512 TMEM columns (one CTA per SM), so the
        // allocation starts at lane 0, column 0: a compile-time base keeps the
        // MMA operands in uniform registers.
        if (tmem != 0) __trap();
        constexpr uint32_t tmem_u = 0;
        constexpr uint32_t idS = tc::instr_desc_mn(TQ, TB, false, false);
        constexpr uint32_t idQ = tc::instr_desc_mn(TQ, HD, false, true);
        // Buffer b of step j is rewritten by the scores of step j+2, issued
        // after grad(j) (which waited for the softmax of j): in-order tcgen05
        // execution orders every TMEM reuse, no extra barriers.
        auto grad = [&](int j) {   // dQ += dS(j) K(j), dS from TMEM (bf16 pairs over S buffer b)
            const int b = j & 1, st = j % kDqStages;
            tc::mbar_wait(&p_full[b], (j >> 1) & 1);
            tc::fence_after();
            const uint32_t sK = (sbase + L::kK + st * L::kSmall);
            static_assert(TB == 64, "one 4-step batch per dS tile");
            tc::mma4_ts<8, 128>(tmem_u + kColQ, tmem_u + kColS + b * TB, tc::smem_desc(sK, TB * 128, 1024), idQ,
                                j != 0);
            tc::commit_w(&kv_empty[st]);
        };
        auto scores = [&](int j) {   // S(j) = Q K(j)^T, dP(j) = dO V(j)^T
            const int b = j & 1, st = j % kDqStages;
            tc::mbar_wait(&kv_full[st], (j / kDqStages) & 1);
            tc::fence_after();
            const uint32_t sK = (sbase + L::kK + st * L::kSmall);
            const uint32_t sV = (sbase + L::kV + st * L::kSmall);
            const uint64_t dk = tc::smem_desc(sK, 16, 1024), dv = tc::smem_desc(sV, 16, 1024);
            // S first, committed on its own: the softmax group starts its
            // exponentials while dP is still on the tensor core
#pragma unroll
            for (int cb = 0; cb < HD / 64; ++cb)   // 64 hd per block: A +32 TMEM columns, B +8 KB
                tc::mma4_ts<8, 2>(tmem_u + kColS + b * TB, tmem_u + kColQin + cb * 32, dk + cb * 512, idS, cb != 0);
            tc::commit_w(&s_full[b]);
#pragma unroll
            for (int cb = 0; cb < HD / 64; ++cb)
                tc::mma4_ts<8, 2>(tmem_u + kColP + b * TB, tmem_u + kColOin + cb * 32, dv + cb * 512, idS, cb != 0);
            tc::commit_w(&dp_full[b]);
        };
        // one step of lookahead: the scores of step j+1 run on the
        // tensor core while the softmax group of step j works
        tc::mbar_wait(q_full, 0);
        tc::fence_after();
        scores(0);
        for (int j = 0; j < nkb; ++j) {
            if (j + 1 < nkb) scores(j + 1);
            grad(j);
        }
        tc::commit_w(acc_full);
        __syncwarp();
    } else if (warp < 8) {
        tc::setmaxnreg_inc<224>();
        const int grp = warp >> 2;
        const int r = threadIdx.x & 127;
        const uint32_t lane_base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
        const int qp = (r < rows) ? sg.kv_ctx + q0 + r : -1;
        const float c2 = a.scale * kLog2e;
        const int first_q = sg.kv_ctx + q0;
        const long long t = row0 + min(r, rows - 1);
        const float lse = a.lse[static_cast<long long>(h) * a.T + t];
        float* sDelta = reinterpret_cast<float*>(smem + L::kDelta);
        {   // stage this row of Q (group 0) / dO (group 1) into TMEM, release
            // the MMA warp, then group 1 forms delta = rowsum(dO * O) (the
            // separate delta pass of the other backends) off the MMA's
            // critical path, shares it through shared memory and writes it for
            // the dK/dV kernel that runs next
            const bf16* src = static_cast<const bf16*>(grp ? a.dout : a.q) + (t * a.H + h) * HD;
            uint4 keep[HD / 8];
#pragma unroll
            for (int c = 0; c < HD / 64; ++c) {
                uint32_t wv[32];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const uint4 u = *reinterpret_cast<const uint4*>(src + c * 64 + i * 8);
                    keep[c * 8 + i] = u;
                    wv[4 * i] = u.x;
                    wv[4 * i + 1] = u.y;
                    wv[4 * i + 2] = u.z;
                    wv[4 * i + 3] = u.w;
                }
                tc::tmem_st32u(lane_base + (grp ? kColOin : kColQin) + c * 32, wv);
            }
            tc::tmem_wait_st();
            tc::fence_before();
            tc::mbar_arrive(q_full);
            if (grp) {
                const bf16* orow = static_cast<const bf16*>(a.o) + (t * a.H + h) * HD;
                float dsum = 0.f;
#pragma unroll
                for (int i = 0; i < HD / 8; ++i) {
                    const uint4 ov = *reinterpret_cast<const uint4*>(orow + i * 8);
                    const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&keep[i]);
                    const __nv_bfloat162* o2 = reinterpret_cast<const __nv_bfloat162*>(&ov);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const float2 gf = __bfloat1622float2(g2[k]), of = __bfloat1622float2(o2[k]);
                        dsum = fmaf(gf.x, of.x, fmaf(gf.y, of.y, dsum));
                    }
                }
                sDelta[r] = dsum;
                if (r < rows) a.delta[static_cast<long long>(h) * a.T + row0 + r] = dsum;
                tc::mbar_arrive(d_full);
            }
        }
        tc::mbar_wait(d_full, 0);
        const float dlt = sDelta[r];
        for (int j = grp; j < nkb; j += 2) {
            const int b = grp;
            tc::mbar_wait(&s_full[b], (j >> 1) & 1);
            tc::fence_after();
#ifdef EPP_BWD_MMA_ONLY   // pipeline experiment: no softmax work at all (wrong results)
            tc::mbar_wait(&dp_full[b], (j >> 1) & 1);
            tc::fence_before();
            tc::mbar_arrive(&p_full[b]);
            continue;
#endif
            const int key0 = j * TB;
            const bool need_mask = (key0 + TB - 1 > first_q) || rows < TQ;
            uint32_t pk[32];
            float sall[TB / 32][32], pall[TB / 32][32];
#pragma unroll
            for (int c = 0; c < TB / 32; ++c) tc::tmem_ld32_async(lane_base + kColS + b * TB + c * 32, sall[c]);
            tc::tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < TB / 32; ++c) tc::reg_fence(sall[c]);
            if (need_mask) dq_p_tile<true>(sall, c2, lse, qp - key0);
            else dq_p_tile<false>(sall, c2, lse, 0);
            tc::mbar_wait(&dp_full[b], (j >> 1) & 1);
            tc::fence_after();
#pragma unroll
            for (int c = 0; c < TB / 32; ++c) tc::tmem_ld32_async(lane_base + kColP + b * TB + c * 32, pall[c]);
            tc::tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < TB / 32; ++c) tc::reg_fence(pall[c]);
            dq_ds_tile(sall, pall, dlt, pk);
            // dS (bf16 pairs) over the first 32 columns of S buffer b: the A
            // operand of the dQ MMA
            tc::tmem_st32u(lane_base + kColS + b * TB, pk);
            tc::tmem_wait_st();
            tc::fence_before();
            tc::mbar_arrive(&p_full[b]);
        }
        // (a group that skipped the last steps must not wait on a buffer
        // barrier whose earlier phases it never observed: parity would alias)
        tc::mbar_wait(acc_full, 0);
        tc::fence_after();
        if (a.dqkv_out) {
            // dQ straight into the q columns of dqkv (bf16) with RoPE undone:
            // group g takes the column pairs (d, d + HD/2) for d in chunk g
            constexpr int HALF = HD / 2;
            const long long t_out = row0 + r;
            const int pos = r < rows ? a.tok_pos[t_out] : 0;
            bf16* drow = static_cast<bf16*>(a.dqkv_out) + t_out * (a.H + 2 * a.Hkv) * HD + h * HD;
#pragma unroll 1
            for (int cc = grp * 32; cc < HALF; cc += 64) {
                float g1[32], g2[32];
                tc::tmem_ld32(lane_base + kColQ + cc, g1);
                tc::tmem_ld32(lane_base + kColQ + HALF + cc, g2);
                if (r < rows) {
                    const float4* c4 = reinterpret_cast<const float4*>(a.rope_cs + static_cast<long long>(pos) * HALF + cc);
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const float4 cs = c4[k];
                        const float x0 = g1[2 * k] * a.scale, y0 = g2[2 * k] * a.scale;
                        const float x1 = g1[2 * k + 1] * a.scale, y1 = g2[2 * k + 1] * a.scale;
                        g1[2 * k] = x0 * cs.x + y0 * cs.y;
                        g2[2 * k] = y0 * cs.x - x0 * cs.y;
                        g1[2 * k + 1] = x1 * cs.z + y1 * cs.w;
                        g2[2 * k + 1] = y1 * cs.z - x1 * cs.w;
                    }
#pragma unroll
                    for (int i = 0; i < 32; i += 8) {
                        uint4 ra, rb;
                        __nv_bfloat162* ha = reinterpret_cast<__nv_bfloat162*>(&ra);
                        __nv_bfloat162* hb = reinterpret_cast<__nv_bfloat162*>(&rb);
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            ha[j] = __floats2bfloat162_rn(g1[i + 2 * j], g1[i + 2 * j + 1]);
                            hb[j] = __floats2bfloat162_rn(g2[i + 2 * j], g2[i + 2 * j + 1]);
                        }
                        *reinterpret_cast<uint4*>(drow + cc + i) = ra;
                        *reinterpret_cast<uint4*>(drow + HALF + cc + i) = rb;
                    }
                }
            }
        } else {
            float* drow = a.dq + ((row0 + r) * a.H + h) * HD;
#pragma unroll 1
            for (int c = grp * (HD / 64); c < (grp + 1) * (HD / 64); ++c) {   // each group: half the columns
                float v[32];
                tc::tmem_ld32(lane_base + kColQ + c * 32, v);
                if (r < rows) {
#pragma unroll
                    for (int i = 0; i < 32; i += 4)
                        *reinterpret_cast<float4*>(drow + c * 32 + i) =
                            make_float4(v[i] * a.scale, v[i + 1] * a.scale, v[i + 2] * a.scale, v[i + 3] * a.scale);
                }
            }
        }
        tc::fence_before();
    }
    __syncthreads();
    if (warp == 8) {
        tc::fence_after();
        tc::tmem_dealloc(tmem, 512);
    }
}

// P^T and dS^T for one 64-query tile of a key row, in two phases (the
// exponentials run while the dP^T MMA is in flight).  The scores arrive with
// lse and delta already subtracted (augmented K-step, see attn_bwd_dkv_tc):
// P^T = 2^(S'^T c2) (in place, MASK: query qi is visible iff qmin <= qi <
// qmax), then dS^T = P^T * dP'^T.
template <bool MASK>
__device__ __forceinline__ void dkv_p_tile(float (&s)[TB / 32][32], float c2, int qmin, int qmax,
                                           uint32_t (&pk)[32]) {
    const uint64_t c2x = f2pack(c2, c2);
#pragma unroll
    for (int c = 0; c < TB / 32; ++c) {
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
            const uint64_t x = fmul2(f2pack(s[c][i], s[c][i + 1]), c2x);
            float p0, p1;
            if (emu_pair<kEmuDkv>(i >> 1)) {
                ex2_fma2(x, p0, p1);
            } else {
                float x0, x1;
                f2unpack(x, x0, x1);
                p0 = ex2(x0);
                p1 = ex2(x1);
            }
            if (MASK) {
                const int q = c * 32 + i;
                p0 = (q >= qmin && q < qmax) ? p0 : 0.f;
                p1 = (q + 1 >= qmin && q + 1 < qmax) ? p1 : 0.f;
            }
            s[c][i] = p0;
            s[c][i + 1] = p1;
            pk[c * 16 + (i >> 1)] = pack_bf2(p0, p1);
        }
    }
}
__device__ __forceinline__ void dkv_ds_tile(const float (&p)[TB / 32][32], const float (&dp)[TB / 32][32],
                                            uint32_t (&dk)[32]) {
#pragma unroll
    for (int c = 0; c < TB / 32; ++c) {
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
            float d0, d1;
            f2unpack(fmul2(f2pack(p[c][i], p[c][i + 1]), f2pack(dp[c][i], dp[c][i + 1])), d0, d1);
            dk[c * 16 + (i >> 1)] = pack_bf2(d0, d1);
        }
    }
}

// Augmented K-step operands (UMMA K-major, 32-byte swizzle: rows of 16 bf16,
// 8-row atoms of 256 B, 16-byte chunk c of row r stored at c ^ ((r >> 2) & 1)).
// Only columns 0-1 are ever non-zero.
__device__ __forceinline__ uint32_t aug_off(int row) {
    return static_cast<uint32_t>(row * 32 + ((((row >> 2) & 1)) << 4));
}
// hi + lo bf16 split of x (16 mantissa bits in the sum).
__device__ __forceinline__ uint32_t bf_hilo(float x) {
    const __nv_bfloat16 hi = __float2bfloat16_rn(x);
    const __nv_bfloat16 lo = __float2bfloat16_rn(x - __bfloat162float(hi));
    __nv_bfloat162 v;
    v.x = hi;
    v.y = lo;
    return *reinterpret_cast<uint32_t*>(&v);
}
// SWIZZLE_32B descriptor (layout type 6), SBO = one 8-row atom.
__device__ __forceinline__ uint64_t smem_desc_sw32(uint32_t addr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((addr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>(1) << 16;
    d |= static_cast<uint64_t>((256 >> 4) & 0x3FFFu) << 32;
    d |= 1ull << 46;
    d |= 6ull << 61;
    return d;
}

// dK/dV epilogue of the key-parallel kernels: softmax group 0 takes dK
// (scaled), group 1 dV, from the TMEM accumulators at colK / colV.
template <int HD>
__device__ __forceinline__ void dkv_epilogue(const AttnArgs& a, const AttnSeg& sg, int kvh, int k0, int nkeys,
                                             int r, int grp, uint32_t lane_base, uint32_t kColK, uint32_t kColV) {
    // group 0 adds dK (scaled), group 1 adds dV into the fp32 accumulators
    const long long kvs = static_cast<long long>(a.Hkv) * HD;
    float* base = grp == 0 ? sg.dk : sg.dv;
    float* drow = base + a.layer * sg.dkv_layer_stride + kvh * HD + (k0 + min(r, nkeys - 1)) * kvs;
    const float mul = grp == 0 ? a.scale : 1.f;
    const uint32_t col = grp == 0 ? kColK : kColV;
    if (a.dqkv_out != nullptr) {
        // Rows of this chunk's own tokens are complete here (later slices,
        // which also attend to them, ran their backward first): add the
        // accumulated fp32 partials, undo RoPE (dK) and write bf16 straight
        // into the k / v columns of dqkv.  Context rows (earlier slices)
        // keep accumulating in fp32.
        constexpr int HALF = HD / 2;
        const int kp = k0 + r;
        const bool valid = r < nkeys;
        const bool own = valid && kp >= sg.kv_ctx;
        const long long t_out = sg.q_start + (kp - sg.kv_ctx);
        bf16* orow = static_cast<bf16*>(a.dqkv_out) + t_out * (a.H + 2 * a.Hkv) * HD +
                     (grp == 0 ? a.H + kvh : a.H + a.Hkv + kvh) * HD;
#pragma unroll 1
        for (int cc = 0; cc < HALF; cc += 32) {
            float g1[32], g2[32];
            tc::tmem_ld32(lane_base + col + cc, g1);          // warp-collective: all lanes
            tc::tmem_ld32(lane_base + col + HALF + cc, g2);
            if (!valid) continue;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                g1[i] *= mul;
                g2[i] *= mul;
            }
            if (sg.dkv_accum == 1) {
#pragma unroll
                for (int i = 0; i < 32; i += 4) {
                    const float4 o1 = *reinterpret_cast<const float4*>(drow + cc + i);
                    const float4 o2 = *reinterpret_cast<const float4*>(drow + HALF + cc + i);
                    g1[i] += o1.x; g1[i + 1] += o1.y; g1[i + 2] += o1.z; g1[i + 3] += o1.w;
                    g2[i] += o2.x; g2[i + 1] += o2.y; g2[i + 2] += o2.z; g2[i + 3] += o2.w;
                }
            }
            if (!own) {
#pragma unroll
                for (int i = 0; i < 32; i += 4) {
                    *reinterpret_cast<float4*>(drow + cc + i) = make_float4(g1[i], g1[i + 1], g1[i + 2], g1[i + 3]);
                    *reinterpret_cast<float4*>(drow + HALF + cc + i) =
                        make_float4(g2[i], g2[i + 1], g2[i + 2], g2[i + 3]);
                }
                continue;
            }
            if (grp == 0) {   // dK: undo the rotation at position kp
                const float4* c4 = reinterpret_cast<const float4*>(a.rope_cs + static_cast<long long>(kp) * HALF + cc);
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const float4 cs = c4[k];
                    const float x0 = g1[2 * k], y0 = g2[2 * k], x1 = g1[2 * k + 1], y1 = g2[2 * k + 1];
                    g1[2 * k] = x0 * cs.x + y0 * cs.y;
                    g2[2 * k] = y0 * cs.x - x0 * cs.y;
                    g1[2 * k + 1] = x1 * cs.z + y1 * cs.w;
                    g2[2 * k + 1] = y1 * cs.z - x1 * cs.w;
                }
            }
#pragma unroll
            for (int i = 0; i < 32; i += 8) {
                uint4 ra, rb;
                __nv_bfloat162* ha = reinterpret_cast<__nv_bfloat162*>(&ra);
                __nv_bfloat162* hb = reinterpret_cast<__nv_bfloat162*>(&rb);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    ha[j] = __floats2bfloat162_rn(g1[i + 2 * j], g1[i + 2 * j + 1]);
                    hb[j] = __floats2bfloat162_rn(g2[i + 2 * j], g2[i + 2 * j + 1]);
                }
                *reinterpret_cast<uint4*>(orow + cc + i) = ra;
                *reinterpret_cast<uint4*>(orow + HALF + cc + i) = rb;
            }
        }
    } else {
#pragma unroll 1
        for (int c = 0; c < HD / 32; ++c) {
            float v[32];
            tc::tmem_ld32(lane_base + col + c * 32, v);    // warp-collective: all lanes
            if (r < nkeys) {
#pragma unroll
                for (int i = 0; i < 32; i += 4) {
                    float4 x = make_float4(v[i] * mul, v[i + 1] * mul, v[i + 2] * mul, v[i + 3] * mul);
                    if (sg.dkv_accum == 1) {   // later slices' contributions are already there
                        const float4 o = *reinterpret_cast<const float4*>(drow + c * 32 + i);
                        x.x += o.x; x.y += o.y; x.z += o.z; x.w += o.w;
                    }
                    *reinterpret_cast<float4*>(drow + c * 32 + i) = x;
                }
            }
        }
    }
}

template <int HD>
struct DkvSmem {
    static constexpr int kStages = kDkvStages;
    static constexpr int kBig = 128 * HD * 2;       // K / V tiles
    static constexpr int kSmall = TB * HD * 2;      // Q / dO tiles
    static constexpr int kK = 0;
    static constexpr int kV = kK + kBig;
    static constexpr int kQ = kV + kBig;                     // kStages stages
    static constexpr int kO = kQ + kStages * kSmall;
    static constexpr int kKa = kO + kStages * kSmall;        // augmented K-step: K, V [128 x 16] (ones)
    static constexpr int kVa = kKa + 128 * 32;
    static constexpr int kQa = kVa + 128 * 32;               // Q, dO [64 x 16] per stage (-lse/c2, -delta)
    static constexpr int kOa = kQa + kStages * TB * 32;
    static constexpr int kBar = kOa + kStages * TB * 32;
    static constexpr int kBytes = kBar + 24 * 8 + 16;
    static constexpr int kAlloc = kBytes + 1024;
};

template <int HD>
__global__ void __launch_bounds__(kThreadsBwd, 1) attn_bwd_dkv_tc(const AttnArgs a,
                                                                  const __grid_constant__ AttnMaps mp) {
    pdl_wait();
    pdl_trigger();
    using L = DkvSmem<HD>;
    constexpr int kDkvStages = L::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    // 32-bit shared-window address of the same (aligned) base: computed from
    // the symbol directly so descriptor math stays on the uniform datapath
    const uint32_t sbase = (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) + 1023u) & ~1023u;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kBar);
    uint64_t* kv_full = bar + 0;
    uint64_t* qd_full = bar + 1;                      // [kDkvStages]
    uint64_t* qd_empty = qd_full + kDkvStages;        // [kDkvStages]
    uint64_t* s_full = qd_empty + kDkvStages;         // [2]
    uint64_t* p_full = s_full + 2;                    // [2]
    uint64_t* acc_full = p_full + 2;                  // all MMAs retired (epilogue)
    uint64_t* dp_full = acc_full + 1;                 // [2] dP^T of the step (s_full: S^T)
    uint64_t* pt_full = dp_full + 2;                  // [2] P^T in TMEM (p_full: dS^T)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pt_full + 2);

    const AttnWork w = a.kwork128[EPP_WORK_INDEX];
    const AttnSeg sg = a.segs[w.seg];
    const int kvh = EPP_HEAD_INDEX;
    const int group = a.H / a.Hkv;
    // warp index broadcast from lane 0: the compiler then knows it is warp-uniform
    // and keeps the role branches and the MMA warp's loop state on the uniform
    // datapath (no R2UR before every tcgen05.mma)
    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    const int k0 = w.block * TK;
    const int kv_len = sg.kv_ctx + sg.q_len;
    const int nkeys = min(TK, kv_len - k0);
    const int qb_first = max(0, k0 - sg.kv_ctx) / TB;
    const int nqb = (sg.q_len + TB - 1) / TB;
    const int per_head = nqb - qb_first;
    const int iters = per_head * group;     // >= 1: the segment's last query sees every key

    if (threadIdx.x == 0) {
        tc::mbar_init(kv_full, 1);
        for (int st = 0; st < kDkvStages; ++st) {
            tc::mbar_init(&qd_full[st], 2);      // TMA expect_tx + the augmented-column writes
            tc::mbar_init(&qd_empty[st], 1);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&s_full[b], 1);
            tc::mbar_init(&p_full[b], TQ);
        }
        tc::mbar_init(acc_full, 1);
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&dp_full[b], 1);
            tc::mbar_init(&pt_full[b], TQ);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 8) tc::tmem_alloc(tmem_slot, 512);
    // Augmented K-step: S'^T = [K | 1 1] [Q | hi lo]^T = S^T - lse/c2 and
    // dP'^T = [V | 1 1] [dO | hi lo]^T = dP^T - delta, so the softmax needs no
    // per-query operands (they would cost 512 B of shared-memory reads per
    // thread and step).  Zero the augmented blocks; K/V get their ones here.
    for (int i = threadIdx.x; i < (L::kBar - L::kKa) / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(smem + L::kKa)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    if (threadIdx.x < 128) {
        *reinterpret_cast<uint32_t*>(smem + L::kKa + aug_off(threadIdx.x)) = 0x3F803F80u;   // bf16 (1, 1)
        *reinterpret_cast<uint32_t*>(smem + L::kVa + aug_off(threadIdx.x)) = 0x3F803F80u;
    }
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;
    constexpr uint32_t kColS = 0, kColP = 128, kColV = 256, kColK = 256 + HD;

    if (warp >= 8) tc::setmaxnreg_dec<56>();
    if (warp == 9) {
        const CUtensorMap* mk = &mp.kv128[2 * sg.tma_map];
        const CUtensorMap* mv = &mp.kv128[2 * sg.tma_map + 1];
        if (lane == 0) {
            tc::mbar_expect_tx(kv_full, 2 * L::kBig);
            load_kv_tile<HD, 128>(smem + L::kK, mk, kv_full, kvh, sg.kv_row0 + k0, a.layer);
            load_kv_tile<HD, 128>(smem + L::kV, mv, kv_full, kvh, sg.kv_row0 + k0, a.layer);
        }
        // augmented columns: -lse/c2 (hi, lo) for Q, -delta (hi, lo) for dO
        // (rows past the end: 0, they are masked).  The global reads of step
        // it+1 are issued before step it's stage is awaited (latency hidden).
        const float inv_c2 = 1.f / (a.scale * kLog2e);
        float lv[2], dv[2];
        auto fetch = [&](int it) {
            const int hq = kvh * group + it / per_head;
            const int q0 = (qb_first + it % per_head) * TB;
            const int rows = min(TB, sg.q_len - q0);
            const long long base = static_cast<long long>(hq) * a.T + sg.q_start + q0;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int i = lane + 32 * u;
                lv[u] = i < rows ? a.lse[base + i] : 0.f;
                dv[u] = i < rows ? a.delta[base + i] : 0.f;
            }
        };
        fetch(0);
        for (int it = 0; it < iters; ++it) {
            const int st = it % kDkvStages;
            const int hq = kvh * group + it / per_head;
            const int q0 = (qb_first + it % per_head) * TB;
            const long long row0 = sg.q_start + q0;
            uint32_t qa[2], oa[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                qa[u] = bf_hilo(-lv[u] * inv_c2);
                oa[u] = bf_hilo(-dv[u]);
            }
            if (it + 1 < iters) fetch(it + 1);
            tc::mbar_wait(&qd_empty[st], ((it / kDkvStages) & 1) ^ 1);
            if (lane == 0) {
                tc::mbar_expect_tx(&qd_full[st], 2 * L::kSmall);
                load_q_tile<HD, TB>(smem + L::kQ + st * L::kSmall, &mp.q64, &qd_full[st], hq, static_cast<int>(row0));
                load_q_tile<HD, TB>(smem + L::kO + st * L::kSmall, &mp.do64, &qd_full[st], hq, static_cast<int>(row0));
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int i = lane + 32 * u;
                *reinterpret_cast<uint32_t*>(smem + L::kQa + st * TB * 32 + aug_off(i)) = qa[u];
                *reinterpret_cast<uint32_t*>(smem + L::kOa + st * TB * 32 + aug_off(i)) = oa[u];
            }
            tc::fence_proxy_async();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&qd_full[st]);
        }
    } else if (warp == 8) {
        // This CTA holds all 512 TMEM columns (one CTA per SM), so the
        // allocation starts at lane 0, column 0: a compile-time base keeps the
        // MMA operands in uniform registers.
        if (tmem != 0) __trap();
        constexpr uint32_t tmem_u = 0;
        constexpr uint32_t idS = tc::instr_desc_mn(TK, TB, false, false);
        constexpr uint32_t idD = tc::instr_desc_mn(TK, HD, false, true);
        const uint32_t sK = (sbase + L::kK);
        const uint32_t sV = (sbase + L::kV);
        const uint32_t sKa = (sbase + L::kKa);
        const uint32_t sVa = (sbase + L::kVa);
        const uint64_t dK = tc::smem_desc(sK, 16, 1024), dV = tc::smem_desc(sV, 16, 1024);
        constexpr uint32_t kColDs = kColP;
        auto grad = [&](int it) {   // dV += P^T dO ; dK += dS^T Q  (P^T, dS^T from TMEM)
            const int b = it & 1, st = it % kDkvStages;
            tc::mbar_wait(&pt_full[b], (it >> 1) & 1);   // P^T is published before dS^T
            tc::fence_after();
            const uint32_t sQ = (sbase + L::kQ + st * L::kSmall);
            const uint32_t sO = (sbase + L::kO + st * L::kSmall);
            tc::mma4_ts<8, 128>(tmem_u + kColV, tmem_u + kColS + b * TB, tc::smem_desc(sO, TB * 128, 1024), idD,
                                it != 0);
            tc::mbar_wait(&p_full[b], (it >> 1) & 1);
            tc::fence_after();
            tc::mma4_ts<8, 128>(tmem_u + kColK, tmem_u + kColDs + b * TB, tc::smem_desc(sQ, TB * 128, 1024), idD,
                                it != 0);
            tc::commit_w(&qd_empty[st]);
        };
        // Buffer b of step it is rewritten by the scores of step it+2,
        // issued after grad(it): in-order tcgen05 execution orders the
        // TMEM reuse, and grad(it) itself waited for the softmax of it.
        auto scores = [&](int it) {   // S^T = K Q^T, dP^T = V dO^T
            const int b = it & 1, st = it % kDkvStages;
            tc::mbar_wait(&qd_full[st], (it / kDkvStages) & 1);
            tc::fence_after();
            const uint32_t sQ = (sbase + L::kQ + st * L::kSmall);
            const uint32_t sO = (sbase + L::kO + st * L::kSmall);
            const uint64_t dq = tc::smem_desc(sQ, 16, 1024), dO = tc::smem_desc(sO, 16, 1024);
#pragma unroll
            for (int cb = 0; cb < HD / 64; ++cb)   // 64-column blocks: +16 KB (K, V), +8 KB (Q, dO)
                tc::mma4_ss<2, 2>(tmem_u + kColS + b * TB, dK + cb * 1024, dq + cb * 512, idS, cb != 0);
            tc::mma_bf16_w(tmem_u + kColS + b * TB, smem_desc_sw32(sKa),
                         smem_desc_sw32((sbase + L::kQa + st * TB * 32)), idS, 1);
            tc::commit_w(&s_full[b]);   // S^T on its own: the exponentials overlap the dP^T MMA
#pragma unroll
            for (int cb = 0; cb < HD / 64; ++cb)
                tc::mma4_ss<2, 2>(tmem_u + kColP + b * TB, dV + cb * 1024, dO + cb * 512, idS, cb != 0);
            tc::mma_bf16_w(tmem_u + kColP + b * TB, smem_desc_sw32(sVa),
                         smem_desc_sw32((sbase + L::kOa + st * TB * 32)), idS, 1);
            tc::commit_w(&dp_full[b]);
        };
        tc::mbar_wait(kv_full, 0);
        scores(0);
        for (int it = 0; it < iters; ++it) {
            if (it + 1 < iters) scores(it + 1);
            grad(it);
        }
        tc::commit_w(acc_full);
        __syncwarp();
    } else if (warp < 8) {
        tc::setmaxnreg_inc<224>();
        const int grp = warp >> 2;
        const int r = threadIdx.x & 127;      // key row == TMEM lane
        const uint32_t lane_base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
        const int kp = k0 + r;
        const float c2 = a.scale * kLog2e;
        for (int it = grp; it < iters; it += 2) {
            const int b = grp;
            const int q0 = (qb_first + it % per_head) * TB;
            const int rows = min(TB, sg.q_len - q0);
            const int first_q = sg.kv_ctx + q0;
            const bool need_mask = (k0 + TK - 1 > first_q) || rows < TB;
            tc::mbar_wait(&s_full[b], (it >> 1) & 1);
            tc::fence_after();
#ifdef EPP_BWD_MMA_ONLY
            tc::fence_before();
            tc::mbar_arrive(&pt_full[b]);
            tc::mbar_wait(&dp_full[b], (it >> 1) & 1);
            tc::fence_before();
            tc::mbar_arrive(&p_full[b]);
            continue;
#endif
            uint32_t pk[32], dk[32];
            float sall[TB / 32][32], dall[TB / 32][32];
#pragma unroll
            for (int c = 0; c < TB / 32; ++c) tc::tmem_ld32_async(lane_base + kColS + b * TB + c * 32, sall[c]);
            tc::tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < TB / 32; ++c) tc::reg_fence(sall[c]);
            // query qi visible to key kp iff kp - first_q <= qi < rows
            if (need_mask) dkv_p_tile<true>(sall, c2, kp - first_q, rows, pk);
            else dkv_p_tile<false>(sall, c2, 0, TB, pk);
            // P^T (bf16 pairs) over the first 32 columns of the S^T buffer: the
            // A operand of the dV MMA, published before dS^T exists
            tc::tmem_st32u(lane_base + kColS + b * TB, pk);
            tc::tmem_wait_st();
            tc::fence_before();
            tc::mbar_arrive(&pt_full[b]);
            tc::mbar_wait(&dp_full[b], (it >> 1) & 1);
            tc::fence_after();
#pragma unroll
            for (int c = 0; c < TB / 32; ++c) tc::tmem_ld32_async(lane_base + kColP + b * TB + c * 32, dall[c]);
            tc::tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < TB / 32; ++c) tc::reg_fence(dall[c]);
            dkv_ds_tile(sall, dall, dk);
            // dS^T (bf16 pairs) over the first 32 columns of the dP^T buffer:
            // the dK MMA's A operand
            tc::tmem_st32u(lane_base + kColP + b * TB, dk);
            tc::tmem_wait_st();
            tc::fence_before();
            tc::mbar_arrive(&p_full[b]);
        }
        tc::mbar_wait(acc_full, 0);
        tc::fence_after();
        dkv_epilogue<HD>(a, sg, kvh, k0, nkeys, r, grp, lane_base, kColK, kColV);
        tc::fence_before();
    }
    __syncthreads();
    if (warp == 8) {
        tc::fence_after();
        tc::tmem_dealloc(tmem, 512);
    }
}

// ---------------------------------------------------------------------------
// dK/dV on CTA pairs (cta_group::2, hd 128): two CTAs of a cluster take 256
// consecutive keys of a head (128 each, the M halves of M=256 MMAs issued by
// the leader CTA).  The score MMAs S^T = K Q^T / dP^T = V dO^T read their A
// operand (the CTA's K / V rows) from shared memory; at N=64 the single-CTA
// kernel's MMA reads 4 KB of A + 2 KB of B per K16 step, more than the
// tensor core's 128 B/clk shared-memory port (48 instead of 32 cycles per
// MMA, tools/micro/mma_issue_bench.cu).  Here each CTA supplies only half of
// B (its 32 query rows of Q / dO; its 64 hd columns of dO^T / Q^T for dV / dK),
// so a step reads 138 instead of 172 KB of shared memory per CTA.
// Per stage each CTA stages two views of the same Q (and dO) tile:
//   Qr: its 32 query rows x all hd   (S^T's B half: N = queries)
//   Qc: all 64 query rows x its 64 hd (dK's B half: N = hd, MN-major)
// Barriers live on the leader (rank 0) where the MMA warp waits: TMA loads
// of both CTAs complete on the leader's barriers (peer bit cleared), the
// softmax warps of both CTAs arrive there (peer: remote arrive), and MMA
// commits multicast to both CTAs.
//
// MEASURED (tools/attn_bench.py, same box, A/B): correct (all attention
// kernel tests pass) but SLOWER: 892-894 vs 1305 TFLOP/s at 16K causal, 809
// vs 1190 at 5.3K context, 352 vs 483 on packed documents.  Every step now
// waits on cross-CTA round trips (the peer's softmax arrives remotely at the
// leader's barriers, commits multicast back), and the leader's MMA waits for
// the slower of the two CTAs' softmax warps; the dependency chain, not the
// shared-memory port, decides this kernel's speed.  Kept as an experiment
// (build with -DEPP_DKV_PAIR=1, e.g. tools/ab_build.sh); the single-CTA
// kernel above is the product.
// ---------------------------------------------------------------------------
#if EPP_DKV_PAIR
__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma3_pair(uint32_t dst, const CUtensorMap* m, uint32_t leader_bar, int c0, int c1,
                                          int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(leader_bar), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void tma4_pair(uint32_t dst, const CUtensorMap* m, uint32_t leader_bar, int c0, int c1,
                                          int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(leader_bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
// arrive on the barrier at the same offset in the leader CTA (local when this is the leader)
__device__ __forceinline__ void arrive_leader(uint64_t* bar) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(tc::smem_u32(bar)));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
// expect_tx on this (the leader's) barrier for bytes that both CTAs' TMA loads deliver
__device__ __forceinline__ void commit_pair_w(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
            tc::smem_u32(bar)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
}
template <int A_STEP, int B_STEP>
__device__ __forceinline__ void mma4_ss_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
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
template <int A_COLS, int B_STEP>
__device__ __forceinline__ void mma4_ts_pair(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                             uint32_t acc0) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b32 a;\n\t.reg .b64 b;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "mov.b32 a, %1;\n\tmov.b64 b, %2;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a], b, %3, p;\n\t"
        "add.s32 a, a, %5;\n\tadd.s64 b, b, %6;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a], b, %3, 1;\n\t"
        "add.s32 a, a, %5;\n\tadd.s64 b, b, %6;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a], b, %3, 1;\n\t"
        "add.s32 a, a, %5;\n\tadd.s64 b, b, %6;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a], b, %3, 1;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc0), "n"(A_COLS), "n"(B_STEP)
        : "memory");
}
__device__ __forceinline__ void mma_ss_pair_w(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

struct Dkv2Smem {   // hd 128, per CTA
    static constexpr int HD = 128;
    static constexpr int kStages = 4;
    static constexpr int kBig = 128 * HD * 2;       // this CTA's K / V rows
    static constexpr int kView = 32 * HD * 2;       // Qr / Or: 32 rows x 128 hd  (= 64 rows x 64 hd for Qc / Oc)
    static constexpr int kStage = 4 * kView;        // Qr Qc Or Oc
    static constexpr int kK = 0;
    static constexpr int kV = kK + kBig;
    static constexpr int kRing = kV + kBig;
    static constexpr int kKa = kRing + kStages * kStage;     // augmented K-step: K, V [128 x 16] (ones)
    static constexpr int kVa = kKa + 128 * 32;
    static constexpr int kQa = kVa + 128 * 32;               // Q, dO [32 x 16] per stage (this CTA's queries)
    static constexpr int kOa = kQa + kStages * 32 * 32;
    static constexpr int kBar = kOa + kStages * 32 * 32;
    static constexpr int kBytes = kBar + 32 * 8 + 16;
    static constexpr int kAlloc = kBytes + 1024;
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsBwd, 1)
    attn_bwd_dkv_tc2(const AttnArgs a, const __grid_constant__ AttnMaps mp) {
    pdl_wait();
    pdl_trigger();
    using L = Dkv2Smem;
    constexpr int HD = L::HD, NS = L::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const uint32_t sbase = (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) + 1023u) & ~1023u;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kBar);
    uint64_t* kv_full = bar + 0;                      // leader: both CTAs' K / V
    uint64_t* qd_full = bar + 1;                      // [NS] leader: both CTAs' Q / dO views + aug columns
    uint64_t* qd_empty = qd_full + NS;                // [NS] each CTA (multicast commit)
    uint64_t* s_full = qd_empty + NS;                 // [2] each CTA (multicast commit)
    uint64_t* dp_full = s_full + 2;                   // [2] each CTA
    uint64_t* pt_full = dp_full + 2;                  // [2] leader: P^T of both CTAs in TMEM (8 warps)
    uint64_t* p_full = pt_full + 2;                   // [2] leader: dS^T of both CTAs (8 warps)
    uint64_t* acc_full = p_full + 2;                  // each CTA: all MMAs retired
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

    const uint32_t rank = cta_rank();
    const bool leader = rank == 0;
    const AttnWork w = a.kwork256[blockIdx.x >> 1];
    const AttnSeg sg = a.segs[w.seg];
    const int kvh = blockIdx.y;
    const int group = a.H / a.Hkv;
    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    const int kp0 = w.block * 2 * TK;                 // first key of the pair
    const int k0 = kp0 + static_cast<int>(rank) * TK; // this CTA's keys
    const int kv_len = sg.kv_ctx + sg.q_len;
    const int nkeys = min(TK, kv_len - k0);           // <= 0: the pair's second block is past the end
    const int qb_first = max(0, kp0 - sg.kv_ctx) / TB;
    const int nqb = (sg.q_len + TB - 1) / TB;
    const int per_head = nqb - qb_first;
    const int iters = per_head * group;

    if (threadIdx.x == 0) {
        tc::mbar_init(kv_full, 1);
        for (int st = 0; st < NS; ++st) {
            tc::mbar_init(&qd_full[st], 3);   // leader expect_tx + both CTAs' aug-column writes
            tc::mbar_init(&qd_empty[st], 1);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&s_full[b], 1);
            tc::mbar_init(&dp_full[b], 1);
            tc::mbar_init(&pt_full[b], 8);
            tc::mbar_init(&p_full[b], 8);
        }
        tc::mbar_init(acc_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 8) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(tmem_slot)),
                     "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    for (int i = threadIdx.x; i < (L::kBar - L::kKa) / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(smem + L::kKa)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    if (threadIdx.x < 128) {
        *reinterpret_cast<uint32_t*>(smem + L::kKa + aug_off(threadIdx.x)) = 0x3F803F80u;   // bf16 (1, 1)
        *reinterpret_cast<uint32_t*>(smem + L::kVa + aug_off(threadIdx.x)) = 0x3F803F80u;
    }
    tc::fence_proxy_async();
    tc::fence_before();
    cluster_sync();          // barrier inits, TMEM allocation and aug blocks visible to the pair
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;
    constexpr uint32_t kColS = 0, kColP = 128, kColV = 256, kColK = 256 + HD;

    if (warp >= 8) tc::setmaxnreg_dec<56>();
    if (warp == 9) {
        const uint32_t lead_kv = tc::smem_u32(kv_full) & 0xFEFFFFFFu;     // peer bit cleared
        const uint32_t lead_qd0 = tc::smem_u32(qd_full) & 0xFEFFFFFFu;
        if (lane == 0) {
            if (leader) tc::mbar_expect_tx(kv_full, 2 * 2 * L::kBig);
            const CUtensorMap* mk = &mp.kv128[2 * sg.tma_map];
            const CUtensorMap* mv = &mp.kv128[2 * sg.tma_map + 1];
#pragma unroll
            for (int c = 0; c < HD / 64; ++c) {
                tma4_pair(sbase + L::kK + c * 128 * 128, mk, lead_kv, c * 64, kvh, sg.kv_row0 + k0, a.layer);
                tma4_pair(sbase + L::kV + c * 128 * 128, mv, lead_kv, c * 64, kvh, sg.kv_row0 + k0, a.layer);
            }
        }
        // aug columns of this CTA's 32 queries of the tile: -lse/c2 (hi, lo), -delta (hi, lo)
        const float inv_c2 = 1.f / (a.scale * kLog2e);
        float lv = 0.f, dv = 0.f;
        auto fetch = [&](int it) {
            const int hq = kvh * group + it / per_head;
            const int q0 = (qb_first + it % per_head) * TB + 32 * static_cast<int>(rank);
            const long long base = static_cast<long long>(hq) * a.T + sg.q_start + q0;
            const bool ok = q0 + lane < sg.q_len;
            lv = ok ? a.lse[base + lane] : 0.f;
            dv = ok ? a.delta[base + lane] : 0.f;
        };
        fetch(0);
        for (int it = 0; it < iters; ++it) {
            const int st = it % NS;
            const int hq = kvh * group + it / per_head;
            const int row0 = sg.q_start + (qb_first + it % per_head) * TB;
            const uint32_t qa = bf_hilo(-lv * inv_c2), oa = bf_hilo(-dv);
            if (it + 1 < iters) fetch(it + 1);
            tc::mbar_wait(&qd_empty[st], ((it / NS) & 1) ^ 1);
            if (lane == 0) {
                if (leader) tc::mbar_expect_tx(&qd_full[st], 2 * L::kStage);
                const uint32_t sq = sbase + L::kRing + st * L::kStage;
                const uint32_t lb = lead_qd0 + st * 8;
                const int rr = row0 + 32 * static_cast<int>(rank);
                // Qr, Or: this CTA's 32 query rows, both 64-column hd blocks
                tma3_pair(sq, &mp.q32, lb, 0, hq, rr);
                tma3_pair(sq + 32 * 128, &mp.q32, lb, 64, hq, rr);
                tma3_pair(sq + 2 * L::kView, &mp.do32, lb, 0, hq, rr);
                tma3_pair(sq + 2 * L::kView + 32 * 128, &mp.do32, lb, 64, hq, rr);
                // Qc, Oc: all 64 query rows, this CTA's hd block
                tma3_pair(sq + L::kView, &mp.q64, lb, 64 * static_cast<int>(rank), hq, row0);
                tma3_pair(sq + 3 * L::kView, &mp.do64, lb, 64 * static_cast<int>(rank), hq, row0);
            }
            *reinterpret_cast<uint32_t*>(smem + L::kQa + st * 32 * 32 + aug_off(lane)) = qa;
            *reinterpret_cast<uint32_t*>(smem + L::kOa + st * 32 * 32 + aug_off(lane)) = oa;
            tc::fence_proxy_async();
            __syncwarp();
            if (lane == 0) arrive_leader(&qd_full[st]);
        }
    } else if (warp == 8) {
        if (tmem != 0) __trap();
        if (leader) {
            constexpr uint32_t tmem_u = 0;
            constexpr uint32_t idS = tc::instr_desc_mn(2 * TK, TB, false, false);   // M 256, N 64
            constexpr uint32_t idD = tc::instr_desc_mn(2 * TK, HD, false, true);    // M 256, N 128, B MN-major
            const uint64_t dK = tc::smem_desc(sbase + L::kK, 16, 1024), dV = tc::smem_desc(sbase + L::kV, 16, 1024);
            const uint32_t sKa = sbase + L::kKa, sVa = sbase + L::kVa;
            auto grad = [&](int it) {   // dV += P^T dO ; dK += dS^T Q
                const int b = it & 1, st = it % NS;
                const uint32_t sq = sbase + L::kRing + st * L::kStage;
                tc::mbar_wait(&pt_full[b], (it >> 1) & 1);
                tc::fence_after();
                mma4_ts_pair<8, 128>(tmem_u + kColV, tmem_u + kColS + b * TB,
                                     tc::smem_desc(sq + 3 * L::kView, TB * 128, 1024), idD, it != 0);
                tc::mbar_wait(&p_full[b], (it >> 1) & 1);
                tc::fence_after();
                mma4_ts_pair<8, 128>(tmem_u + kColK, tmem_u + kColP + b * TB,
                                     tc::smem_desc(sq + L::kView, TB * 128, 1024), idD, it != 0);
                commit_pair_w(&qd_empty[st]);
            };
            auto scores = [&](int it) {   // S^T = K Q^T, dP^T = V dO^T
                const int b = it & 1, st = it % NS;
                const uint32_t sq = sbase + L::kRing + st * L::kStage;
                tc::mbar_wait(&qd_full[st], (it / NS) & 1);
                tc::fence_after();
                const uint64_t dq = tc::smem_desc(sq, 16, 1024), dO = tc::smem_desc(sq + 2 * L::kView, 16, 1024);
#pragma unroll
                for (int cb = 0; cb < HD / 64; ++cb)   // 64-column blocks: A +16 KB, B (32 rows) +4 KB
                    mma4_ss_pair<2, 2>(tmem_u + kColS + b * TB, dK + cb * 1024, dq + cb * 256, idS, cb != 0);
                mma_ss_pair_w(tmem_u + kColS + b * TB, smem_desc_sw32(sKa),
                              smem_desc_sw32(sbase + L::kQa + st * 32 * 32), idS, 1);
                commit_pair_w(&s_full[b]);
#pragma unroll
                for (int cb = 0; cb < HD / 64; ++cb)
                    mma4_ss_pair<2, 2>(tmem_u + kColP + b * TB, dV + cb * 1024, dO + cb * 256, idS, cb != 0);
                mma_ss_pair_w(tmem_u + kColP + b * TB, smem_desc_sw32(sVa),
                              smem_desc_sw32(sbase + L::kOa + st * 32 * 32), idS, 1);
                commit_pair_w(&dp_full[b]);
            };
            tc::mbar_wait(kv_full, 0);
            tc::fence_after();
            scores(0);
            for (int it = 0; it < iters; ++it) {
                if (it + 1 < iters) scores(it + 1);
                grad(it);
            }
            commit_pair_w(acc_full);
        }
        __syncwarp();
    } else if (warp < 8) {
        tc::setmaxnreg_inc<224>();
        const int grp = warp >> 2;
        const int r = threadIdx.x & 127;      // key row == TMEM lane
        const uint32_t lane_base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
        const int kp = k0 + r;
        const float c2 = a.scale * kLog2e;
        for (int it = grp; it < iters; it += 2) {
            const int b = grp;
            const int q0 = (qb_first + it % per_head) * TB;
            const int rows = min(TB, sg.q_len - q0);
            const int first_q = sg.kv_ctx + q0;
            const bool need_mask = (k0 + TK - 1 > first_q) || rows < TB;
            tc::mbar_wait(&s_full[b], (it >> 1) & 1);
            tc::fence_after();
            uint32_t pk[32], dk[32];
            float sall[TB / 32][32], dall[TB / 32][32];
#pragma unroll
            for (int c = 0; c < TB / 32; ++c) tc::tmem_ld32_async(lane_base + kColS + b * TB + c * 32, sall[c]);
            tc::tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < TB / 32; ++c) tc::reg_fence(sall[c]);
            if (need_mask) dkv_p_tile<true>(sall, c2, kp - first_q, rows, pk);
            else dkv_p_tile<false>(sall, c2, 0, TB, pk);
            tc::tmem_st32u(lane_base + kColS + b * TB, pk);
            tc::tmem_wait_st();
            tc::fence_before();
            __syncwarp();
            if (lane == 0) arrive_leader(&pt_full[b]);
            tc::mbar_wait(&dp_full[b], (it >> 1) & 1);
            tc::fence_after();
#pragma unroll
            for (int c = 0; c < TB / 32; ++c) tc::tmem_ld32_async(lane_base + kColP + b * TB + c * 32, dall[c]);
            tc::tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < TB / 32; ++c) tc::reg_fence(dall[c]);
            dkv_ds_tile(sall, dall, dk);
            tc::tmem_st32u(lane_base + kColP + b * TB, dk);
            tc::tmem_wait_st();
            tc::fence_before();
            __syncwarp();
            if (lane == 0) arrive_leader(&p_full[b]);
        }
        tc::mbar_wait(acc_full, 0);
        tc::fence_after();
        if (nkeys > 0) dkv_epilogue<HD>(a, sg, kvh, k0, nkeys, r, grp, lane_base, kColK, kColV);
        tc::fence_before();
    }
    __syncthreads();
    cluster_sync();          // the leader's MMAs and the peer's arrivals are done on both sides
    if (warp == 8) {
        tc::fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    }
}
#endif  // EPP_DKV_PAIR

template <int HD>
void launch_bwd_tc(const AttnArgs& a, cudaStream_t s) {
    static bool cfg = false;
    if (!cfg) {
        EPP_CUDA(cudaFuncSetAttribute(attn_bwd_dq_tc<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      DqSmem<HD>::kAlloc));
        EPP_CUDA(cudaFuncSetAttribute(attn_bwd_dkv_tc<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      DkvSmem<HD>::kAlloc));
        cfg = true;
    }
    if (a.nqwork128 > 0) {
        ProfScope prof(kProfAttnBwdDq, 6.0 * a.H * a.hd * a.pairs, s);     // executed: 3 matmuls
        AttnArgs b = a;
        b.hfast = attn_hfast(a.H, a.nqwork128);
        launch_k(attn_bwd_dq_tc<HD>, attn_grid(a.H, a.nqwork128), kThreadsBwd, DqSmem<HD>::kAlloc, s, b, *a.maps);
        EPP_CHECK_LAUNCH();
    }
#if EPP_DKV_PAIR
    if (HD == 128 && a.nkwork256 > 0 && a.kwork256) {
        // CTA pairs: cluster (2 x 128 keys) per 256-key block, grid (2 x blocks, Hkv)
        ProfScope prof(kProfAttnBwdDkv, 8.0 * a.H * a.hd * a.pairs, s);    // executed: 4 matmuls
        static bool cfg2 = false;
        if (!cfg2) {
            EPP_CUDA(cudaFuncSetAttribute(attn_bwd_dkv_tc2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          Dkv2Smem::kAlloc));
            cfg2 = true;
        }
        launch_k(attn_bwd_dkv_tc2, dim3(2 * a.nkwork256, a.Hkv), kThreadsBwd, Dkv2Smem::kAlloc, s, a, *a.maps);
        EPP_CHECK_LAUNCH();
        return;
    }
#endif
    if (a.nkwork128 > 0) {
        ProfScope prof(kProfAttnBwdDkv, 8.0 * a.H * a.hd * a.pairs, s);    // executed: 4 matmuls
        AttnArgs b = a;
        b.hfast = attn_hfast(a.Hkv, a.nkwork128);
        launch_k(attn_bwd_dkv_tc<HD>, attn_grid(a.Hkv, a.nkwork128), kThreadsBwd, DkvSmem<HD>::kAlloc,
                                     s, b, *a.maps);
        EPP_CHECK_LAUNCH();
    }
}

}  // namespace

bool attn_fwd_tc_supported(const AttnArgs& a) {
    return a.dtype == DType::BF16 && (a.hd == 64 || a.hd == 128) && a.qwork256 != nullptr &&
           a.maps != nullptr;
}

bool attn_bwd_tc_supported(const AttnArgs& a) {
    return a.dtype == DType::BF16 && (a.hd == 64 || a.hd == 128) && a.qwork128 != nullptr &&
           a.kwork128 != nullptr && a.maps != nullptr;
}

// dq + dk/dv kernels; the dq kernel also forms delta = rowsum(dO * O) for the dk/dv kernel.
void attn_bwd_tc_main(const AttnArgs& a, cudaStream_t s) {
    if (a.hd == 64) launch_bwd_tc<64>(a, s);
    else launch_bwd_tc<128>(a, s);
}

void attn_fwd_tc(const AttnArgs& a, cudaStream_t s) {
    if (a.nqwork256 == 0) return;
    ProfScope prof(kProfAttnFwd, 4.0 * a.H * a.hd * a.pairs, s);
    if (a.hd == 64) launch_fwd_tc<64>(a, s);
    else launch_fwd_tc<128>(a, s);
}

void attn_maps_q(AttnMaps& m, const void* q, const void* dout, int T, int H, int hd) {
    const unsigned long long dims[3] = {static_cast<unsigned long long>(hd), static_cast<unsigned long long>(H),
                                        static_cast<unsigned long long>(T)};
    const unsigned long long st[2] = {static_cast<unsigned long long>(hd) * 2,
                                      static_cast<unsigned long long>(H) * hd * 2};
    const unsigned b128[3] = {64, 1, 128}, b64[3] = {64, 1, 64}, b32[3] = {64, 1, 32};
    if (q) {
        m.q128 = make_tma_map(q, 3, dims, st, b128);
        m.q64 = make_tma_map(q, 3, dims, st, b64);
        m.q32 = make_tma_map(q, 3, dims, st, b32);
    }
    if (dout) {
        m.do128 = make_tma_map(dout, 3, dims, st, b128);
        m.do64 = make_tma_map(dout, 3, dims, st, b64);
        m.do32 = make_tma_map(dout, 3, dims, st, b32);
    }
}

void attn_maps_kv(AttnMaps& m, int which, const void* k, const void* v, long long rows, int layers, int Hkv,
                  int hd, long long stride_rows) {
    if (!k || rows <= 0) return;
    if (stride_rows <= 0) stride_rows = rows;
    const unsigned long long dims[4] = {static_cast<unsigned long long>(hd), static_cast<unsigned long long>(Hkv),
                                        static_cast<unsigned long long>(rows),
                                        static_cast<unsigned long long>(layers)};
    const unsigned long long st[3] = {static_cast<unsigned long long>(hd) * 2,
                                      static_cast<unsigned long long>(Hkv) * hd * 2,
                                      static_cast<unsigned long long>(stride_rows) * Hkv * hd * 2};
    const unsigned b128[4] = {64, 1, 128, 1}, b64[4] = {64, 1, 64, 1};
    m.kv128[2 * which] = make_tma_map(k, 4, dims, st, b128);
    m.kv128[2 * which + 1] = make_tma_map(v, 4, dims, st, b128);
    m.kv64[2 * which] = make_tma_map(k, 4, dims, st, b64);
    m.kv64[2 * which + 1] = make_tma_map(v, 4, dims, st, b64);
}

}  // namespace eppk
