// epp-b200 GPU executor: host-side launch interface of every kernel family.
// All launches are stream-ordered; pointers are device pointers.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace eppk {

enum class DType : int { F32 = 0, BF16 = 1 };

inline size_t dtype_size(DType t) { return t == DType::F32 ? 4 : 2; }

// ---------------------------------------------------------------- GEMM ----
// C[M,N] = epilogue( sum_k A(m,k) * B(n,k) )
//   A(m,k) = a_kmajor ? A[m*lda + k] : A[k*lda + m]
//   B(n,k) = b_kmajor ? B[n*ldb + k] : B[k*ldb + n]
// Operand/output element type follows `dtype` (F32: all fp32; BF16: A/B bf16,
// fp32 accumulation, C bf16 for Store/AddRes, fp32 for AccumF32/StoreF32).
enum class Epi : int {
    Store = 0,      // C = acc
    AccumF32 = 1,   // C(fp32) += acc          (weight-gradient accumulation)
    AddRes = 2,     // C = acc + R             (residual stream update)
    StoreF32 = 3,   // C(fp32) = acc
    StoreGelu = 4,  // C = acc, C2 = gelu_tanh(acc)          (MLP up-projection)
    GeluBwd = 5,    // C = acc * gelu_tanh'(R) [, C2 = gelu_tanh(R)]  (MLP dgrad -> dh [+ act for dW2])
    RopeScatter = 6,  // QKV projection: RoPE on q/k, q -> [T,H,hd], k/v -> the segments' KV rows
    // SwiGLU (Llama MLP), CTA-pair kernel only (gemm_swiglu_fusable):
    SwiGlu = 7,       // up-projection, N = 2F (B = w13 = [gate; up], K-major): each tile pairs gate
                      // rows j..j+127 with up rows F+j..: C = h = [g | u] (ldc 2F), C2 = silu(g)*u
    SwiGluBwd = 8,    // dA = dY W2 (N = F): C = dh = [dA*u*silu'(g) | dA*silu(g)] (ldc 2F),
                      // R = h (ldr 2F), C2 = silu(g)*u (W2's weight-gradient operand)
};

struct AttnSeg;
// Destination of the fused QKV epilogue (Epi::RopeScatter), the same mapping
// as rope_qkv_scatter: token t of the chunk sits at position tok_pos[t] of
// segment tok_seg[t]; cs is the (cos, sin) table [pos][hd/2].
struct RopeScatterArgs {
    void* q_out = nullptr;
    const AttnSeg* segs = nullptr;
    const int* tok_seg = nullptr;
    const int* tok_pos = nullptr;
    const float2* cs = nullptr;
    int H = 0, Hkv = 0, hd = 0, layer = 0;
};

struct GemmArgs {
    int M = 0, N = 0, K = 0;
    const void* A = nullptr; long long lda = 0; bool a_kmajor = true;
    const void* B = nullptr; long long ldb = 0; bool b_kmajor = true;
    void* C = nullptr; long long ldc = 0;
    const void* R = nullptr; long long ldr = 0;
    void* C2 = nullptr; long long ldc2 = 0;
    const RopeScatterArgs* rope = nullptr;   // Epi::RopeScatter
    Epi epi = Epi::Store;
    DType dtype = DType::BF16;
    // Deferred dependency wait (tcgen05 kernels): the caller guarantees this
    // GEMM neither reads nor writes anything the PREVIOUS kernel in the stream
    // touches (e.g. a weight gradient behind an independent data gradient).
    // The kernel then skips its programmatic-launch wait at entry and waits
    // only before exiting, so its CTAs take the SMs the previous GEMM's last
    // wave leaves idle; its completion still implies the previous kernel's.
    bool defer_wait = false;
};

void gemm(const GemmArgs& a, cudaStream_t s);
// True when gemm() runs `a` on the CTA-pair kernel and the SwiGlu /
// SwiGluBwd epilogues apply (the caller otherwise runs the separate pass).
bool gemm_swiglu_fusable(const GemmArgs& a);
// Number of GEMM kernel launches issued so far on this process (bench counter).
long long gemm_launch_count();

// ----------------------------------------------------------- attention ----
// Segment of a chunk's token layout.  Queries are rows [q_start, q_start+q_len)
// of the chunk; they sit at key positions [kv_ctx, kv_ctx+q_len) of the
// segment's key/value rows, which live at k/v (+ layer * kv_layer_stride),
// row stride Hkv*hd elements.  Key j is visible to query i iff j <= kv_ctx+i.
struct AttnSeg {
    int q_start;
    int q_len;
    int kv_ctx;
    int tma_map;     // tcgen05 kernels: 0 -> AttnMaps::kv[0..1] (sequence), 1 -> kv[2..3]
    int kv_row0;     // row of key 0 in that map's row coordinate
    int dkv_accum;   // 1: dK/dV accumulate into a persistent (sequence) buffer;
                     // 2: first writer of that buffer (tcgen05: the tail slice);
                     // 0: chunk-local scratch, written once (tcgen05 backward)
    const void* k;       // layer-0 base
    const void* v;
    float* dk;           // fp32 gradient accumulators (backward), may be null in fwd
    float* dv;
    long long kv_layer_stride;    // elements between layers
    long long dkv_layer_stride;
};

// TMA descriptors of one attention call (tcgen05 kernels).  Q/dO: 3-D
// {hd, H, T}; K/V: 4-D {hd, Hkv, rows, layers}, two buffer families (a
// sequence's KV buffer and the chunk-local one).  All bf16, 128-byte swizzle,
// boxes of 64 hd-columns x 1 head x {64,128} rows.
struct AttnMaps {
    CUtensorMap q128, q64, q32;      // Q with 128- / 64- / 32-row boxes
    CUtensorMap do128, do64, do32;   // dO
    CUtensorMap kv128[4];        // k0, v0, k1, v1 with 128-row boxes
    CUtensorMap kv64[4];         // ... 64-row boxes
};
// Helpers filling AttnMaps (attention_tc.cu).
void attn_maps_q(AttnMaps& m, const void* q, const void* dout, int T, int H, int hd);
// rows: the map's row extent (reads past it return zeros); stride_rows: the
// buffer's rows per layer (0 = rows)
void attn_maps_kv(AttnMaps& m, int which, const void* k, const void* v, long long rows, int layers, int Hkv,
                  int hd, long long stride_rows = 0);
CUtensorMap make_tma_map(const void* base, int rank, const unsigned long long* dims,
                         const unsigned long long* strides_b, const unsigned* box);

// Work item (segment index, 64-row block index).
struct AttnWork {
    int seg;
    int block;
};
constexpr int kAttnBlock = 64;

struct AttnArgs {
    const AttnSeg* segs = nullptr;   // device array
    int nseg = 0;
    const AttnWork* qwork = nullptr;   // query blocks (fwd, dq)
    int nqwork = 0;
    const AttnWork* kwork = nullptr;   // key blocks (dk/dv)
    int nkwork = 0;
    const AttnWork* qwork128 = nullptr;   // 128-row query blocks (tcgen05 kernels)
    int nqwork128 = 0;
    const AttnWork* kwork128 = nullptr;   // 128-key blocks (tcgen05 kernels)
    int nkwork128 = 0;
    const AttnWork* qwork256 = nullptr;   // 256-row query blocks (tcgen05 forward: 2 tiles / CTA)
    int nqwork256 = 0;
    const AttnWork* kwork256 = nullptr;   // 256-key blocks (CTA-pair dK/dV: 128 keys per CTA)
    int nkwork256 = 0;
    int hfast = 0;                        // launch order: grid (head, work) instead of (work, head)
    int T = 0;
    int H = 0, Hkv = 0, hd = 0;
    int layer = 0;
    float scale = 0.f;
    double pairs = 0;     // visible (query, key) pairs, for FLOP accounting
    DType dtype = DType::BF16;
    // forward
    const void* q = nullptr;   // [T, H, hd]
    void* o = nullptr;         // [T, H, hd]
    float* lse = nullptr;      // [H, T], log2 domain: max2 + log2(sum)
    // backward
    const void* dout = nullptr;   // [T, H, hd]
    float* delta = nullptr;       // [H, T] scratch
    float* dq = nullptr;          // [T, H, hd] fp32 (fully written by attn_bwd)
    // tcgen05 dQ kernel: when set, dQ is written instead as bf16 into the q
    // columns of dqkv [T, (H+2Hkv) hd] with RoPE undone (rope_cs = the
    // (cos, sin) table, tok_pos = each query's position); dq is then unused
    void* dqkv_out = nullptr;
    const int* tok_pos = nullptr;
    const float2* rope_cs = nullptr;
    const AttnMaps* maps = nullptr;   // host struct, required by the tcgen05 kernels
};

void attn_fwd(const AttnArgs& a, cudaStream_t s);
// tcgen05 kernels (attention_tc.cu): the bf16 implementation.
bool attn_fwd_tc_supported(const AttnArgs& a);
void attn_fwd_tc(const AttnArgs& a, cudaStream_t s);
bool attn_bwd_tc_supported(const AttnArgs& a);
void attn_delta(const AttnArgs& a, cudaStream_t s);   // delta = rowsum(dO * O)
void attn_bwd_tc_main(const AttnArgs& a, cudaStream_t s);
void attn_bwd(const AttnArgs& a, cudaStream_t s);

// ------------------------------------------------------- elementwise ------
void embed_fwd(DType t, const int32_t* ids, const void* table, void* out, int T, int D,
               cudaStream_t s);
void embed_bwd(DType t, const int32_t* ids, const void* dout, float* dtable, int T, int D,
               cudaStream_t s);
// LayerNorm (has_bias, rms=false) or RMSNorm (rms=true): y = norm(x)*w (+b)
void norm_fwd(DType t, bool rms, const void* x, const void* w, const void* b, void* y,
              float* mean, float* rstd, int T, int D, float eps, cudaStream_t s);
// dx = dres + norm_bwd(dy);  dw/db accumulated (fp32) via per-block partials.
// xn_out (optional): also re-create y = norm(x)*w (+bias) from the saved stats
// in the same pass over x (the weight-gradient GEMM's operand).
void norm_bwd(DType t, bool rms, const void* x, const void* w, const void* dy,
              const float* mean, const float* rstd, const void* dres, void* dx, float* dw,
              float* db, int T, int D, cudaStream_t s, const void* bias = nullptr, void* xn_out = nullptr);
// Recompute y = norm(x) from saved stats.
void norm_apply(DType t, bool rms, const void* x, const void* w, const void* b,
                const float* mean, const float* rstd, void* y, int T, int D, cudaStream_t s);

// Ensure the RoPE cos/sin table covers positions [0, max_pos).
void rope_reserve(int max_pos, int hd, float theta, cudaStream_t s);
// The (cos, sin) table for head_dim hd (after rope_reserve).
const float2* rope_table_ptr(int hd, float theta, cudaStream_t s);
// RoPE + scatter of a packed [T, (H+2Hkv)*hd] QKV row block: q -> q_out [T,H,hd],
// k/v -> each segment's key/value rows for `layer`.
void rope_qkv_scatter(DType t, const void* qkv, void* q_out, const AttnSeg* segs_dev, int nseg,
                      const int* tok_seg, const int* tok_pos, int T, int H, int Hkv, int hd,
                      int layer, float theta, cudaStream_t s);
// Inverse: dq (fp32 [T,H,hd]) and segment dk/dv (fp32) -> dqkv [T,(H+2Hkv)hd],
// un-rotating dq/dk.
void rope_qkv_gather_grad(DType t, const float* dq, const AttnSeg* segs_dev, const int* tok_seg,
                          const int* tok_pos, void* dqkv, int T, int H, int Hkv, int hd,
                          int layer, float theta, cudaStream_t s);

// act: 0 = GELU(tanh), 1 = SwiGLU (input [T,2F] gate|up -> [T,F])
void act_fwd(DType t, int act, const void* h, void* a, int T, int F, cudaStream_t s);
// dh from da; for SwiGLU dh is [T,2F].  Writes dh (may alias nothing).
void act_bwd(DType t, int act, const void* h, const void* da, void* dh, int T, int F,
             cudaStream_t s);

// Cross entropy over logits rows [T, V] (in place: logits -> dlogits * scale);
// row_loss[t] = CE of row t (0 where targets[t] < 0).
void cross_entropy(DType t, void* logits, const int32_t* targets, float* row_loss, int T, int V,
                   float grad_scale, cudaStream_t s);
// slot = (sum row_loss, #targets >= 0) in fp64 (fixed order); acc += slot.
void chunk_loss(const float* row_loss, const int32_t* targets, int T, double* slot, double* acc, cudaStream_t s);

void fill_zero(void* p, size_t bytes, cudaStream_t s);
void cast_f32_to(DType t, const float* src, void* dst, long long n, cudaStream_t s);
void add_inplace(DType t, void* y, const void* x, long long n, cudaStream_t s);
// One optimizer segment: arena elements [off, off + n) with Adam state at
// [mv, mv + n) of the (possibly ZeRO-sharded) state arenas; start4 = prefix
// of float4 groups over the segment list.
struct AdamSeg {
    long long off, n, mv;
    int decay, pad;
    long long start4;
};
// Multi-tensor AdamW over every segment in ONE launch: fp32 masters, working
// copy (bf16 or fp32) written, gradients of the segments zeroed.
void adamw_multi(const AdamSeg* segs, int nseg, long long total4, float* master, void* work, DType t, float* grad,
                 float* m, float* v, float lr, float b1, float b2, float eps, float wd, float bc1, float bc2,
                 cudaStream_t s);
// Deterministic normal(0, std) init from (seed, offset) counter-based hashing.
void init_normal(float* dst, long long n, float std, unsigned long long seed, cudaStream_t s);
void init_const(float* dst, long long n, float v, cudaStream_t s);

}  // namespace eppk
