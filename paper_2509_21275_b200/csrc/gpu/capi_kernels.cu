// epp-b200: kernel-level C ABI (include/epp_gpu.h epp_kernel_*) used by the
// unit tests and micro-benchmarks to drive single kernels on raw pointers.
#include <string>
#include <vector>

#include "common.cuh"
#include "epp_gpu.h"
#include "kernels.h"

namespace eppk {
std::string& gpu_error_slot();
namespace {

template <typename F>
int kguard(F&& f) {
    gpu_error_slot().clear();
    try {
        f();
        return EPP_GPU_OK;
    } catch (const CudaError& e) {
        gpu_error_slot() = e.what();
        return EPP_GPU_ECUDA;
    } catch (const std::invalid_argument& e) {
        gpu_error_slot() = e.what();
        return EPP_GPU_EARG;
    } catch (const std::exception& e) {
        gpu_error_slot() = e.what();
        return EPP_GPU_EOTHER;
    }
}

// Build + upload segment table and work lists for a standalone attention call.
struct AttnTables {
    AttnMaps maps{};
    void* kcat = nullptr;      // all segments' K (then V) rows, concatenated (tcgen05 path)
    void* segs = nullptr;
    void* qw = nullptr;
    void* kw = nullptr;
    void* qw128 = nullptr;
    void* kw128 = nullptr;
    void* qw256 = nullptr;
    void* kw256 = nullptr;
    int nq = 0, nk = 0, nq128 = 0, nk128 = 0, nq256 = 0, nk256 = 0;
    cudaStream_t s;
    AttnTables(int nseg, const int32_t* q_start, const int32_t* q_len, const int32_t* kv_ctx,
               const void* const* k, const void* const* v, float* const* dk, float* const* dv,
               cudaStream_t st, int T = 0, int H = 0, int Hkv = 0, int hd = 0, int dtype = 0,
               const void* qptr = nullptr, const void* dout = nullptr)
        : s(st) {
        std::vector<AttnSeg> sg(nseg);
        long long total_rows = 0;
        for (int i = 0; i < nseg; ++i) total_rows += kv_ctx[i] + q_len[i];
        const bool tc = dtype == static_cast<int>(DType::BF16) && total_rows > 0;
        const size_t row_bytes = static_cast<size_t>(Hkv) * hd * 2;
        if (tc) {
            EPP_CUDA(cudaMalloc(&kcat, 2 * total_rows * row_bytes));
            EPP_CUDA(cudaMemset(kcat, 0, 2 * total_rows * row_bytes));
        }
        long long row = 0;
        std::vector<AttnWork> q, kk, q128, k128, q256, k256;
        for (int i = 0; i < nseg; ++i) {
            sg[i] = AttnSeg{};
            sg[i].dkv_accum = 1;   // kernel-level ABI: dK/dV accumulate into the caller's buffers
            sg[i].q_start = q_start[i];
            sg[i].q_len = q_len[i];
            sg[i].kv_ctx = kv_ctx[i];
            sg[i].k = k[i];
            sg[i].v = v[i];
            sg[i].dk = dk ? dk[i] : nullptr;
            sg[i].dv = dv ? dv[i] : nullptr;
            sg[i].tma_map = 1;
            sg[i].kv_row0 = static_cast<int>(row);
            if (tc) {
                const size_t n = static_cast<size_t>(kv_ctx[i] + q_len[i]) * row_bytes;
                EPP_CUDA(cudaMemcpy(static_cast<uint8_t*>(kcat) + row * row_bytes, k[i], n, cudaMemcpyDeviceToDevice));
                EPP_CUDA(cudaMemcpy(static_cast<uint8_t*>(kcat) + (total_rows + row) * row_bytes, v[i], n,
                                    cudaMemcpyDeviceToDevice));
            }
            row += kv_ctx[i] + q_len[i];
            for (int b = 0; b * kAttnBlock < q_len[i]; ++b) q.push_back({i, b});
            for (int b = 0; b * kAttnBlock < kv_ctx[i] + q_len[i]; ++b) kk.push_back({i, b});
            for (int b = 0; b * 128 < q_len[i]; ++b) q128.push_back({i, b});
            for (int b = 0; b * 128 < kv_ctx[i] + q_len[i]; ++b) k128.push_back({i, b});
            for (int b = 0; b * 256 < q_len[i]; ++b) q256.push_back({i, b});
            for (int b = 0; b * 256 < kv_ctx[i] + q_len[i]; ++b) k256.push_back({i, b});
        }
        nq128 = static_cast<int>(q128.size());
        nk128 = static_cast<int>(k128.size());
        EPP_CUDA(cudaMalloc(&qw128, sizeof(AttnWork) * (nq128 ? nq128 : 1)));
        EPP_CUDA(cudaMalloc(&kw128, sizeof(AttnWork) * (nk128 ? nk128 : 1)));
        EPP_CUDA(cudaMemcpy(qw128, q128.data(), sizeof(AttnWork) * nq128, cudaMemcpyHostToDevice));
        EPP_CUDA(cudaMemcpy(kw128, k128.data(), sizeof(AttnWork) * nk128, cudaMemcpyHostToDevice));
        nq256 = static_cast<int>(q256.size());
        EPP_CUDA(cudaMalloc(&qw256, sizeof(AttnWork) * (nq256 ? nq256 : 1)));
        EPP_CUDA(cudaMemcpy(qw256, q256.data(), sizeof(AttnWork) * nq256, cudaMemcpyHostToDevice));
        nk256 = static_cast<int>(k256.size());
        EPP_CUDA(cudaMalloc(&kw256, sizeof(AttnWork) * (nk256 ? nk256 : 1)));
        EPP_CUDA(cudaMemcpy(kw256, k256.data(), sizeof(AttnWork) * nk256, cudaMemcpyHostToDevice));
        if (tc) {
            attn_maps_kv(maps, 1, kcat, static_cast<uint8_t*>(kcat) + total_rows * row_bytes, total_rows, 1, Hkv, hd);
            attn_maps_q(maps, qptr, dout, T, H, hd);
        }
        nq = static_cast<int>(q.size());
        nk = static_cast<int>(kk.size());
        EPP_CUDA(cudaMalloc(&segs, sizeof(AttnSeg) * (nseg ? nseg : 1)));
        EPP_CUDA(cudaMalloc(&qw, sizeof(AttnWork) * (nq ? nq : 1)));
        EPP_CUDA(cudaMalloc(&kw, sizeof(AttnWork) * (nk ? nk : 1)));
        EPP_CUDA(cudaMemcpy(segs, sg.data(), sizeof(AttnSeg) * nseg, cudaMemcpyHostToDevice));
        EPP_CUDA(cudaMemcpy(qw, q.data(), sizeof(AttnWork) * nq, cudaMemcpyHostToDevice));
        EPP_CUDA(cudaMemcpy(kw, kk.data(), sizeof(AttnWork) * nk, cudaMemcpyHostToDevice));
    }
    ~AttnTables() {
        cudaStreamSynchronize(s);
        cudaFree(segs);
        cudaFree(qw);
        cudaFree(kw);
        cudaFree(qw128);
        cudaFree(kw128);
        cudaFree(qw256);
        cudaFree(kw256);
        if (kcat) cudaFree(kcat);
    }
};
}  // namespace
}  // namespace eppk

extern "C" {

int epp_kernel_gemm_ex(int32_t M, int32_t N, int32_t K, const void* A, int64_t lda, int32_t a_kmajor,
                       const void* B, int64_t ldb, int32_t b_kmajor, void* C, int64_t ldc,
                       const void* R, int64_t ldr, void* C2, int64_t ldc2, int32_t epi, int32_t dtype,
                       void* stream) {
    return eppk::kguard([&] {
        eppk::GemmArgs g;
        g.M = M; g.N = N; g.K = K;
        g.A = A; g.lda = lda; g.a_kmajor = a_kmajor != 0;
        g.B = B; g.ldb = ldb; g.b_kmajor = b_kmajor != 0;
        g.C = C; g.ldc = ldc; g.R = R; g.ldr = ldr;
        g.C2 = C2; g.ldc2 = ldc2;
        EPP_REQUIRE((epi >= 0 && epi <= 5) || epi == 7 || epi == 8, "bad epilogue");
        g.epi = static_cast<eppk::Epi>(epi);
        EPP_REQUIRE(g.epi != eppk::Epi::StoreGelu || C2 != nullptr, "StoreGelu needs C2");
        EPP_REQUIRE(g.epi != eppk::Epi::GeluBwd || R != nullptr, "GeluBwd needs R (the pre-activation)");
        EPP_REQUIRE(epi < 7 || eppk::gemm_swiglu_fusable(g), "SwiGlu epilogue: shape not taken by the pair kernel");
        g.dtype = static_cast<eppk::DType>(dtype);
        eppk::gemm(g, static_cast<cudaStream_t>(stream));
    });
}

int epp_kernel_gemm(int32_t M, int32_t N, int32_t K, const void* A, int64_t lda, int32_t a_kmajor,
                    const void* B, int64_t ldb, int32_t b_kmajor, void* C, int64_t ldc,
                    const void* R, int64_t ldr, int32_t epi, int32_t dtype, void* stream) {
    if (epi < 0 || epi > 3) {
        eppk::gpu_error_slot() = "epp: bad epilogue";
        return EPP_GPU_EARG;
    }
    return epp_kernel_gemm_ex(M, N, K, A, lda, a_kmajor, B, ldb, b_kmajor, C, ldc, R, ldr, nullptr, 0, epi,
                              dtype, stream);
}

int epp_kernel_attention_fwd(int32_t T, int32_t H, int32_t Hkv, int32_t hd, float scale, int32_t nseg,
                             const int32_t* q_start, const int32_t* q_len, const int32_t* kv_ctx,
                             const void* const* k, const void* const* v, const void* q, void* o,
                             float* lse, int32_t dtype, void* stream) {
    return eppk::kguard([&] {
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        eppk::AttnTables tb(nseg, q_start, q_len, kv_ctx, k, v, nullptr, nullptr, s, T, H, Hkv, hd, dtype, q, nullptr);
        eppk::AttnArgs a;
        a.segs = static_cast<const eppk::AttnSeg*>(tb.segs);
        a.nseg = nseg;
        a.qwork = static_cast<const eppk::AttnWork*>(tb.qw);
        a.nqwork = tb.nq;
        a.kwork = static_cast<const eppk::AttnWork*>(tb.kw);
        a.nkwork = tb.nk;
        a.qwork128 = static_cast<const eppk::AttnWork*>(tb.qw128);
        a.nqwork128 = tb.nq128;
        a.kwork128 = static_cast<const eppk::AttnWork*>(tb.kw128);
        a.nkwork128 = tb.nk128;
        a.qwork256 = static_cast<const eppk::AttnWork*>(tb.qw256);
        a.nqwork256 = tb.nq256;
        a.kwork256 = static_cast<const eppk::AttnWork*>(tb.kw256);
        a.nkwork256 = tb.nk256;
        a.T = T; a.H = H; a.Hkv = Hkv; a.hd = hd; a.layer = 0; a.scale = scale;
        a.dtype = static_cast<eppk::DType>(dtype);
        a.q = q; a.o = o; a.lse = lse;
        a.maps = tb.kcat ? &tb.maps : nullptr;
        for (int i = 0; i < nseg; ++i)
            a.pairs += static_cast<double>(q_len[i]) * kv_ctx[i] + 0.5 * static_cast<double>(q_len[i]) * (q_len[i] + 1);
        eppk::attn_fwd(a, s);
    });
}

int epp_kernel_attention_bwd(int32_t T, int32_t H, int32_t Hkv, int32_t hd, float scale, int32_t nseg,
                             const int32_t* q_start, const int32_t* q_len, const int32_t* kv_ctx,
                             const void* const* k, const void* const* v, float* const* dk,
                             float* const* dv, const void* q, const void* o, const float* lse,
                             const void* dout, float* dq, int32_t dtype, void* stream) {
    return eppk::kguard([&] {
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        eppk::AttnTables tb(nseg, q_start, q_len, kv_ctx, k, v, dk, dv, s, T, H, Hkv, hd, dtype, q, dout);
        float* delta = nullptr;
        EPP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&delta), sizeof(float) * H * (T ? T : 1), s));
        eppk::AttnArgs a;
        a.segs = static_cast<const eppk::AttnSeg*>(tb.segs);
        a.nseg = nseg;
        a.qwork = static_cast<const eppk::AttnWork*>(tb.qw);
        a.nqwork = tb.nq;
        a.kwork = static_cast<const eppk::AttnWork*>(tb.kw);
        a.nkwork = tb.nk;
        a.qwork128 = static_cast<const eppk::AttnWork*>(tb.qw128);
        a.nqwork128 = tb.nq128;
        a.kwork128 = static_cast<const eppk::AttnWork*>(tb.kw128);
        a.nkwork128 = tb.nk128;
        a.qwork256 = static_cast<const eppk::AttnWork*>(tb.qw256);
        a.nqwork256 = tb.nq256;
        a.kwork256 = static_cast<const eppk::AttnWork*>(tb.kw256);
        a.nkwork256 = tb.nk256;
        a.T = T; a.H = H; a.Hkv = Hkv; a.hd = hd; a.layer = 0; a.scale = scale;
        a.dtype = static_cast<eppk::DType>(dtype);
        a.q = q; a.o = const_cast<void*>(o); a.lse = const_cast<float*>(lse);
        a.dout = dout; a.delta = delta; a.dq = dq;
        a.maps = tb.kcat ? &tb.maps : nullptr;
        for (int i = 0; i < nseg; ++i)
            a.pairs += static_cast<double>(q_len[i]) * kv_ctx[i] + 0.5 * static_cast<double>(q_len[i]) * (q_len[i] + 1);
        eppk::attn_bwd(a, s);
        EPP_CUDA(cudaFreeAsync(delta, s));
    });
}

}  // extern "C"
