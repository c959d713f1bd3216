// epp-b200: opt-in per-launch timing of the dominant kernels (GEMM,
// attention) with CUDA events recorded on the launching stream, so bench.py
// can report achieved TFLOP/s of the kernel class live over its timed region.
#include <mutex>
#include <vector>

#include "common.cuh"
#include "epp_gpu.h"
#include "profile.h"

namespace eppk {
namespace {
struct Rec {
    cudaEvent_t a, b;
    double flops;
    int cls;
};
std::mutex g_mu;
bool g_on = false;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_free;

cudaEvent_t take() {
    if (!g_free.empty()) {
        cudaEvent_t e = g_free.back();
        g_free.pop_back();
        return e;
    }
    cudaEvent_t e;
    EPP_CUDA(cudaEventCreate(&e));
    return e;
}
}  // namespace

bool profiling() { return g_on; }

ProfScope::ProfScope(int cls, double flops, cudaStream_t s) : cls_(cls), flops_(flops), s_(s) {
    if (!g_on) return;
    std::lock_guard<std::mutex> lk(g_mu);
    a_ = take();
    b_ = take();
    EPP_CUDA(cudaEventRecord(a_, s_));
}

ProfScope::~ProfScope() {
    if (!a_) return;
    std::lock_guard<std::mutex> lk(g_mu);
    cudaEventRecord(b_, s_);
    g_recs.push_back({a_, b_, flops_, cls_});
}
}  // namespace eppk

extern "C" {
int epp_gpu_profile(int32_t enable) {
    std::lock_guard<std::mutex> lk(eppk::g_mu);
    eppk::g_on = enable != 0;
    return 0;
}

int epp_gpu_profile_read(int32_t cls, double* ms, double* flops, int64_t* launches, int32_t reset) {
    std::lock_guard<std::mutex> lk(eppk::g_mu);
    double t = 0, f = 0;
    int64_t n = 0;
    std::vector<eppk::Rec> keep;
    for (auto& r : eppk::g_recs) {
        if (r.cls != cls) {
            keep.push_back(r);
            continue;
        }
        float e = 0;
        if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&e, r.a, r.b) != cudaSuccess)
            return EPP_GPU_ECUDA;
        t += e;
        f += r.flops;
        ++n;
        if (reset) {
            eppk::g_free.push_back(r.a);
            eppk::g_free.push_back(r.b);
        } else {
            keep.push_back(r);
        }
    }
    eppk::g_recs.swap(keep);
    if (ms) *ms = t;
    if (flops) *flops = f;
    if (launches) *launches = n;
    return 0;
}
}
