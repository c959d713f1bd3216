// epp-b200: opt-in per-launch timing of the dominant kernels (GEMM,
// attention) with CUDA events recorded on the launching stream, so bench.py
// can report achieved TFLOP/s of the kernel class live over its timed region.
#include <cxxabi.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
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
std::vector<Rec> g_recs;       // oldest first
size_t g_head = 0;             // first record not yet harvested
std::vector<cudaEvent_t> g_free;
struct Acc {
    double ms = 0, flops = 0;
    int64_t n = 0;
};
Acc g_acc[32];                 // harvested totals per class

// Fold completed records (oldest first) into the per-class totals and
// recycle their events, so a long timed region keeps a bounded event pool
// instead of creating two events per launch.
void harvest() {
    while (g_head < g_recs.size()) {
        const Rec& r = g_recs[g_head];
        if (cudaEventQuery(r.b) != cudaSuccess) break;
        float e = 0;
        if (cudaEventElapsedTime(&e, r.a, r.b) != cudaSuccess) break;
        Acc& a = g_acc[r.cls];
        a.ms += e;
        a.flops += r.flops;
        ++a.n;
        g_free.push_back(r.a);
        g_free.push_back(r.b);
        ++g_head;
    }
    if (g_head > 4096 && g_head * 2 > g_recs.size()) {
        g_recs.erase(g_recs.begin(), g_recs.begin() + static_cast<long>(g_head));
        g_head = 0;
    }
}

cudaEvent_t take() {
    if (g_free.empty()) harvest();
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
    if (cls < 0 || cls >= 32) return EPP_GPU_EARG;
    for (size_t i = eppk::g_head; i < eppk::g_recs.size(); ++i)
        if (cudaEventSynchronize(eppk::g_recs[i].b) != cudaSuccess) return EPP_GPU_ECUDA;
    eppk::harvest();
    const eppk::Acc a = eppk::g_acc[cls];
    if (reset) eppk::g_acc[cls] = eppk::Acc{};
    if (ms) *ms = a.ms;
    if (flops) *flops = a.flops;
    if (launches) *launches = a.n;
    return 0;
}
}

namespace eppk {
namespace {
std::mutex g_kmu;
std::unordered_map<const void*, long long> g_kcount;
std::vector<std::pair<std::string, long long>> g_kview;   // last epp_gpu_kernel_stats snapshot
}  // namespace

void note_launch(const void* kernel) {
    std::lock_guard<std::mutex> lk(g_kmu);
    ++g_kcount[kernel];
}
}  // namespace eppk

extern "C" int epp_gpu_kernel_stats(int32_t idx, const char** name, int64_t* count) {
    std::lock_guard<std::mutex> lk(eppk::g_kmu);
    if (idx == 0) {   // snapshot: demangled name -> launches, sorted by name
        std::map<std::string, long long> agg;
        for (const auto& kv : eppk::g_kcount) {
            const char* raw = nullptr;
            std::string nm = "?";
            if (cudaFuncGetName(&raw, kv.first) == cudaSuccess && raw) {
                int st = 0;
                char* dm = abi::__cxa_demangle(raw, nullptr, nullptr, &st);
                nm = (st == 0 && dm) ? dm : raw;
                std::free(dm);
            }
            agg[nm] += kv.second;
        }
        eppk::g_kview.assign(agg.begin(), agg.end());
    }
    if (idx < 0 || idx >= static_cast<int32_t>(eppk::g_kview.size())) return EPP_GPU_EARG;
    if (name) *name = eppk::g_kview[idx].first.c_str();
    if (count) *count = eppk::g_kview[idx].second;
    return EPP_GPU_OK;
}

namespace eppk {
bool pdl_enabled() {
    static const bool on = [] {
        const char* v = getenv("EPP_PDL");
        return !(v && v[0] == '0');
    }();
    return on;
}
}  // namespace eppk
