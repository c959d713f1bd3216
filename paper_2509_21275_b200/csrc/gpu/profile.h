// epp-b200: launch-scoped profiling of kernel classes (see profile.cu).
#pragma once
#include <cuda_runtime.h>

namespace eppk {
enum ProfClass {
    kProfGemm = 0, kProfAttnFwd = 1, kProfAttnBwd = 2, kProfAttnBwdDq = 3, kProfAttnBwdDkv = 4,
    kProfNormFwd = 5, kProfNormBwd = 6, kProfRope = 7, kProfAct = 8, kProfCe = 9, kProfAdam = 10,
    kProfEmbed = 11, kProfCopy = 12,
    kProfGemmEpi0 = 13,   // + Epi: per-epilogue GEMM sub-classes 13..21 (also counted in kProfGemm)
};
bool profiling();
// Records an event pair around the launches issued during its lifetime.
class ProfScope {
public:
    ProfScope(int cls, double flops, cudaStream_t s);
    ~ProfScope();
private:
    int cls_;
    double flops_;
    cudaStream_t s_;
    cudaEvent_t a_ = nullptr, b_ = nullptr;
};
}  // namespace eppk
