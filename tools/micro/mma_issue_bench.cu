// tcgen05.mma issue/execution probe: one warp per CTA (one CTA per SM)
// issues K16 BF16 MMAs back to back (batches of 4, as the attention kernels
// do) on fixed TMEM / shared-memory operands, then commits and waits.
// Reports SM cycles per MMA for M=128 and N in {32, 64, 128, 256}, A from
// shared memory (SS) or TMEM (TS).  The execution floor is N/2 cycles
// (M=128: 128*N*16 MACs at 4096 MAC/clk); a larger figure is the issue cost.
//   nvcc -gencode arch=compute_100a,code=sm_100a -I../../paper_2509_21275_b200/csrc/gpu mma_issue_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "tc.cuh"
using namespace eppk;

template <int N, bool TS>
__global__ void probe(int iters, long long* clk) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t done;
    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
    if (warp == 0) tc::tmem_alloc(&slot, 512);
    if (threadIdx.x == 0) {
        tc::mbar_init(&done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t sb = tc::smem_u32(smem);
    constexpr uint32_t idesc = tc::instr_desc_mn(128, N, false, false);
    long long t0 = 0, t1 = 0;
    if (warp == 0) {
        const uint64_t ad = tc::smem_desc(sb, 16, 1024), bd = tc::smem_desc(sb + 32768, 16, 1024);
        t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            if (TS)
                tc::mma4_ts<8, 2>(0u, 384u, bd, idesc, i != 0);
            else
                tc::mma4_ss<2, 2>(0u, ad, bd, idesc, i != 0);
        }
        tc::commit_w(&done);
        tc::mbar_wait(&done, 0);
        t1 = clock64();
    }
    __syncthreads();
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(slot, 512);
}

template <int N, bool TS>
void run(long long* clk) {
    const int iters = 4096;
    cudaFuncSetAttribute(probe<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    probe<N, TS><<<148, 128, 160 * 1024>>>(iters, clk);
    probe<N, TS><<<148, 128, 160 * 1024>>>(iters, clk);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
    double s = 0;
    for (long long v : h) s += v;
    printf("N=%3d %s: %.1f cycles per MMA (floor %d)  %s\n", N, TS ? "TS" : "SS", s / 148 / (4.0 * iters), N / 2,
           cudaGetErrorString(e));
}

int main() {
    long long* clk;
    cudaMalloc(&clk, 148 * sizeof(long long));
    run<32, false>(clk);
    run<32, true>(clk);
    run<64, false>(clk);
    run<64, true>(clk);
    run<128, false>(clk);
    run<128, true>(clk);
    run<256, false>(clk);
    run<256, true>(clk);
    return 0;
}
