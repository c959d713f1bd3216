// TMEM read throughput probe: W warps (W/4 per TMEM lane quarter) each issue
// tcgen05.ld 32x32b.x32 (4 KB per warp-instruction) in a loop; reports bytes
// per SM clock.  nvcc -gencode arch=compute_100a,code=sm_100a -I../../paper_2509_21275_b200/csrc/gpu
#include <cstdio>
#include <cuda_runtime.h>
#include "tc.cuh"
using namespace eppk;

__global__ void probe(int iters, float* out, long long* clk, int loads_per_wait) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tc::tmem_alloc(&slot, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = slot;
    const uint32_t base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + (warp >> 2) * 64;
    float acc = 0.f;
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        float v[2][32];
        tc::tmem_ld32_async(base, v[0]);
        if (loads_per_wait > 1) tc::tmem_ld32_async(base + 32, v[1]);
        tc::tmem_wait_ld();
        tc::reg_fence(v[0]);
#pragma unroll
        for (int k = 0; k < 32; ++k) acc += v[0][k];
        if (loads_per_wait > 1) {
            tc::reg_fence(v[1]);
#pragma unroll
            for (int k = 0; k < 32; ++k) acc += v[1][k];
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

int main() {
    float* out;
    long long* clk;
    cudaMalloc(&out, 148 * 1024 * sizeof(float));
    cudaMalloc(&clk, 148 * sizeof(long long));
    for (int warps : {4, 8, 16}) {
        for (int lpw : {1, 2}) {
            const int iters = 20000;
            probe<<<148, warps * 32>>>(iters, out, clk, lpw);
            cudaDeviceSynchronize();
            long long c[148];
            cudaMemcpy(c, clk, sizeof(c), cudaMemcpyDeviceToHost);
            double bytes = double(iters) * warps * lpw * 4096.0;
            printf("warps %2d loads/wait %d: %.1f B/clk per SM (%lld clk)\n", warps, lpw, bytes / c[0], c[0]);
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
