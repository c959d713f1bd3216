#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <vector>
int main() {
    cudaStream_t s; cudaStreamCreate(&s);
    cudaMemPool_t mp; cudaDeviceGetDefaultMemPool(&mp, 0);
    unsigned long long thr = ~0ull; cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr);
    size_t fr, tot; cudaMemGetInfo(&fr, &tot);
    void* big; cudaMallocAsync(&big, fr - (size_t)8e9, s); cudaFreeAsync(big, s); cudaStreamSynchronize(s);
    for (size_t sz : {size_t(4096), size_t(1) << 20, size_t(64) << 20, size_t(1) << 30}) {
        std::vector<void*> live;
        auto t0 = std::chrono::high_resolution_clock::now();
        const int n = 2000;
        for (int i = 0; i < n; ++i) {
            void* p; cudaMallocAsync(&p, sz, s); live.push_back(p);
            if (live.size() > 64) { cudaFreeAsync(live.front(), s); live.erase(live.begin()); }
        }
        for (void* p : live) cudaFreeAsync(p, s);
        auto t1 = std::chrono::high_resolution_clock::now();
        cudaStreamSynchronize(s);
        printf("size %zu: %.2f us per malloc+free (host)\n", sz, std::chrono::duration<double, std::micro>(t1 - t0).count() / n);
    }
    return 0;
}
