// epp-b200 GPU executor: shared device helpers (sm_100a only).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <utility>

namespace eppk {

typedef __nv_bfloat16 bf16;

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define EPP_CUDA(call)                                                                   \
    do {                                                                                 \
        cudaError_t err_ = (call);                                                       \
        if (err_ != cudaSuccess)                                                         \
            throw ::eppk::CudaError(std::string(#call " failed: ") +                    \
                                    cudaGetErrorString(err_) + " at " __FILE__ ":" +     \
                                    std::to_string(__LINE__));                           \
    } while (0)

// Every kernel launch is followed by EPP_CHECK_LAUNCH(), which also feeds the
// process-wide launch counter reported by epp_gpu_kernel_launches().
long long& launch_counter();
#define EPP_CHECK_LAUNCH()                                                               \
    do {                                                                                 \
        EPP_CUDA(cudaGetLastError());                                                    \
        ++::eppk::launch_counter();                                                      \
    } while (0)

// Programmatic dependent launch.  Every kernel starts with pdl_wait() (the
// previous grid in the stream has completed and its writes are visible) and
// then pdl_trigger() (the next grid may be scheduled), and is launched with
// launch_k(), which sets programmatic stream serialisation: the next
// kernel's launch and CTA rasterisation overlap the tail of the current one
// instead of following its completion (~8 us per transition between the
// large tcgen05 kernels).  EPP_PDL=0 launches conventionally.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
bool pdl_enabled();
// Per-kernel launch counts of this library (epp_gpu_kernel_stats): which
// kernel variants a run actually executed.
void note_launch(const void* kernel);
template <typename... KArgs, typename... Args>
inline void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    EPP_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
    note_launch(reinterpret_cast<const void*>(kernel));
}

#define EPP_REQUIRE(cond, msg)                                                           \
    do {                                                                                 \
        if (!(cond)) throw std::invalid_argument(std::string("epp: ") + (msg));          \
    } while (0)

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(bf16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ bf16 from_f<bf16>(float x) { return __float2bfloat16_rn(x); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-wide sum for blockDim.x <= 1024; `scratch` holds >= 32 floats.
__device__ __forceinline__ float block_sum(float v, float* scratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    const int nw = (blockDim.x + 31) >> 5;
    v = (threadIdx.x < nw) ? scratch[threadIdx.x] : 0.f;
    if (wid == 0) v = warp_sum(v);
    if (threadIdx.x == 0) scratch[0] = v;
    __syncthreads();
    const float r = scratch[0];
    __syncthreads();
    return r;
}

__device__ __forceinline__ float gelu_tanh_f(float x) {
    const float k = 0.7978845608028654f;
    return 0.5f * x * (1.f + tanhf(k * (x + 0.044715f * x * x * x)));
}
__device__ __forceinline__ float gelu_tanh_grad_f(float x) {
    const float k = 0.7978845608028654f;
    const float t = tanhf(k * (x + 0.044715f * x * x * x));
    return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * k * (1.f + 3.f * 0.044715f * x * x);
}

// bf16-path variants: gelu_tanh(x) = 0.5 x (1 + tanh(u)) = x * sigmoid(2u),
// u = k (x + 0.044715 x^3), with the sigmoid from MUFU exp2 + a fast divide
// (relative error ~1e-7 everywhere).  tanh.approx (abs. error ~5e-4) was
// cheaper by one MUFU op but its error is relative to 1 + tanh(u): ~20 % of
// gelu(x) at x = -3, a systematic bias that made the GPT-width gradients 1.6x
// less accurate than a torch autocast run of the same model
// (tools/bf16_error_table.py).
__device__ __forceinline__ float gelu_sigmoid_arg_(float x, float& du) {
    const float k2 = 2.f * 0.7978845608028654f;
    du = k2 * fmaf(3.f * 0.044715f * x, x, 1.f);            // d(2u)/dx
    return k2 * fmaf(0.044715f * x, x * x, x);               // 2u
}
__device__ __forceinline__ float gelu_tanh_fast_f(float x) {
    float du;
    const float z = gelu_sigmoid_arg_(x, du);
    return __fdividef(x, 1.f + __expf(-z));
}
// gelu(x) and gelu'(x) from one sigmoid
__device__ __forceinline__ float gelu_tanh_and_grad_fast_f(float x, float& grad) {
    float du;
    const float z = gelu_sigmoid_arg_(x, du);
    const float s = __fdividef(1.f, 1.f + __expf(-z));
    grad = fmaf(x * s * (1.f - s), du, s);
    return x * s;
}
__device__ __forceinline__ float gelu_tanh_grad_fast_f(float x) {
    float du;
    const float z = gelu_sigmoid_arg_(x, du);
    const float s = __fdividef(1.f, 1.f + __expf(-z));
    return fmaf(x * s * (1.f - s), du, s);
}

inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace eppk
