// Shared host/device helpers for libznn_cuda.so (sm_100a only).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace znn_gpu {

// Shape/config violation -> status 1 (reference structural_error, types.hpp:57-74).
struct shape_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
// CUDA failure -> status 2.
struct cuda_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void require(bool cond, const std::string& what) {
    if (!cond) throw shape_error(what);
}

#define ZNN_CUDA_CHECK(expr)                                                             \
    do {                                                                                 \
        cudaError_t e_ = (expr);                                                         \
        if (e_ != cudaSuccess)                                                           \
            throw ::znn_gpu::cuda_error(std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// Launch bookkeeping: every kernel launch in the library goes through
// launch_check so the context can count its own launches (gpu_launches).
struct launch_stats {
    int64_t launches = 0;
};
launch_stats& stats();

inline void launch_check(const char* what) {
    stats().launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw cuda_error(std::string(what) + ": " + cudaGetErrorString(e));
}

struct dims3 {
    int64_t x, y, z;
    int64_t vol() const { return x * y * z; }
};

inline dims3 d3(const int64_t* p) { return dims3{p[0], p[1], p[2]}; }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

#if defined(__CUDACC__)
// Transfer functions (transfer.hpp:29-53) on device.
__device__ __forceinline__ float act_value(int kind, float x) {
    if (kind == 2) return x > 0.f ? x : 0.f;
    if (kind == 0) return 1.f / (1.f + expf(-x));
    if (kind == 1) return tanhf(x);
    return x;
}
// derivative from the transfer INPUT x (+bias already added); relu'(0)=0
__device__ __forceinline__ float act_deriv_in(int kind, float x) {
    if (kind == 2) return x > 0.f ? 1.f : 0.f;
    if (kind == 0) {
        const float v = 1.f / (1.f + expf(-x));
        return v * (1.f - v);
    }
    if (kind == 1) {
        const float v = tanhf(x);
        return 1.f - v * v;
    }
    return 1.f;
}
// derivative from the transfer OUTPUT y = phi(x)
__device__ __forceinline__ float act_deriv_out(int kind, float y) {
    if (kind == 2) return y > 0.f ? 1.f : 0.f;
    if (kind == 0) return y * (1.f - y);
    if (kind == 1) return 1.f - y * y;
    return 1.f;
}

#endif  // __CUDACC__

}  // namespace znn_gpu
