// Shared host/device helpers for libznn_cuda.so (sm_100a only).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

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
    int64_t allocs = 0;        // device allocations made by the library itself
    int64_t alloc_bytes = 0;
};
launch_stats& stats();

// Every internal device allocation goes through dmalloc so the steady state
// can be checked for zero allocations (reference acceptance.cpp:637-656).
template <typename T>
inline void dmalloc(T** p, size_t bytes) {
    void* v = nullptr;
    const cudaError_t e = cudaMalloc(&v, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw cuda_error("cudaMalloc(" + std::to_string(bytes) + " bytes): " + cudaGetErrorString(e));
    }
    stats().allocs++;
    stats().alloc_bytes += int64_t(bytes);
    *p = static_cast<T*>(v);
}

inline void launch_check(const char* what) {
    stats().launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw cuda_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// In-step kernel timing (bench.py's roofline): with profiling on, a
// prof_scope records a CUDA event pair on the launch stream around one
// launch; report() aggregates per kernel label (launches, total ms, and the
// algorithmic bytes / flops the caller declared per launch). Off by default;
// never active inside a stream capture.
struct prof_entry {
    std::string name;
    int64_t launches = 0;
    double ms = 0, bytes = 0, flops = 0;
};
void prof_enable(bool on);
bool prof_on();
std::vector<prof_entry> prof_report();  // synchronises on the recorded events, then clears
class prof_scope {
public:
    prof_scope(cudaStream_t st, std::string name, double bytes, double flops);
    ~prof_scope();
    prof_scope(const prof_scope&) = delete;
    prof_scope& operator=(const prof_scope&) = delete;

private:
    cudaStream_t st_;
    int slot_ = -1;
};

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
