// Internal C++ launcher API shared by the C-ABI (capi.cpp) and the network
// executor (net.cpp). All pointers are device pointers; all launches go to
// the given stream.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "common.cuh"

namespace znn_gpu {

// Grow-only device scratch arena (the steady state does no cudaMalloc; the
// analogue of the reference's never-freeing chunk_pool, mempool.hpp:29-154).
class scratch {
public:
    ~scratch();
    void* get(size_t bytes);
    size_t capacity() const { return cap_; }
    // a frozen arena throws instead of growing (zero-allocation steady state)
    void freeze(bool on) { frozen_ = on; }
    int64_t grows() const { return grows_; }

private:
    void* ptr_ = nullptr;
    size_t cap_ = 0;
    bool frozen_ = false;
    int64_t grows_ = 0;
};

// One fully connected conv layer: f_in maps of n -> f_out maps of m = n - s(k-1).
struct conv_shape {
    int64_t B = 1, f_in = 1, f_out = 1;
    dims3 n{1, 1, 1}, k{1, 1, 1}, s{1, 1, 1}, m{1, 1, 1};
    int64_t taps() const { return k.vol(); }
    static conv_shape make(int64_t B, int64_t f_in, int64_t f_out, dims3 n, dims3 k, dims3 s);
};

// ---- direct convolution, SIMT fp32 (conv_simt.cu) ----
void conv_fwd_simt(cudaStream_t st, const conv_shape& c, const float* x, const float* w,
                   const float* bias, int act, float* y);
void conv_dgrad_simt(cudaStream_t st, const conv_shape& c, const float* g, const float* w,
                     float* dx);
void conv_wgrad_simt(cudaStream_t st, const conv_shape& c, const float* x, const float* g,
                     float* dw, float scale, scratch& ws);

// ---- direct convolution, tcgen05 3xTF32 implicit GEMM (conv_tc.cu) ----
bool conv_tc_supported(const conv_shape& c, int pass);  // pass 0 fwd, 1 dgrad, 2 wgrad
void conv_fwd_tc(cudaStream_t st, const conv_shape& c, const float* x, const float* w,
                 const float* bias, int act, float* y, scratch& ws);
void conv_dgrad_tc(cudaStream_t st, const conv_shape& c, const float* g, const float* w,
                   float* dx, scratch& ws);
// single-input-map forward (conv1_tc.cu): weights resident in shared memory,
// persistent CTAs, double-buffered TMEM accumulator
bool conv1_tc_supported(const conv_shape& c);
void conv1_fwd_tc(cudaStream_t st, const conv_shape& c, const float* x, const float* w, const float* bias, int act,
                  float* y);
// SGD(+momentum) applied in a kernel epilogue right where the gradient is
// final (v = mu v + g; w -= lr v, the arithmetic of sgd_momentum)
struct sgd_fuse {
    float* w = nullptr;
    float* v = nullptr;
    float lr = 0.f, mu = 0.f;
};
// upd != nullptr: the split-K reduction also applies the update to the
// weights (dw is still written)
void conv_wgrad_tc(cudaStream_t st, const conv_shape& c, const float* x, const float* g,
                   float* dw, float scale, scratch& ws, const sgd_fuse* upd = nullptr);

// ---- pointwise (pointwise.cu) ----
void transfer_fwd(cudaStream_t st, const float* x, int64_t B, int64_t f, int64_t vox,
                  const int32_t* kinds_dev, const float* bias, float* y);
void transfer_bwd(cudaStream_t st, const float* g, const float* xy, bool from_output, int64_t B,
                  int64_t f, int64_t vox, const int32_t* kinds_dev, const float* bias,
                  float* gx, float* dbias, scratch& ws);
// returns unscaled loss sum (synchronises the stream)
double loss_grad(cudaStream_t st, int kind, const float* a, const float* d, int64_t count,
                 float scale, float* grad, scratch& ws);
// asynchronous variant: writes the unscaled loss sum into *loss_dev (double)
void loss_grad_async(cudaStream_t st, int kind, const float* a, const float* d, int64_t count,
                     float scale, float* grad, double* loss_dev, scratch& ws);
void sgd_momentum(cudaStream_t st, float* w, float* v, const float* g, int64_t count, float lr,
                  float mu);
void fill_zero(cudaStream_t st, float* p, int64_t count);

// ---- max ops (maxops.cu) ----
void maxpool_fwd(cudaStream_t st, const float* x, int64_t maps, dims3 n, dims3 p, float* y,
                 int32_t* mask);
void maxpool_bwd(cudaStream_t st, const float* g, const int32_t* mask, int64_t maps, dims3 m,
                 dims3 p, float* dx);
void maxfilter_fwd(cudaStream_t st, const float* x, int64_t maps, dims3 n, dims3 k, dims3 s,
                   float* y, int32_t* mask);
void maxfilter_bwd(cudaStream_t st, const float* g, const int32_t* mask, int64_t maps, dims3 m,
                   dims3 k, dims3 s, float* dx);
// one-byte window codes (a ky + b) kz + c instead of flat indices (windows of
// at most 256 taps; the executor's internal max-filters)
// relu_gate: windows whose maximum is not > 0 get code bit 7 (the backward
// then also applies the ReLU backward of the layer feeding the filter)
// pm: the filter's output image y (forward) / its gradient g (backward) is
// phase-major for sparsity pm.s ([B S][pm.f][m / s], phase (rx sy + ry) sz + rz,
// maps = B pm.f, power-of-two sz) instead of [maps][m]: the order the FFT
// layer consuming it wants (executor::plan_layouts); codes stay natural
struct pm_order {
    int on = 0, f = 1;
    dims3 s{1, 1, 1};
};
void maxfilter_fwd(cudaStream_t st, const float* x, int64_t maps, dims3 n, dims3 k, dims3 s,
                   float* y, uint8_t* code, bool relu_gate = false, pm_order pm = {});
// sum_part (2^3 windows, natural-order g only): the kernel also leaves per-warp partial sums of dx,
// [sum_f][maps / sum_f][maxfilter_bwd_sum_cols] floats; reduce_rows over the last two
// gives the per-map sums over the batch = the bias gradient of a ReLU layer whose
// backward the codes carry (no separate pass over dx)
void maxfilter_bwd(cudaStream_t st, const float* g, const uint8_t* code, int64_t maps, dims3 m,
                   dims3 k, dims3 s, float* dx, pm_order pm = {}, float* sum_part = nullptr, int sum_f = 1);
int64_t maxfilter_bwd_sum_cols(dims3 m, dims3 k, dims3 s);  // 0: this window has no partial-sum path
// out[r] = sum of part[r][0..cols) in fixed order (deterministic)
void reduce_rows(cudaStream_t st, const float* part, int64_t rows, int64_t cols, float* out);

}  // namespace znn_gpu
