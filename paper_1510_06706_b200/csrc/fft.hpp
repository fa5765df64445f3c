// FFT-memoised convolution engine (conv_fft.hpp:25-192 / fft.hpp:57-192 of
// the reference), B200-native: batched 3D transforms of images by
// hand-written shared-memory kernels (radix 2/3/4/5/8 codelets, pads
// 2^a 3^b 5^c <= 128), kernel spectra straight from the weights by
// sparse-tap plane DFTs and the kernel-gradient inverse as their adjoint,
// per-image spectra memoised from the forward pass into the backward and
// update passes as the reference's memo_store does (image spectrum once per
// node, kernel spectrum once per edge per iteration; the largest layers
// share one kernel-spectrum buffer and recompute when it was overwritten),
// and the frequency-domain sum over converging edges as register-tiled
// per-frequency complex multiply-accumulate kernels (FP32-FMA bound at
// 16 patches).
#pragma once

#include <cstdint>
#include <memory>

#include "ops.hpp"

namespace znn_fft {

using znn_gpu::conv_shape;

// per-pass transform counters, mirroring fft.hpp:19-49 (phase x kind)
struct transform_counts {
    int64_t fwd_image = 0, fwd_kernel = 0, fwd_inverse = 0;
    int64_t bwd_image = 0, bwd_kernel = 0, bwd_inverse = 0;
    int64_t upd_image = 0, upd_kernel = 0, upd_inverse = 0;
};

struct plan;  // pad dims + memoised spectra (device memory)
struct plan_deleter {
    void operator()(plan* p) const;
};
using plan_ptr = std::unique_ptr<plan, plan_deleter>;

// Kernel spectra are the big per-layer object (f_in*f_out*bins complex: 52 GB
// for c5 conv2). A layer either keeps its own (memoised from the forward into
// the backward, conv_fft.hpp:38-96) or borrows one buffer shared by several
// layers; a borrowed buffer is recomputed in the backward pass when another
// layer has overwritten it since this layer's forward. Either way the weight
// gradient's product spectra dK reuse the kernel-spectrum buffer (K is dead
// once the data gradient is formed).
struct kpool {
    float2* buf = nullptr;
    int64_t bytes = 0;
    const void* owner = nullptr;  // plan whose current K the buffer holds
    ~kpool();
    float2* get(int64_t need);
};

int64_t kernel_spectrum_bytes(const conv_shape& c);
int64_t image_spectrum_bytes(const conv_shape& c);  // the memoised X of a plan
int64_t workspace_bytes(const conv_shape& c);       // scratch arena of conv_fwd / conv_bwd
bool supported(const conv_shape& c);
// phase_ws: arena for the phase-split tensors of dilated layers (shared by
// the layers of one executor; a plan gets its own when null)
plan_ptr make_plan(const conv_shape& c, std::shared_ptr<kpool> pool = nullptr,
                   std::shared_ptr<znn_gpu::scratch> phase_ws = nullptr);
int64_t phase_bytes(const conv_shape& c);  // phase-split tensors of a dilated layer (0 if none)
const transform_counts& counts(const plan& p);
void pad_dims(const plan& p, int64_t out[3]);

// forward: y = act(bias + sum_i IFFT(X_i * conj(K_oi))) cropped (conv_fft.hpp:38-60);
// memoises X (image spectra) and K (kernel spectra) in the plan.
// x_pm / y_pm: the input / output tensor is phase-major ([B s^3][maps][n / s],
// phase r = (rx sy + ry) sz + rz) instead of [B][maps][n]; phase_major_ok(c)
// says whether the layer's plan can take such tensors.
bool phase_major_ok(const conv_shape& c);
bool phase_major_pays(const conv_shape& c);  // worth a scattering producer (small-cube plans)
void conv_fwd(cudaStream_t st, plan& p, const conv_shape& c, const float* x, const float* w,
              const float* bias, int act, float* y, znn_gpu::scratch& ws, bool x_pm = false, bool y_pm = false);
// backward + update from the memo: gin = IFFT(sum_o G_o * K_oi) (no conjugate,
// conv_fft.hpp:67-96, skipped when gin == nullptr) and
// gw = IFFT(sum_b X_bi * conj(G_bo))[s*w] (conv_fft.hpp:98-125). With relu_y,
// the layer's fused ReLU backward is applied while g is transformed (g * (y > 0))
// and dbias[o] receives its bias gradient (the DC term summed over patches).
void conv_bwd(cudaStream_t st, plan& p, const conv_shape& c, const float* x, const float* g,
              const float* w, float* gw, float* gin, znn_gpu::scratch& ws, const float* relu_y = nullptr,
              float* dbias = nullptr, bool x_pm = false, bool y_pm = false);

// average device time (ms) of one CMAC launch on synthetic spectra (roofline probe)
float time_cmac(cudaStream_t st, int which, const conv_shape& c, int reps, int64_t* bins_out);

// measured FP32 FMA throughput (TFLOP/s) of this GPU: the CMAC roofline
float fma_peak_tflops(cudaStream_t st);

}  // namespace znn_fft
