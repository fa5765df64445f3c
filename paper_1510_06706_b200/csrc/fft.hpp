// FFT-memoised convolution engine (conv_fft.hpp:25-125 / fft.hpp:57-192 of
// the reference): batched 3D R2C/C2R transforms, per-image spectra reused
// across the f x f' edges of a layer, per-frequency complex MAC over
// converging edges. Implemented in fft.cu.
#pragma once

#include "ops.hpp"

namespace znn_fft {

using znn_gpu::conv_shape;

bool supported(const conv_shape& c);
void conv_fwd(cudaStream_t st, const conv_shape& c, const float* x, const float* w,
              const float* bias, int act, float* y, znn_gpu::scratch& ws);
// wgrad into gw (overwritten); dgrad into gin when non-null
void conv_bwd(cudaStream_t st, const conv_shape& c, const float* x, const float* g,
              const float* w, float* gw, float* gin, znn_gpu::scratch& ws);

}  // namespace znn_fft
