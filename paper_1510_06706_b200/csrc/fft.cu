#include "fft.hpp"

namespace znn_fft {

bool supported(const conv_shape&) { return false; }

void conv_fwd(cudaStream_t, const conv_shape&, const float*, const float*, const float*, int,
              float*, znn_gpu::scratch&) {
    throw znn_gpu::shape_error("fft engine: not available for this layer");
}

void conv_bwd(cudaStream_t, const conv_shape&, const float*, const float*, const float*, float*,
              float*, znn_gpu::scratch&) {
    throw znn_gpu::shape_error("fft engine: not available for this layer");
}

}  // namespace znn_fft
