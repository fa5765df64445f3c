#include "ops.hpp"

namespace znn_gpu {

bool conv_tc_supported(const conv_shape&, int) { return false; }

void conv_fwd_tc(cudaStream_t, const conv_shape&, const float*, const float*, const float*, int,
                 float*, scratch&) {
    throw shape_error("tcgen05 conv: unsupported");
}
void conv_dgrad_tc(cudaStream_t, const conv_shape&, const float*, const float*, float*, scratch&) {
    throw shape_error("tcgen05 conv: unsupported");
}
void conv_wgrad_tc(cudaStream_t, const conv_shape&, const float*, const float*, float*, float,
                   scratch&) {
    throw shape_error("tcgen05 conv: unsupported");
}

}  // namespace znn_gpu
