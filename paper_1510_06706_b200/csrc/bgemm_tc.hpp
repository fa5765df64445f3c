// Per-bin complex GEMMs of the FFT engine's frequency-domain sums on the
// tcgen05 tensor cores (3xTF32); see bgemm_tc.cu. Spectra are image-major
// [img][bins] complex64; Bn = images per map group (B s^3 phase images).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "ops.hpp"

namespace znn_gpu {

// workspace bytes (bin-major hi / lo operands + the bin-major product) of the
// largest of the three sums for a layer
int64_t tc_cmac_bytes(int64_t Bn, int64_t f, int64_t fo, int64_t bins);
// shapes the kernels take: 2 f, 2 f' <= 256 (N of one MMA), Bn >= 256 (reuse)
bool tc_cmac_supported(int64_t Bn, int64_t f, int64_t fo);
// Y[n][o] = sum_i X[n][i] conj K[o][i]
void tc_cmac_fwd(cudaStream_t st, const float2* X, const float2* K, float2* Y, int64_t Bn, int64_t f, int64_t fo,
                 int64_t bins, void* ws);
// DX[n][i] = sum_o G[n][o] K[o][i]
void tc_cmac_dgrad(cudaStream_t st, const float2* G, const float2* K, float2* DX, int64_t Bn, int64_t f, int64_t fo,
                   int64_t bins, void* ws);
// dK[o][i] = sum_n X[n][i] conj G[n][o]
void tc_cmac_upd(cudaStream_t st, const float2* X, const float2* G, float2* DK, int64_t Bn, int64_t f, int64_t fo,
                 int64_t bins, void* ws);

}  // namespace znn_gpu
