// Per-bin complex GEMMs of the FFT engine's frequency-domain sums on the
// tcgen05 tensor cores (3xTF32); see bgemm_tc.cu.
//
// Spectra of tensor-core plans are stored ROW-BIN-MAJOR: the images
// img = r * F + c of a spectrum (r = row-side index: phase image n, or output
// map o for kernel spectra; c = one of the F maps) are interleaved bin by bin:
//   element (img, bin) at float2 index (r * bins + bin) * F + c.
// Per (row, bin) the F maps are one contiguous 8 F-byte piece, so the GEMMs
// load per-bin operand tiles straight from the transforms' output with 3-D
// TMA boxes of whole lines (no bin-major operand copies), and a transform CTA
// that handles a few consecutive maps still reads / writes whole sectors.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "ops.hpp"

namespace znn_gpu {

// shapes the kernels take: f, f' <= 128 and multiples of 8 (N of one MMA),
// Bn >= 32 phase images (reuse of every kernel-spectrum bin; below, the
// register-tiled FMA CMACs are faster: an M = 128 tile would be mostly empty)
bool tc_cmac_supported(int64_t Bn, int64_t f, int64_t fo);
// row-bin-major spectra: X [Bn][f], K [fo][f], G / Y [Bn][fo], DX [Bn][f], DK [fo][f]
// Y[n][o] = sum_i X[n][i] conj K[o][i]
void tc_cmac_fwd(cudaStream_t st, const float2* X, const float2* K, float2* Y, int64_t Bn, int64_t f, int64_t fo,
                 int64_t bins);
// DX[n][i] = sum_o G[n][o] K[o][i]
void tc_cmac_dgrad(cudaStream_t st, const float2* G, const float2* K, float2* DX, int64_t Bn, int64_t f, int64_t fo,
                   int64_t bins);
// dK[o][i] = sum_n X[n][i] conj G[n][o]
void tc_cmac_upd(cudaStream_t st, const float2* X, const float2* G, float2* DK, int64_t Bn, int64_t f, int64_t fo,
                 int64_t bins);

}  // namespace znn_gpu
