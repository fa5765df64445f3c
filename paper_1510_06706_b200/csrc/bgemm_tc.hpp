// Per-bin complex GEMMs of the FFT engine's frequency-domain sums on the
// tcgen05 tensor cores (3xTF32); see bgemm_tc.cu.
//
// Spectra of tensor-core plans are stored in the GROUP layout: the images
// img = r * F + c of a spectrum (r = row-side index: phase image n, or output
// map o for kernel spectra; c = map) are grouped in runs of kGrp = 8
// consecutive maps, and a group's 8 spectra are interleaved bin by bin:
//   element (img, bin) at float2 index ((img / 8) * bins + bin) * 8 + img % 8.
// Every bin of a group is one 64-byte half line, so the transforms (one image
// per CTA, eight CTAs per cluster) write / read whole lines and the GEMMs
// load per-bin operand tiles straight from the transforms' output with 4-D
// TMA boxes of 64-byte pieces (no bin-major operand copies).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "ops.hpp"

namespace znn_gpu {

constexpr int kGrp = 8;

// shapes the kernels take: f, f' <= 128 and multiples of 8 (N of one MMA,
// whole groups), Bn >= 128 phase images (reuse of every kernel-spectrum bin)
bool tc_cmac_supported(int64_t Bn, int64_t f, int64_t fo);
// group-layout spectra: X [Bn][f], K [fo][f], G / Y [Bn][fo], DX [Bn][f], DK [fo][f]
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
