// Frequency-domain sums over converging edges (the CMACs of the FFT engine,
// conv_fft.hpp:38-125 summed by merge_payload, engine.hpp:345-353) as
// per-bin complex GEMMs on the tcgen05 tensor cores, 3xTF32.
//
// For the polyphase plans of dilated layers every kernel-spectrum bin feeds
// B s^3 phase images (c5 conv3-5: 1024), so per bin the three sums are
// real GEMMs with a large reuse dimension:
//   fwd  : Y[n][o]  = sum_i X[n][i] conj K[o][i]   D[n][(o,c')]  = A(X)  . B(K)
//   dgrad: DX[n][i] = sum_o G[n][o] K[o][i]         D[n][(i,c')]  = A(G)  . B(K^T)
//   upd  : dK[o][i] = sum_n X[n][i] conj G[n][o]    D[o][(i,c')]  = A(G^T). B(X^T)
// with complex numbers embedded as (re, im) pairs along K and the output
// columns (o, c') interleaved, so D rows are the natural complex layout. A
// rows are the natural complex rows of the left operand; B rows come in two
// variants per column ((re, im) and a swapped / negated copy), e.g. for fwd
// Yr = sum (Xr Kr + Xi Ki) = A . (Kr, Ki), Yi = sum (Xi Kr - Xr Ki) = A . (-Ki, Kr).
//
// Spectra live image-major ([img][bins], bins contiguous: what the
// transforms produce). prep_k transposes them bin-major ([bin][row][k]) and
// splits fp32 into hi (the raw value: the MMA reads the top 19 bits) and
// lo = x - tf32(x); unprep_k transposes D back. The GEMM kernel is a TMA ->
// tcgen05 pipeline: persistent CTAs over (bin, 128-row) tiles, K in 32-wide
// chunks (SWIZZLE_128B K-major tiles, 2 stages), D (N <= 256 columns) in a
// double-buffered TMEM accumulator, D += Ahi Bhi + Ahi Blo + Alo Bhi.
#include <cuda.h>

#include <algorithm>

#include "bgemm_tc.hpp"
#include "tc_common.cuh"

namespace znn_gpu {

CUtensorMap make_panel_map_rows(const float* ptr, int64_t cols, int64_t rows, int box_rows);

namespace {

using namespace znn_tc;

constexpr int TB = 32;  // transpose tile (images or k-side indices) x bins

// variant code: bit0 swap (re, im) -> (im, re), bit1 negate the first, bit2 the second
__device__ __forceinline__ float2 variant(float2 z, int code) {
    float2 r = (code & 1) ? make_float2(z.y, z.x) : z;
    if (code & 2) r.x = -r.x;
    if (code & 4) r.y = -r.y;
    return r;
}

// S [img = p * F + q][bins] complex -> T [bin][row][k] fp32, the bin-major
// operand the GEMM's TMA reads (hi / lo and B's row variants are made in
// shared memory by the GEMM). ROWQ = false: row = p (R = Pn), k = 2 q + c
// (K = 2 F); ROWQ = true: row = q (R = F), k = 2 p + c (K = 2 Pn).
// block: one row-side index, TB k-side indices x TB bins; threads 32 x 8
template <bool ROWQ>
__global__ void __launch_bounds__(256) prep_k(const float2* __restrict__ S, int64_t bins, int Pn, int F,
                                              float* __restrict__ T) {
    __shared__ float2 tile[TB][TB + 1];
    const int rs = blockIdx.z;                // row-side index (p, or q when ROWQ)
    const int j0 = blockIdx.y * TB;           // k-side indices (q, or p when ROWQ)
    const int64_t w0 = int64_t(blockIdx.x) * TB;
    const int nk = ROWQ ? Pn : F;             // k-side extent
    const int K = 2 * nk;
    const int R = ROWQ ? F : Pn;              // rows per bin
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (int jj = ty; jj < TB; jj += 8) {
        const int j = j0 + jj;
        const int64_t w = w0 + tx;
        float2 v = make_float2(0.f, 0.f);
        if (j < nk && w < bins) {
            const int64_t img = ROWQ ? int64_t(j) * F + rs : int64_t(rs) * F + j;
            v = __ldcs(S + img * bins + w);
        }
        tile[jj][tx] = v;
    }
    __syncthreads();
    // out row (bin, rs): the k-side pairs j0..j0+TB as 2 TB consecutive floats
    for (int ww = ty; ww < TB; ww += 8) {
        const int64_t w = w0 + ww;
        if (w >= bins) continue;
        float* o = T + (w * R + rs) * K + 2 * j0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int e = tx + 32 * h, jj = e >> 1;
            if (j0 + jj < nk) {
                const float2 z = tile[jj][ww];
                o[e] = (e & 1) ? z.y : z.x;
            }
        }
    }
}

// D [bin][p][2 Q] fp32 (complex rows) -> S [p * Q + q][bins] complex
__global__ void __launch_bounds__(256) unprep_k(const float* __restrict__ D, int64_t bins, int Pn, int Q,
                                                int ldd, float2* __restrict__ S) {
    __shared__ float2 tile[TB][TB + 1];
    const int p = blockIdx.z, q0 = blockIdx.y * TB;
    const int64_t w0 = int64_t(blockIdx.x) * TB;
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (int ww = ty; ww < TB; ww += 8) {
        const int64_t w = w0 + ww;
        float2 v = make_float2(0.f, 0.f);
        if (w < bins && q0 + tx < Q) v = *reinterpret_cast<const float2*>(D + (w * Pn + p) * int64_t(ldd) + 2 * (q0 + tx));
        tile[ww][tx] = v;
    }
    __syncthreads();
    for (int qq = ty; qq < TB; qq += 8) {
        const int q = q0 + qq;
        const int64_t w = w0 + tx;
        if (q < Q && w < bins) __stcs(S + (int64_t(p) * Q + q) * bins + w, tile[tx][qq]);
    }
}

constexpr int BM = 128;   // rows per CTA tile (TMEM lanes)
constexpr int BKC = 32;   // K per stage (one 128-byte swizzle row)
constexpr int STAGES = 2;

struct bg_params {
    int M, N, K;          // per bin: D[M][N] = sum_k A[M][k] B[N][k]
    int NB;               // raw B rows per bin loaded by TMA (N, or N / 2 with two variants per row)
    int v0, v1;           // variant codes of B rows 2r, 2r + 1 (NB = N / 2)
    int ldd;              // D row pitch (floats)
    int mtiles;
};

// the 16-byte chunk q of row r of a 128B-swizzled K-major tile
__device__ __forceinline__ uint32_t sw_chunk(uint32_t r, uint32_t q) { return r * 128u + (((q ^ (r & 7u)) & 7u) << 4); }

__device__ __forceinline__ float4 lo4(float4 v) {
    return make_float4(v.x - tf32_hi(v.x), v.y - tf32_hi(v.y), v.z - tf32_hi(v.z), v.w - tf32_hi(v.w));
}
__device__ __forceinline__ float4 var4(float4 v, int code) {  // two complex pairs
    const float2 a = variant(make_float2(v.x, v.y), code), b = variant(make_float2(v.z, v.w), code);
    return make_float4(a.x, a.y, b.x, b.y);
}

// Persistent: one CTA per SM walks the (bin, 128-row) tiles t = blockIdx.x,
// blockIdx.x + gridDim.x, ...; the stage ring runs across tiles and the
// accumulator is double-buffered in TMEM (2 x 256 columns), so the drain of
// tile t overlaps the loads and MMAs of tile t + 1.
// warps 0-3: operand expansion (lo = x - tf32(x) of A and B, B's two row
//            variants) of every stage;
// warps 4-7: epilogue (TMEM lane quarter = warp % 4): drain D rows to HBM;
// warp 8   : TMA of the raw A (128 rows) and raw B (NB rows) tiles;
// warp 9   : TMEM allocation and the MMA issue (Ahi.Bhi + Ahi.Blo + Alo.Bhi).
// Stage layout: [A raw = A hi][A lo][B raw][B hi][B lo] (B hi = B raw when NB == N).
constexpr int BG_THREADS = 320;
__global__ void __launch_bounds__(BG_THREADS, 1)
bgemm_tc_k(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB, float* __restrict__ D,
           bg_params p, int64_t ntiles) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* base_ptr = smem_raw + (base - raw);
    const bool expand = p.NB != p.N;
    const uint32_t a_bytes = BM * 128u, braw_bytes = uint32_t(p.NB) * 128u, b_bytes = uint32_t(p.N) * 128u;
    const uint32_t off_alo = a_bytes, off_braw = 2u * a_bytes, off_bhi = off_braw + (expand ? braw_bytes : 0u);
    const uint32_t off_blo = off_bhi + b_bytes;
    const uint32_t stage_bytes = ((off_blo + b_bytes + 1023u) / 1024u) * 1024u;
    const uint32_t tma_bytes = a_bytes + braw_bytes;
    const uint32_t bar_base = base + STAGES * stage_bytes;
    auto full_bar = [&](int s) { return bar_base + 8u * uint32_t(s); };
    auto conv_bar = [&](int s) { return bar_base + 8u * uint32_t(STAGES + s); };
    auto empty_bar = [&](int s) { return bar_base + 8u * uint32_t(2 * STAGES + s); };
    auto accf_bar = [&](int b) { return bar_base + 8u * uint32_t(3 * STAGES + b); };
    auto acce_bar = [&](int b) { return bar_base + 8u * uint32_t(3 * STAGES + 2 + b); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base_ptr + (bar_base - base) + 8u * uint32_t(3 * STAGES + 4));

    const int warp = threadIdx.x >> 5;
    const int nchunks = (p.K + BKC - 1) / BKC;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(conv_bar(s), 128);
            mbar_init(empty_bar(s), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(accf_bar(b), 1);
            mbar_init(acce_bar(b), 128);
        }
        fence_barrier_init();
    }
    if (warp == 9) tmem_alloc(smem_u32(tmem_slot), 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 8) {
        int s = 0;
        uint32_t ph = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const int64_t bin = t / p.mtiles;
            const int m0 = int(t - bin * p.mtiles) * BM;
            const int arow = int(bin * p.M + m0), brow = int(bin * p.NB);
            for (int c = 0; c < nchunks; ++c) {
                mbar_wait(empty_bar(s), ph ^ 1u);
                const uint32_t st0 = base + uint32_t(s) * stage_bytes;
                asm volatile(
                    "{\n\t.reg .pred pe;\n\t"
                    "elect.sync _|pe, 0xffffffff;\n\t"
                    "@pe mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t}" ::"r"(full_bar(s)),
                    "r"(tma_bytes)
                    : "memory");
                tma_w(full_bar(s), st0, &tA, c * BKC, arow);
                tma_w(full_bar(s), st0 + off_braw, &tB, c * BKC, brow);
                if (++s == STAGES) s = 0, ph ^= 1u;
            }
        }
    } else if (warp == 9) {
        const uint32_t idesc = idesc_tf32(BM, p.N);
        int s = 0;
        uint32_t ph = 0;
        int it = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const int b = it & 1;
            mbar_wait(acce_bar(b), uint32_t((it >> 1) & 1) ^ 1u);  // the epilogue drained this buffer
            tc_fence_after();
            const uint32_t d = tmem + uint32_t(b) * 256u;
            for (int c = 0; c < nchunks; ++c) {
                mbar_wait(conv_bar(s), ph);
                tc_fence_after();
                const uint32_t st0 = base + uint32_t(s) * stage_bytes;
                const uint32_t a_hi = st0, a_lo = st0 + off_alo, b_hi = st0 + off_bhi, b_lo = st0 + off_blo;
                const int ksteps = min(BKC, p.K - c * BKC) / 8;
                for (int kk = 0; kk < ksteps; ++kk) {
                    const uint32_t ko = uint32_t(kk) * 32u;  // 8 fp32 along K
                    const uint64_t ah = sw128_desc(a_hi + ko), al = sw128_desc(a_lo + ko);
                    const uint64_t bh = sw128_desc(b_hi + ko), bl = sw128_desc(b_lo + ko);
                    mma_tf32_w(d, ah, bh, idesc, (c == 0 && kk == 0) ? 0u : 1u);
                    mma_tf32_w(d, ah, bl, idesc, 1u);
                    mma_tf32_w(d, al, bh, idesc, 1u);
                }
                mma_commit_w(empty_bar(s));
                if (++s == STAGES) s = 0, ph ^= 1u;
            }
            mma_commit_w(accf_bar(b));
        }
    } else if (warp < 4) {
        // ---- operand expansion of every stage ----
        const int t0 = threadIdx.x;  // 0..127
        int s = 0;
        uint32_t ph = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            for (int c = 0; c < nchunks; ++c) {
                mbar_wait(full_bar(s), ph);
                uint8_t* st0 = base_ptr + size_t(s) * stage_bytes;
                for (int i = t0; i < BM * 8; i += 128) {  // A lo
                    const uint32_t o = sw_chunk(uint32_t(i >> 3), uint32_t(i & 7));
                    *reinterpret_cast<float4*>(st0 + off_alo + o) = lo4(*reinterpret_cast<const float4*>(st0 + o));
                }
                if (expand) {  // B rows 2r + c' = variant c' of raw row r, hi and lo
                    for (int i = t0; i < p.NB * 8; i += 128) {
                        const uint32_t r = uint32_t(i >> 3), q = uint32_t(i & 7);
                        const float4 v = *reinterpret_cast<const float4*>(st0 + off_braw + sw_chunk(r, q));
                        const float4 h0 = var4(v, p.v0), h1 = var4(v, p.v1);
                        const uint32_t o0 = sw_chunk(2u * r, q), o1 = sw_chunk(2u * r + 1u, q);
                        *reinterpret_cast<float4*>(st0 + off_bhi + o0) = h0;
                        *reinterpret_cast<float4*>(st0 + off_bhi + o1) = h1;
                        *reinterpret_cast<float4*>(st0 + off_blo + o0) = lo4(h0);
                        *reinterpret_cast<float4*>(st0 + off_blo + o1) = lo4(h1);
                    }
                } else {
                    for (int i = t0; i < p.N * 8; i += 128) {
                        const uint32_t o = sw_chunk(uint32_t(i >> 3), uint32_t(i & 7));
                        *reinterpret_cast<float4*>(st0 + off_blo + o) =
                            lo4(*reinterpret_cast<const float4*>(st0 + off_braw + o));
                    }
                }
                fence_proxy_async();  // generic-proxy writes -> visible to the tensor cores
                mbar_arrive(conv_bar(s));
                if (++s == STAGES) s = 0, ph ^= 1u;
            }
        }
    } else {
        // ---- epilogue: warps 4-7, lane = row of the tile ----
        const int r = threadIdx.x - 128;  // 0..127
        const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
        int it = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const int b = it & 1;
            const int64_t bin = t / p.mtiles;
            const int row = int(t - bin * p.mtiles) * BM + r;
            mbar_wait(accf_bar(b), uint32_t((it >> 1) & 1));
            tc_fence_after();
            float* drow = D + (bin * p.M + row) * int64_t(p.ldd);
            const uint32_t acol = tmem + lane_base + uint32_t(b) * 256u;
            for (int c0 = 0; c0 < p.N; c0 += 16) {
                float v[16];
                tmem_ld16(acol + uint32_t(c0), v);
                tmem_wait_ld();
                if (row < p.M) {
#pragma unroll
                    for (int q = 0; q < 16; q += 4)
                        __stcs(reinterpret_cast<float4*>(drow + c0 + q), make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]));
                }
            }
            tc_fence_before();
            mbar_arrive(acce_bar(b));
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 9) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// S [img = p * F + q][bins] complex -> T [bin][row][k] fp32 (transpose only)
template <bool ROWQ>
void prep(cudaStream_t st, const float2* S, int64_t bins, int Pn, int F, float* T) {
    const int nk = ROWQ ? Pn : F, rsn = ROWQ ? F : Pn;
    require(rsn < 65536 && ceil_div(nk, TB) < 65536, "tc cmac: prep grid exceeds 65535");
    const dim3 grid(unsigned(ceil_div(bins, TB)), unsigned(ceil_div(nk, TB)), unsigned(rsn));
    prep_k<ROWQ><<<grid, dim3(32, 8, 1), 0, st>>>(S, bins, Pn, F, T);
    launch_check("tc_cmac_prep");
}

void unprep(cudaStream_t st, const float* Dp, int64_t bins, int Pn, int Q, int ldd, float2* S) {
    require(Pn < 65536, "tc cmac: unprep grid exceeds 65535");
    const dim3 grid(unsigned(ceil_div(bins, TB)), unsigned(ceil_div(Q, TB)), unsigned(Pn));
    unprep_k<<<grid, dim3(32, 8, 1), 0, st>>>(Dp, bins, Pn, Q, ldd, S);
    launch_check("tc_cmac_unprep");
}

// D[bin][M][N] = A[bin][M][K] . B[bin][N][K]^T with B rows 2r + c' = variant
// c' of the raw row r (raw B: [bin][N / 2][K])
void bgemm(cudaStream_t st, const float* A, const float* B, float* Dp, int64_t nb, int M, int N, int K, int v0, int v1) {
    require(N % 16 == 0 && N <= 256 && K % 8 == 0, "tc cmac: bad GEMM shape");
    const int NB = N / 2;
    require(nb * M < (int64_t(1) << 31) && nb * NB < (int64_t(1) << 31), "tc cmac: operand rows exceed 2^31");
    const CUtensorMap ta = make_panel_map_rows(A, K, nb * M, BM), tb = make_panel_map_rows(B, K, nb * NB, NB);
    bg_params p{M, N, K, NB, v0, v1, N, int(ceil_div(M, BM))};
    const size_t stage = ((size_t(2 * BM * 128 + NB * 128 + 2 * N * 128) + 1023) / 1024) * 1024;
    const size_t smem = size_t(STAGES) * stage + 1024 + 256;
    require(smem <= 227 * 1024, "tc cmac: stage does not fit in shared memory");
    const int64_t ntiles = nb * p.mtiles;
    int dev = 0, sms = 148;
    ZNN_CUDA_CHECK(cudaGetDevice(&dev));
    ZNN_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const unsigned grid = unsigned(std::min<int64_t>(ntiles, sms));  // persistent: one CTA per SM
    ZNN_CUDA_CHECK(cudaFuncSetAttribute(bgemm_tc_k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    bgemm_tc_k<<<grid, BG_THREADS, smem, st>>>(ta, tb, Dp, p, ntiles);
    launch_check("tc_cmac_gemm");
}

}  // namespace

int64_t tc_cmac_bytes(int64_t Bn, int64_t f, int64_t fo, int64_t bins) {
    // bin-major A + raw B + D of the largest of the three GEMMs
    const int64_t fwd = bins * Bn * 2 * f + bins * fo * 2 * f + bins * Bn * 2 * fo;
    const int64_t dgr = bins * Bn * 2 * fo + bins * f * 2 * fo + bins * Bn * 2 * f;
    const int64_t upd = bins * fo * 2 * Bn + bins * f * 2 * Bn + bins * fo * 2 * f;
    return int64_t(sizeof(float)) * std::max(fwd, std::max(dgr, upd)) + 4096;
}

bool tc_cmac_supported(int64_t Bn, int64_t f, int64_t fo) {
    // N = 2 f' (fwd), 2 f (dgrad / upd) <= 256 and a multiple of 16; enough
    // reuse per kernel-spectrum bin to pay the operand transposes
    return Bn >= 128 && 2 * f <= 256 && 2 * fo <= 256 && (2 * f) % 16 == 0 && (2 * fo) % 16 == 0;
}

namespace {
float* carve_f(char*& cur, int64_t n) {
    float* p = reinterpret_cast<float*>(cur);
    cur += ((int64_t(sizeof(float)) * n + 1023) / 1024) * 1024;
    return p;
}
}  // namespace

// Y[n][o] = sum_i X[n][i] conj K[o][i]; X [n f + i][bins], K [o f + i][bins], Y [n fo + o][bins]
void tc_cmac_fwd(cudaStream_t st, const float2* X, const float2* K, float2* Y, int64_t Bn, int64_t f, int64_t fo,
                 int64_t bins, void* ws) {
    char* cur = static_cast<char*>(ws);
    const int kk = int(2 * f), nn = int(2 * fo);
    float* A = carve_f(cur, bins * Bn * kk);
    float* B = carve_f(cur, bins * fo * kk);
    float* Dp = carve_f(cur, bins * Bn * nn);
    prep<false>(st, X, bins, int(Bn), int(f), A);
    prep<false>(st, K, bins, int(fo), int(f), B);
    // rows (o, re): (Kr, Ki) over i; (o, im): (-Ki, Kr)
    bgemm(st, A, B, Dp, bins, int(Bn), nn, kk, 0, 1 | 2);
    unprep(st, Dp, bins, int(Bn), int(fo), nn, Y);
}

// DX[n][i] = sum_o G[n][o] K[o][i]; G [n fo + o][bins], DX [n f + i][bins]
void tc_cmac_dgrad(cudaStream_t st, const float2* G, const float2* K, float2* DX, int64_t Bn, int64_t f, int64_t fo,
                   int64_t bins, void* ws) {
    char* cur = static_cast<char*>(ws);
    const int kk = int(2 * fo), nn = int(2 * f);
    float* A = carve_f(cur, bins * Bn * kk);
    float* B = carve_f(cur, bins * f * kk);
    float* Dp = carve_f(cur, bins * Bn * nn);
    prep<false>(st, G, bins, int(Bn), int(fo), A);
    prep<true>(st, K, bins, int(fo), int(f), B);  // K images o f + i: rows i, k = (o, c)
    // rows (i, re): (Kr, -Ki) over o; (i, im): (Ki, Kr)
    bgemm(st, A, B, Dp, bins, int(Bn), nn, kk, 4, 1);
    unprep(st, Dp, bins, int(Bn), int(f), nn, DX);
}

// dK[o][i] = sum_n X[n][i] conj G[n][o]; dK [o f + i][bins]
void tc_cmac_upd(cudaStream_t st, const float2* X, const float2* G, float2* DK, int64_t Bn, int64_t f, int64_t fo,
                 int64_t bins, void* ws) {
    char* cur = static_cast<char*>(ws);
    const int kk = int(2 * Bn), nn = int(2 * f);
    float* A = carve_f(cur, bins * fo * kk);
    float* B = carve_f(cur, bins * f * kk);
    float* Dp = carve_f(cur, bins * fo * nn);
    prep<true>(st, G, bins, int(Bn), int(fo), A);  // rows o: (Gr, Gi) over n
    prep<true>(st, X, bins, int(Bn), int(f), B);   // rows i: (Xr, Xi) over n
    // rows (i, re): (Xr, Xi); (i, im): (Xi, -Xr)
    bgemm(st, A, B, Dp, bins, int(fo), nn, kk, 0, 1 | 4);
    unprep(st, Dp, bins, int(fo), int(f), nn, DK);
}

}  // namespace znn_gpu
