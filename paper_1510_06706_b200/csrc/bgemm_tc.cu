// Frequency-domain sums over converging edges (the CMACs of the FFT engine,
// conv_fft.hpp:38-125 summed by merge_payload, engine.hpp:345-353) as
// per-bin complex GEMMs on the tcgen05 tensor cores, 3xTF32.
//
// For the polyphase plans of dilated layers every kernel-spectrum bin feeds
// B s^3 phase images (c5: 128 at conv2, 1024 at conv3-5), so per bin the
// three sums are real GEMMs with a large reuse dimension:
//   fwd  : Y[n][o]  = sum_i X[n][i] conj K[o][i]
//   dgrad: DX[n][i] = sum_o G[n][o] K[o][i]
//   upd  : dK[o][i] = sum_n X[n][i] conj G[n][o]
// Complex numbers are (re, im) pairs along K. The B operand is always the raw
// right-hand spectrum (rows = output columns, K = (index, re / im)); the real
// and imaginary outputs are two accumulators D_r = A . B, D_i = A' . B whose
// left operands are per-element variants of the left spectrum, e.g. fwd:
// Yr = sum Xr Kr + Xi Ki -> A = (Xr, Xi), Yi = sum Xi Kr - Xr Ki -> A' = (Xi, -Xr).
//
// Operands come straight from the row-bin-major spectra (bgemm_tc.hpp) by 3-D
// TMA boxes of whole 128-byte (or longer) pieces: a 128-row x 16-complex
// tile, or a 16-row x all-columns tile for the operands that are transposed
// within the bin. Kernel layout:
//   * A (and A') hi / lo live in TMEM (tcgen05.mma A-from-TMEM form), written
//     by 8 expansion warps from the raw tile: no A copies in shared memory;
//   * B hi / lo are written by the same warps in the canonical 128B-swizzled
//     K-major layout (transposing where the box is K-outer);
//   * one MMA warp issues D_r += Ahi Bhi + Ahi Blo + Alo Bhi and the same for
//     D_i (M = 128 rows, N <= 128);
//   * the TMA ring of raw tiles (4 stages) is released as soon as the
//     expansion warps hold the values, so loads run ahead of the MMAs;
//   * 4 epilogue warps drain D (D_r / D_i interleaved into complex) through
//     two 16-column shared staging tiles and TMA tensor stores into the
//     row-bin-major output (128-byte pieces).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "bgemm_tc.hpp"
#include "tc_common.cuh"

namespace znn_gpu {

void* tensor_map_encoder();  // conv_tc.cu

namespace {

using namespace znn_tc;

typedef CUresult (*encode_fn_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// 3-D view (floats) of a row-bin-major spectrum with R row-side images x F
// maps: (2 F floats of a row-bin, bin, row); box (bc floats, 1, br rows)
CUtensorMap rbm_map(const float2* ptr, int64_t bins, int64_t F, int64_t R, int bc, int br) {
    CUtensorMap m;
    const cuuint64_t dims[3] = {cuuint64_t(2 * F), cuuint64_t(bins), cuuint64_t(R)};
    const cuuint64_t strides[2] = {cuuint64_t(8 * F), cuuint64_t(bins) * cuuint64_t(8 * F)};
    const cuuint32_t box[3] = {cuuint32_t(bc), 1, cuuint32_t(br)};
    const cuuint32_t estr[3] = {1, 1, 1};
    auto enc = reinterpret_cast<encode_fn_t>(tensor_map_encoder());
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float2*>(ptr), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw cuda_error("cuTensorMapEncodeTiled (row-bin-major spectrum) failed: " + std::to_string(int(r)));
    return m;
}

// variant code: bit0 swap (re, im) -> (im, re), bit1 negate the first, bit2 the second
__device__ __forceinline__ float2 variant(float2 z, int code) {
    float2 r = (code & 1) ? make_float2(z.y, z.x) : z;
    if (code & 2) r.x = -r.x;
    if (code & 4) r.y = -r.y;
    return r;
}
__device__ __forceinline__ float4 lo4(float4 v) {
    return make_float4(v.x - tf32_hi(v.x), v.y - tf32_hi(v.y), v.z - tf32_hi(v.z), v.w - tf32_hi(v.w));
}
// byte offset of 16-byte chunk q of row r in a 128B-swizzled K-major tile
__device__ __forceinline__ uint32_t sw_chunk(uint32_t r, uint32_t q) { return r * 128u + (((q ^ (r & 7u)) & 7u) << 4); }

__device__ __forceinline__ void tma3_w(uint32_t bar, uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2) {
    asm volatile(
        "{\n\t.reg .pred pe;\n\t"
        "elect.sync _|pe, 0xffffffff;\n\t"
        "@pe cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n\t}" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma3_store(const CUtensorMap* m, uint32_t src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                     reinterpret_cast<uint64_t>(m)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(src)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

__device__ __forceinline__ void tmem_st16(uint32_t addr, const float (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            addr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
        "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
        "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
        "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])),
        "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
        : "memory");
}

// two 16-column TMEM loads of this thread's lane and their completion wait in
// one asm statement (the outputs cannot be consumed before the wait)
__device__ __forceinline__ void tmem_ld16_pair(uint32_t addr0, uint32_t addr1, float (&a)[16], float (&b)[16]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%32];\n\t"
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%33];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(addr0), "r"(addr1)
        : "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = __uint_as_float(r[i]), b[i] = __uint_as_float(r[16 + i]);
}

constexpr int RS = 4;                 // raw operand stages (TMA ring)
constexpr int XS = 2;                 // expanded stages (B hi / lo in smem, A / A' hi / lo in TMEM)
constexpr int NH = 128;               // output columns per tile (N <= 128)
constexpr int OB = 16;                // output columns per staging block
constexpr uint32_t A_BYTES = 16384;   // A tile: 128 rows x 32 floats, or 16 K-rows x <= 128 complex
constexpr uint32_t B_BYTES = 16384;   // B tile: 128 rows x 32 floats, or 16 K-rows x <= 128 complex
constexpr uint32_t RAW_BYTES = A_BYTES + B_BYTES;
constexpr uint32_t X_BYTES = 2 * B_BYTES;  // B hi, B lo (128B-swizzled K-major, 128 rows)
constexpr uint32_t STG_BYTES = 128 * OB * 8;  // output staging: 128 rows x OB complex
constexpr int CG_THREADS = 448;            // warps 0-7 expansion, 8-11 epilogue, 12 TMA, 13 MMA
constexpr size_t CG_SMEM = 1024 + RS * size_t(RAW_BYTES) + XS * size_t(X_BYTES) + 2 * size_t(STG_BYTES) + 256;

struct cg_params {
    int M, N;             // D rows, D columns (complex)
    int nchunks, klast;   // K chunks of 16 complex; K steps (8 floats) of the last chunk
    int mtiles;           // 128-row tiles
    int a_trans, b_trans; // operand tile is K-outer (16 rows of K x columns)
    int aF, bF;           // maps (complex columns) per row of the A / B tensors
    int va, vap;          // variant codes of A and A'
    uint32_t tx_bytes;    // A box + B box
};

// Persistent CTAs over tiles t = (bin, 128-row tile). TMEM: D_r at columns
// [0, 128), D_i at [128, 256), A buffers (Ahi, Alo, A'hi, A'lo: 32 columns
// each) at [256, 384) / [384, 512). D is single-buffered: the epilogue
// releases it after its last TMEM load, while the TMA ring (released by the
// expansion warps, not the MMAs) and the expanded stages keep filling.
__global__ void __launch_bounds__(CG_THREADS, 1)
cgemm_tc_k(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
           const __grid_constant__ CUtensorMap tD, cg_params p, int64_t ntiles) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* base_ptr = smem_raw + (base - raw);
    const uint32_t xbase = base + RS * RAW_BYTES;
    const uint32_t stg = xbase + XS * X_BYTES;
    uint8_t* stg_ptr = base_ptr + (stg - base);
    const uint32_t bar_base = stg + 2 * STG_BYTES;
    auto rfull = [&](int s) { return bar_base + 8u * uint32_t(s); };
    auto rempty = [&](int s) { return bar_base + 8u * uint32_t(RS + s); };
    auto xfull = [&](int s) { return bar_base + 8u * uint32_t(2 * RS + s); };
    auto xempty = [&](int s) { return bar_base + 8u * uint32_t(2 * RS + XS + s); };
    auto accf = [&](int b) { return bar_base + 8u * uint32_t(2 * RS + 2 * XS + b); };
    auto acce = [&](int b) { return bar_base + 8u * uint32_t(2 * RS + 2 * XS + 2 + b); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base_ptr + (bar_base - base) + 8u * uint32_t(2 * RS + 2 * XS + 4));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < RS; ++s) {
            mbar_init(rfull(s), 1);
            mbar_init(rempty(s), 8);  // one elected arrive per expansion warp
        }
        for (int s = 0; s < XS; ++s) {
            mbar_init(xfull(s), 8);
            mbar_init(xempty(s), 1);
        }
        mbar_init(accf(0), 1);
        mbar_init(acce(0), 4);  // one elected arrive per epilogue warp
        fence_barrier_init();
    }
    if (warp == 13) tmem_alloc(smem_u32(tmem_slot), 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 12) {
        // ---- TMA producer ----
        int s = 0;
        uint32_t ph = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const int64_t bin = t / p.mtiles;
            const int m0 = int(t - bin * p.mtiles) * 128;
            for (int c = 0; c < p.nchunks; ++c) {
                mbar_wait(rempty(s), ph ^ 1u);
                const uint32_t st0 = base + uint32_t(s) * RAW_BYTES;
                asm volatile(
                    "{\n\t.reg .pred pe;\n\t"
                    "elect.sync _|pe, 0xffffffff;\n\t"
                    "@pe mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t}" ::"r"(rfull(s)),
                    "r"(p.tx_bytes)
                    : "memory");
                if (p.a_trans)  // K-rows 16 c.., all columns
                    tma3_w(rfull(s), st0, &tA, 0, int(bin), 16 * c);
                else            // 128 rows, the 16 complex of chunk c
                    tma3_w(rfull(s), st0, &tA, 32 * c, int(bin), m0);
                if (p.b_trans)
                    tma3_w(rfull(s), st0 + A_BYTES, &tB, 0, int(bin), 16 * c);
                else            // rows = output columns
                    tma3_w(rfull(s), st0 + A_BYTES, &tB, 32 * c, int(bin), 0);
                if (++s == RS) s = 0, ph ^= 1u;
            }
        }
    } else if (warp == 13) {
        // ---- MMA issue ----
        const uint32_t idesc = idesc_tf32(128, ((p.N + 15) / 16) * 16);
        int x = 0;
        uint32_t xph = 0;
        int it = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            mbar_wait(acce(0), uint32_t(it & 1) ^ 1u);  // the epilogue drained D
            tc_fence_after();
            const uint32_t d_r = tmem, d_i = tmem + 128u;
            for (int c = 0; c < p.nchunks; ++c) {
                mbar_wait(xfull(x), xph);
                tc_fence_after();
                const uint32_t bhi = xbase + uint32_t(x) * X_BYTES, blo = bhi + B_BYTES;
                const uint32_t a0 = tmem + 256u + 128u * uint32_t(x);
                const int ks = (c == p.nchunks - 1) ? p.klast : 4;
                for (int kk = 0; kk < ks; ++kk) {
                    const uint64_t bh = sw128_desc(bhi + uint32_t(kk) * 32u), bl = sw128_desc(blo + uint32_t(kk) * 32u);
                    const uint32_t a = a0 + uint32_t(kk) * 8u;
                    const uint32_t acc = (c == 0 && kk == 0) ? 0u : 1u;
                    mma_tf32_ts_w(d_r, a, bh, idesc, acc);
                    mma_tf32_ts_w(d_r, a, bl, idesc, 1u);
                    mma_tf32_ts_w(d_r, a + 32u, bh, idesc, 1u);
                    mma_tf32_ts_w(d_i, a + 64u, bh, idesc, acc);
                    mma_tf32_ts_w(d_i, a + 64u, bl, idesc, 1u);
                    mma_tf32_ts_w(d_i, a + 96u, bh, idesc, 1u);
                }
                mma_commit_w(xempty(x));
                if (++x == XS) x = 0, xph ^= 1u;
            }
            mma_commit_w(accf(0));
        }
    } else if (warp < 8) {
        // ---- operand expansion: A -> TMEM (hi, lo, A' hi, A' lo), B -> smem hi / lo ----
        const int q = warp & 3, h = warp >> 2;
        const int row = q * 32 + lane;  // TMEM lane = A row
        const uint32_t lane_base = uint32_t(q * 32) << 16;
        const int tid = threadIdx.x;    // 0..255
        int s = 0, x = 0;
        uint32_t ph = 0, xph = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            for (int c = 0; c < p.nchunks; ++c) {
                mbar_wait(rfull(s), ph);
                mbar_wait(xempty(x), xph ^ 1u);
                tc_fence_after();
                const uint8_t* st0 = base_ptr + size_t(s) * RAW_BYTES;
                // A: 8 complex (16 floats) of this row: K floats [16 h, 16 h + 16) of the chunk
                float2 xa[8];
                if (p.a_trans) {  // tile [16 k-rows][aF complex]; A row = column index
                    const float2* src = reinterpret_cast<const float2*>(st0);
                    const bool ok = row < p.M;
#pragma unroll
                    for (int u = 0; u < 8; ++u) xa[u] = ok ? src[(8 * h + u) * p.aF + row] : make_float2(0.f, 0.f);
                } else {  // tile [128 rows][32 floats]: chunks 4h..4h+3 of the row, rotated by lane (bank spread)
                    const float4* src = reinterpret_cast<const float4*>(st0 + size_t(row) * 128);
                    float4 t4[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) t4[u] = src[4 * h + ((u + lane) & 3)];
                    const int rot = lane & 3;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int src_i = (k - rot) & 3;  // t4[u] holds chunk (u + rot) & 3
                        float4 v = t4[0];
                        if (src_i == 1) v = t4[1];
                        if (src_i == 2) v = t4[2];
                        if (src_i == 3) v = t4[3];
                        xa[2 * k] = make_float2(v.x, v.y);
                        xa[2 * k + 1] = make_float2(v.z, v.w);
                    }
                }
                // B: 128 rows = output columns, 8 chunks of 16 bytes (4 per thread)
                float4 vb[4];
                if (p.b_trans) {  // tile [16 k-rows][bF complex]: transpose into K-major rows
                    const float2* src = reinterpret_cast<const float2*>(st0 + A_BYTES);
                    const int ncol = p.bF;
#pragma unroll
                    for (int tt = 0; tt < 4; ++tt) {
                        const int u = tid + 256 * tt;
                        const int i = u & 127, j = u >> 7;
                        vb[tt] = make_float4(0.f, 0.f, 0.f, 0.f);
                        if (i < ncol) {
                            const float2 a = src[(2 * j) * ncol + i], b = src[(2 * j + 1) * ncol + i];
                            vb[tt] = make_float4(a.x, a.y, b.x, b.y);
                        }
                    }
                } else {  // tile [128 rows][32 floats]
                    const uint8_t* src = st0 + A_BYTES;
#pragma unroll
                    for (int tt = 0; tt < 4; ++tt) {
                        const int u = tid + 256 * tt;
                        vb[tt] = *reinterpret_cast<const float4*>(src + (u >> 3) * 128 + (u & 7) * 16);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(rempty(s));  // the raw stage is consumed (values in registers)
                {
                    float vh[16], vl[16], wh[16], wl[16];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const float2 lo = make_float2(xa[u].x - tf32_hi(xa[u].x), xa[u].y - tf32_hi(xa[u].y));
                        const float2 a = variant(xa[u], p.va), al = variant(lo, p.va);
                        const float2 b = variant(xa[u], p.vap), bl = variant(lo, p.vap);
                        vh[2 * u] = a.x, vh[2 * u + 1] = a.y;
                        vl[2 * u] = al.x, vl[2 * u + 1] = al.y;
                        wh[2 * u] = b.x, wh[2 * u + 1] = b.y;
                        wl[2 * u] = bl.x, wl[2 * u + 1] = bl.y;
                    }
                    const uint32_t a0 = tmem + lane_base + 256u + 128u * uint32_t(x) + uint32_t(16 * h);
                    tmem_st16(a0, vh);
                    tmem_st16(a0 + 32u, vl);
                    tmem_st16(a0 + 64u, wh);
                    tmem_st16(a0 + 96u, wl);
                }
                {
                    uint8_t* bhi = base_ptr + (xbase - base) + size_t(x) * X_BYTES;
                    uint8_t* blo = bhi + B_BYTES;
#pragma unroll
                    for (int tt = 0; tt < 4; ++tt) {
                        const int u = tid + 256 * tt;
                        const uint32_t r = p.b_trans ? uint32_t(u & 127) : uint32_t(u >> 3);
                        const uint32_t j = p.b_trans ? uint32_t(u >> 7) : uint32_t(u & 7);
                        const uint32_t o = sw_chunk(r, j);
                        *reinterpret_cast<float4*>(bhi + o) = vb[tt];
                        *reinterpret_cast<float4*>(blo + o) = lo4(vb[tt]);
                    }
                }
                tmem_wait_st();
                tc_fence_before();
                fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor cores
                __syncwarp();
                if (lane == 0) mbar_arrive(xfull(x));
                if (++s == RS) s = 0, ph ^= 1u;
                if (++x == XS) x = 0, xph ^= 1u;
            }
        }
    } else {
        // ---- epilogue: warps 8-11 (TMEM lane quarter = warp % 4), row = lane of the tile ----
        const int q = warp & 3;
        const int r = q * 32 + lane;
        const uint32_t lane_base = uint32_t(q * 32) << 16;
        const bool leader = threadIdx.x == 256;
        int it = 0, sb = 0;
        const int nob = (p.N + OB - 1) / OB;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const int64_t bin = t / p.mtiles;
            const int m0 = int(t - bin * p.mtiles) * 128;
            mbar_wait(accf(0), uint32_t(it & 1));
            tc_fence_after();
            for (int ob = 0; ob < nob; ++ob) {
                float dr[16], di[16];
                tmem_ld16_pair(tmem + lane_base + uint32_t(OB * ob), tmem + lane_base + 128u + uint32_t(OB * ob), dr, di);
                if (ob == nob - 1) {  // D fully read: the next tile's MMAs may start
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(acce(0));
                }
                // staging buffer sb is free once at most one store (from the other buffer) is pending
                if (leader) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                epi_bar();
                // row r: OB complex = 8 chunks of 16 bytes (a 128-byte row); the chunk order
                // rotates with the lane, so a warp's 16-byte stores cover all 8 bank groups
                float4* dst = reinterpret_cast<float4*>(stg_ptr + size_t(sb) * STG_BYTES + size_t(r) * (OB * 8));
                const int rot = lane & 7;
                float4 cc[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) cc[k] = make_float4(dr[2 * k], di[2 * k], dr[2 * k + 1], di[2 * k + 1]);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int k = (u + rot) & 7;
                    const float4 a0 = (k & 1) ? cc[1] : cc[0], a1 = (k & 1) ? cc[3] : cc[2];
                    const float4 a2 = (k & 1) ? cc[5] : cc[4], a3 = (k & 1) ? cc[7] : cc[6];
                    const float4 b0 = (k & 2) ? a1 : a0, b1 = (k & 2) ? a3 : a2;
                    dst[k] = (k & 4) ? b1 : b0;
                }
                fence_proxy_async();
                epi_bar();
                if (leader) tma3_store(&tD, stg + uint32_t(sb) * STG_BYTES, 2 * OB * ob, int(bin), m0);
                sb ^= 1;
            }
        }
        if (leader) bulk_wait0();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 13) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// mode 0 fwd, 1 dgrad, 2 upd
void cgemm(cudaStream_t st, int mode, const float2* Ap, const float2* Bp, float2* Dp, int64_t Bn, int64_t f,
           int64_t fo, int64_t bins) {
    require(tc_cmac_supported(Bn, f, fo), "tc cmac: unsupported shape");
    require(bins < (int64_t(1) << 31), "tc cmac: too many bins");
    cg_params p{};
    CUtensorMap ta, tb, td;
    int64_t kdim = 0;  // complex K extent
    if (mode == 0) {            // A = X [Bn][f] rows n; B = K [fo][f] rows o; D = Y [Bn][fo]
        p.M = int(Bn), p.N = int(fo), kdim = f;
        p.a_trans = 0, p.b_trans = 0;
        ta = rbm_map(Ap, bins, f, Bn, 32, 128);
        tb = rbm_map(Bp, bins, f, fo, 32, NH);
        td = rbm_map(Dp, bins, fo, Bn, 2 * OB, 128);
        p.va = 0, p.vap = 1 | 4;  // A = (re, im), A' = (im, -re)
    } else if (mode == 1) {     // A = G [Bn][fo] rows n; B = K [fo][f] K-outer (rows o), columns i; D = DX [Bn][f]
        p.M = int(Bn), p.N = int(f), kdim = fo;
        p.a_trans = 0, p.b_trans = 1;
        ta = rbm_map(Ap, bins, fo, Bn, 32, 128);
        tb = rbm_map(Bp, bins, f, fo, int(2 * f), 16);
        td = rbm_map(Dp, bins, f, Bn, 2 * OB, 128);
        p.va = 4, p.vap = 1;      // A = (re, -im), A' = (im, re)
    } else {                    // A = G [Bn][fo] K-outer (rows n), columns o; B = X [Bn][f] K-outer; D = DK [fo][f]
        p.M = int(fo), p.N = int(f), kdim = Bn;
        p.a_trans = 1, p.b_trans = 1;
        ta = rbm_map(Ap, bins, fo, Bn, int(2 * fo), 16);
        tb = rbm_map(Bp, bins, f, Bn, int(2 * f), 16);
        td = rbm_map(Dp, bins, f, fo, 2 * OB, 128);
        p.va = 0, p.vap = 1 | 2;  // A = (re, im), A' = (-im, re)
    }
    p.aF = int(mode == 0 ? f : fo);
    p.bF = int(f);
    p.nchunks = int(ceil_div(kdim, 16));
    p.klast = int(ceil_div(2 * (kdim - 16 * (p.nchunks - 1)), 8));
    p.mtiles = mode == 2 ? 1 : int(ceil_div(Bn, 128));
    const uint32_t a_box = p.a_trans ? uint32_t(16 * p.aF * 8) : A_BYTES;
    const uint32_t b_box = p.b_trans ? uint32_t(16 * p.bF * 8) : B_BYTES;
    p.tx_bytes = a_box + b_box;
    const int64_t ntiles = bins * p.mtiles;
    int dev = 0, sms = 148;
    ZNN_CUDA_CHECK(cudaGetDevice(&dev));
    ZNN_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const unsigned grid = unsigned(std::min<int64_t>(ntiles, sms));  // persistent: one CTA per SM
    ZNN_CUDA_CHECK(cudaFuncSetAttribute(cgemm_tc_k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(CG_SMEM)));
    cgemm_tc_k<<<grid, CG_THREADS, CG_SMEM, st>>>(ta, tb, td, p, ntiles);
    launch_check("tc_cmac_gemm");
}

}  // namespace

bool tc_cmac_supported(int64_t Bn, int64_t f, int64_t fo) {
    const char* e = std::getenv("ZNN_TC_MIN_BN");
    return Bn >= (e ? std::atoi(e) : 32) && f <= 128 && fo <= 128 && f % 8 == 0 && fo % 8 == 0;
}

void tc_cmac_fwd(cudaStream_t st, const float2* X, const float2* K, float2* Y, int64_t Bn, int64_t f, int64_t fo,
                 int64_t bins) {
    cgemm(st, 0, X, K, Y, Bn, f, fo, bins);
}
void tc_cmac_dgrad(cudaStream_t st, const float2* G, const float2* K, float2* DX, int64_t Bn, int64_t f, int64_t fo,
                   int64_t bins) {
    cgemm(st, 1, G, K, DX, Bn, f, fo, bins);
}
void tc_cmac_upd(cudaStream_t st, const float2* X, const float2* G, float2* DK, int64_t Bn, int64_t f, int64_t fo,
                 int64_t bins) {
    cgemm(st, 2, G, X, DK, Bn, f, fo, bins);
}

}  // namespace znn_gpu
