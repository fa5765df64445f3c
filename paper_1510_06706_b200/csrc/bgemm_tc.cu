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
// Operands come straight from the group-layout spectra (bgemm_tc.hpp) by 4-D
// TMA boxes (a 128-row x 16-complex tile, or a 16-row x all-columns tile for
// the operands that are transposed within the bin). Kernel layout:
//   * A (and A') hi / lo live in TMEM (tcgen05.mma A-from-TMEM form), written
//     by 8 expansion warps from the raw tile: no A copies in shared memory;
//   * B hi / lo are written by the same warps in the canonical 128B-swizzled
//     K-major layout (transposing where the box is K-outer);
//   * one MMA warp issues D_r += Ahi Bhi + Ahi Blo + Alo Bhi and the same for
//     D_i (M = 128 rows, N <= 128), 3 smem stages, 2 TMEM A buffers;
//   * 4 epilogue warps drain D (D_r / D_i interleaved into complex) through a
//     shared staging tile and TMA tensor stores into the group-layout output.
// Persistent CTAs walk the (bin, 128-row tile) list.
#include <cuda.h>

#include <algorithm>

#include "bgemm_tc.hpp"
#include "tc_common.cuh"

namespace znn_gpu {

void* tensor_map_encoder();  // conv_tc.cu

namespace {

using namespace znn_tc;

typedef CUresult (*encode_fn_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// 4-D view of a group-layout spectrum with R row-side images x F maps:
// (2 kGrp floats of a group-bin, bin, group = map / kGrp, row); box (2 kGrp, 1, bq, br)
CUtensorMap grp_map(const float2* ptr, int64_t bins, int64_t F, int64_t R, int bq, int br) {
    CUtensorMap m;
    const int64_t fq = F / kGrp;
    constexpr int64_t gb = 8 * kGrp;  // bytes of a group-bin
    const cuuint64_t dims[4] = {2 * kGrp, cuuint64_t(bins), cuuint64_t(fq), cuuint64_t(R)};
    const cuuint64_t strides[3] = {gb, cuuint64_t(bins) * gb, cuuint64_t(fq * bins) * gb};
    const cuuint32_t box[4] = {2 * kGrp, 1, cuuint32_t(bq), cuuint32_t(br)};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    auto enc = reinterpret_cast<encode_fn_t>(tensor_map_encoder());
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float2*>(ptr), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw cuda_error("cuTensorMapEncodeTiled (group spectrum) failed: " + std::to_string(int(r)));
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

__device__ __forceinline__ void tma4_w(uint32_t bar, uint32_t dst, const CUtensorMap* m, int c1, int c2, int c3) {
    asm volatile(
        "{\n\t.reg .pred pe;\n\t"
        "elect.sync _|pe, 0xffffffff;\n\t"
        "@pe cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n\t}" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma4_store(const CUtensorMap* m, uint32_t src, int c1, int c2, int c3) {
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(
                     reinterpret_cast<uint64_t>(m)),
                 "r"(0), "r"(c1), "r"(c2), "r"(c3), "r"(src)
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

constexpr int CG_STAGES = 3;
constexpr uint32_t BOX_BYTES = 16384;            // one operand tile (128 x 32 floats, or 16 x <= 128 complex)
constexpr uint32_t STAGE_BYTES = 4 * BOX_BYTES;  // [A raw][B raw][B hi][B lo]
constexpr uint32_t STG_BYTES = 32768;            // output staging: 128 rows x 32 complex
constexpr int CG_THREADS = 448;                  // warps 0-7 expansion, 8-11 epilogue, 12 TMA, 13 MMA
constexpr size_t CG_SMEM = 1024 + CG_STAGES * size_t(STAGE_BYTES) + STG_BYTES + 256;

struct cg_params {
    int M, N, nmma;       // D rows, D columns (complex), MMA N (N rounded up to 16)
    int nchunks, klast;   // K chunks of 16 complex; K steps (8 floats) of the last chunk
    int mtiles;
    int a_trans, b_trans; // operand tile is K-outer (16 rows of K x all columns)
    int aq, bq;           // groups per row of the A / B tensors
    int va, vap;          // variant codes of A and A'
    int nob;              // 32-column output blocks
    uint32_t tx_bytes;    // A box + B box
};

__global__ void __launch_bounds__(CG_THREADS, 1)
cgemm_tc_k(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
           const __grid_constant__ CUtensorMap tD, cg_params p, int64_t ntiles) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* base_ptr = smem_raw + (base - raw);
    const uint32_t stg = base + CG_STAGES * STAGE_BYTES;
    uint8_t* stg_ptr = base_ptr + CG_STAGES * STAGE_BYTES;
    const uint32_t bar_base = stg + STG_BYTES;
    auto full_bar = [&](int s) { return bar_base + 8u * uint32_t(s); };
    auto conv_bar = [&](int s) { return bar_base + 8u * uint32_t(CG_STAGES + s); };
    auto empty_bar = [&](int s) { return bar_base + 8u * uint32_t(2 * CG_STAGES + s); };
    auto aempty_bar = [&](int b) { return bar_base + 8u * uint32_t(3 * CG_STAGES + b); };
    const uint32_t accf_bar = bar_base + 8u * uint32_t(3 * CG_STAGES + 2);
    const uint32_t acce_bar = accf_bar + 8u;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base_ptr + (acce_bar + 8u - base));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < CG_STAGES; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(conv_bar(s), 256);
            mbar_init(empty_bar(s), 1);
        }
        mbar_init(aempty_bar(0), 1);
        mbar_init(aempty_bar(1), 1);
        mbar_init(accf_bar, 1);
        mbar_init(acce_bar, 128);
        fence_barrier_init();
    }
    if (warp == 13) tmem_alloc(smem_u32(tmem_slot), 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;  // D_r: cols [0, 128), D_i: [128, 256), A buffers: [256, 384), [384, 512)

    if (warp == 12) {
        // ---- TMA producer ----
        int s = 0;
        uint32_t ph = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const int64_t bin = t / p.mtiles;
            const int m0 = int(t - bin * p.mtiles) * 128;
            for (int c = 0; c < p.nchunks; ++c) {
                mbar_wait(empty_bar(s), ph ^ 1u);
                const uint32_t st0 = base + uint32_t(s) * STAGE_BYTES;
                asm volatile(
                    "{\n\t.reg .pred pe;\n\t"
                    "elect.sync _|pe, 0xffffffff;\n\t"
                    "@pe mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t}" ::"r"(full_bar(s)),
                    "r"(p.tx_bytes)
                    : "memory");
                if (p.a_trans)
                    tma4_w(full_bar(s), st0, &tA, int(bin), 0, 16 * c);
                else
                    tma4_w(full_bar(s), st0, &tA, int(bin), (16 / kGrp) * c, m0);
                if (p.b_trans)
                    tma4_w(full_bar(s), st0 + BOX_BYTES, &tB, int(bin), 0, 16 * c);
                else
                    tma4_w(full_bar(s), st0 + BOX_BYTES, &tB, int(bin), (16 / kGrp) * c, 0);
                if (++s == CG_STAGES) s = 0, ph ^= 1u;
            }
        }
    } else if (warp == 13) {
        // ---- MMA issue ----
        const uint32_t idesc = idesc_tf32(128, p.nmma);
        const uint32_t d_r = tmem, d_i = tmem + 128u;
        int s = 0;
        uint32_t ph = 0;
        int g = 0;  // global chunk counter (TMEM A buffer = g & 1)
        int it = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            mbar_wait(acce_bar, uint32_t(it & 1) ^ 1u);  // the epilogue drained the previous tile's D
            tc_fence_after();
            for (int c = 0; c < p.nchunks; ++c, ++g) {
                mbar_wait(conv_bar(s), ph);
                tc_fence_after();
                const uint32_t st0 = base + uint32_t(s) * STAGE_BYTES;
                const uint32_t bhi = st0 + 2 * BOX_BYTES, blo = st0 + 3 * BOX_BYTES;
                const uint32_t a0 = tmem + 256u + 128u * uint32_t(g & 1);
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
                mma_commit_w(empty_bar(s));
                mma_commit_w(aempty_bar(g & 1));
                if (++s == CG_STAGES) s = 0, ph ^= 1u;
            }
            mma_commit_w(accf_bar);
        }
    } else if (warp < 8) {
        // ---- operand expansion: A -> TMEM (hi, lo, A' hi, A' lo), B -> smem hi / lo ----
        const int q = warp & 3, h = warp >> 2;
        const int row = q * 32 + lane;  // TMEM lane = A row
        const uint32_t lane_base = uint32_t(q * 32) << 16;
        const int tid = threadIdx.x;    // 0..255
        int s = 0;
        uint32_t ph = 0;
        int g = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            for (int c = 0; c < p.nchunks; ++c, ++g) {
                mbar_wait(full_bar(s), ph);
                mbar_wait(aempty_bar(g & 1), uint32_t((g >> 1) & 1) ^ 1u);
                tc_fence_after();
                uint8_t* st0 = base_ptr + size_t(s) * STAGE_BYTES;
                // A: 8 complex (16 floats) of this row: K floats [16 h, 16 h + 16) of the chunk
                float2 x[8];
                if (p.a_trans) {  // tile [16 k-rows][aq groups][2 kGrp floats]; A row = column index
                    const float2* src = reinterpret_cast<const float2*>(st0);
                    const bool ok = row < p.M;
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        x[u] = ok ? src[(8 * h + u) * (p.aq * kGrp) + row] : make_float2(0.f, 0.f);
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
                        x[2 * k] = make_float2(v.x, v.y);
                        x[2 * k + 1] = make_float2(v.z, v.w);
                    }
                }
                {
                    float vh[16], vl[16], wh[16], wl[16];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const float2 lo = make_float2(x[u].x - tf32_hi(x[u].x), x[u].y - tf32_hi(x[u].y));
                        const float2 a = variant(x[u], p.va), al = variant(lo, p.va);
                        const float2 b = variant(x[u], p.vap), bl = variant(lo, p.vap);
                        vh[2 * u] = a.x, vh[2 * u + 1] = a.y;
                        vl[2 * u] = al.x, vl[2 * u + 1] = al.y;
                        wh[2 * u] = b.x, wh[2 * u + 1] = b.y;
                        wl[2 * u] = bl.x, wl[2 * u + 1] = bl.y;
                    }
                    const uint32_t a0 = tmem + lane_base + 256u + 128u * uint32_t(g & 1) + uint32_t(16 * h);
                    tmem_st16(a0, vh);
                    tmem_st16(a0 + 32u, vl);
                    tmem_st16(a0 + 64u, wh);
                    tmem_st16(a0 + 96u, wl);
                }
                // B: rows = output columns (128, zero / unused beyond N), 8 chunks of 16 bytes
                uint8_t* bhi = st0 + 2 * BOX_BYTES;
                uint8_t* blo = st0 + 3 * BOX_BYTES;
                if (p.b_trans) {  // tile [16 k-rows][bq groups][2 kGrp floats]: transpose into K-major rows
                    const float2* src = reinterpret_cast<const float2*>(st0 + BOX_BYTES);
                    const int ncol = p.bq * kGrp;
#pragma unroll
                    for (int tt = 0; tt < 4; ++tt) {
                        const int u = tid + 256 * tt;
                        const int i = u & 127, j = u >> 7;
                        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                        if (i < ncol) {
                            const float2 a = src[(2 * j) * ncol + i], b = src[(2 * j + 1) * ncol + i];
                            v = make_float4(a.x, a.y, b.x, b.y);
                        }
                        const uint32_t o = sw_chunk(uint32_t(i), uint32_t(j));
                        *reinterpret_cast<float4*>(bhi + o) = v;
                        *reinterpret_cast<float4*>(blo + o) = lo4(v);
                    }
                } else {  // tile [128 rows][32 floats]
                    const uint8_t* src = st0 + BOX_BYTES;
#pragma unroll
                    for (int tt = 0; tt < 4; ++tt) {
                        const int u = tid + 256 * tt;
                        const int r = u >> 3, j = u & 7;
                        const float4 v = *reinterpret_cast<const float4*>(src + r * 128 + j * 16);
                        const uint32_t o = sw_chunk(uint32_t(r), uint32_t(j));
                        *reinterpret_cast<float4*>(bhi + o) = v;
                        *reinterpret_cast<float4*>(blo + o) = lo4(v);
                    }
                }
                tmem_wait_st();
                tc_fence_before();
                fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor cores
                mbar_arrive(conv_bar(s));
                if (++s == CG_STAGES) s = 0, ph ^= 1u;
            }
        }
    } else {
        // ---- epilogue: warps 8-11 (TMEM lane quarter = warp % 4), row = lane of the tile ----
        const int q = warp & 3;
        const int r = q * 32 + lane;
        const uint32_t lane_base = uint32_t(q * 32) << 16;
        const bool leader = threadIdx.x == 256;
        int it = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const int64_t bin = t / p.mtiles;
            const int m0 = int(t - bin * p.mtiles) * 128;
            mbar_wait(accf_bar, uint32_t(it & 1));
            tc_fence_after();
            for (int ob = 0; ob < p.nob; ++ob) {
                // the staging tile is free once the previous TMA store has read it
                if (leader) bulk_wait_read0();
                epi_bar();
                // row r: 32 complex = 16 chunks of 16 bytes, chunk k = (re, im) of columns 2k, 2k + 1;
                // within each half row the chunk order rotates with the lane, so a
                // warp's 16-byte stores cover all 8 bank groups (4 wavefronts)
                float4* dst = reinterpret_cast<float4*>(stg_ptr + size_t(r) * 256);
                const int rot = lane & 7;
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    float dr[16], di[16];
                    const uint32_t col = uint32_t(32 * ob + 16 * hh);
                    tmem_ld16_pair(tmem + lane_base + col, tmem + lane_base + 128u + col, dr, di);
                    if (ob == p.nob - 1 && hh == 1) {  // D fully read: the next tile's MMAs may start
                        tc_fence_before();
                        mbar_arrive(acce_bar);
                    }
                    float4 c[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) c[k] = make_float4(dr[2 * k], di[2 * k], dr[2 * k + 1], di[2 * k + 1]);
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int k = (u + rot) & 7;
                        const float4 a0 = (k & 1) ? c[1] : c[0], a1 = (k & 1) ? c[3] : c[2];
                        const float4 a2 = (k & 1) ? c[5] : c[4], a3 = (k & 1) ? c[7] : c[6];
                        const float4 b0 = (k & 2) ? a1 : a0, b1 = (k & 2) ? a3 : a2;
                        dst[8 * hh + k] = (k & 4) ? b1 : b0;
                    }
                }
                fence_proxy_async();
                epi_bar();
                if (leader) tma4_store(&tD, stg, int(bin), (32 / kGrp) * ob, m0);
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
        ta = grp_map(Ap, bins, f, Bn, 16 / kGrp, 128);
        tb = grp_map(Bp, bins, f, fo, 16 / kGrp, 128);
        td = grp_map(Dp, bins, fo, Bn, 32 / kGrp, 128);
        p.va = 0, p.vap = 1 | 4;  // A = (re, im), A' = (im, -re)
    } else if (mode == 1) {     // A = G [Bn][fo] rows n; B = K [fo][f] K-outer (rows o), columns i; D = DX [Bn][f]
        p.M = int(Bn), p.N = int(f), kdim = fo;
        p.a_trans = 0, p.b_trans = 1;
        ta = grp_map(Ap, bins, fo, Bn, 16 / kGrp, 128);
        tb = grp_map(Bp, bins, f, fo, int(f / kGrp), 16);
        td = grp_map(Dp, bins, f, Bn, 32 / kGrp, 128);
        p.va = 4, p.vap = 1;      // A = (re, -im), A' = (im, re)
    } else {                    // A = G [Bn][fo] K-outer (rows n), columns o; B = X [Bn][f] K-outer; D = DK [fo][f]
        p.M = int(fo), p.N = int(f), kdim = Bn;
        p.a_trans = 1, p.b_trans = 1;
        ta = grp_map(Ap, bins, fo, Bn, int(fo / kGrp), 16);
        tb = grp_map(Bp, bins, f, Bn, int(f / kGrp), 16);
        td = grp_map(Dp, bins, f, fo, 32 / kGrp, 128);
        p.va = 0, p.vap = 1 | 2;  // A = (re, im), A' = (-im, re)
    }
    p.aq = int((mode == 0 ? f : fo) / kGrp);
    p.bq = int(f / kGrp);
    p.nmma = ((p.N + 15) / 16) * 16;
    p.nchunks = int(ceil_div(kdim, 16));
    p.klast = int(ceil_div(2 * (kdim - 16 * (p.nchunks - 1)), 8));
    p.mtiles = mode == 2 ? 1 : int(ceil_div(Bn, 128));
    p.nob = int(ceil_div(p.N, 32));
    const uint32_t a_box = p.a_trans ? uint32_t(16 * p.aq * kGrp * 8) : BOX_BYTES;
    const uint32_t b_box = p.b_trans ? uint32_t(16 * p.bq * kGrp * 8) : BOX_BYTES;
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
    return Bn >= 128 && f <= 128 && fo <= 128 && f % 8 == 0 && fo % 8 == 0;
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
