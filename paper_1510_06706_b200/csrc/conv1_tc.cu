// Forward of single-input-map layers (f_in = 1: the first layer of every
// config, conv_valid_direct conv_direct.hpp:39-68 with one source map) as a
// persistent tcgen05 implicit GEMM, 3xTF32.
//
// With one input map the GEMM K is just the kernel taps (<= 128), so the
// general kernel (conv_tc.cu: one CTA per 128-voxel tile, weight panels
// streamed per CTA) spends its time reloading the whole weight matrix for
// every tile. Here every CTA keeps the weights resident:
//   * B = W [f_out (<= 128 rows)][taps (<= 128)] split hi / lo once into the
//     canonical 128B-swizzled K-major layout in shared memory (<= 128 KB);
//   * A = the im2col tile: 8 producer warps gather each voxel's taps straight
//     from global memory (one voxel per TMEM lane, a warp's 32 voxels are
//     consecutive: every tap load is a coalesced 128-byte line, the source
//     map stays in L2), split hi / lo and write them into TMEM, one 32-tap
//     K-block slot at a time (4 slots, per-slot barriers);
//   * one MMA warp issues D += Ahi Bhi + Ahi Blo + Alo Bhi (A from TMEM);
//   * D is double-buffered in TMEM, so 4 epilogue warps add bias, apply the
//     transfer function and store (coalesced along voxels) while the next
//     tile accumulates.
// Measured (c5 conv1, 1 -> 120, 95^3, 5^3, B = 16): 6.8 ms vs 8.4 for the
// general kernel. Without the output stores it runs in 3.8 ms (MMAs ~29%
// busy: the per-slot TMEM fill / MMA round trips); the stores themselves are
// 128-byte pieces scattered over 120 output maps, which the DRAM serves at
// ~0.8 TB/s.
// TMEM: D buffers at columns [0, 128) / [128, 256), A slots (32 hi + 32 lo)
// at [256 + 64 kb, 320 + 64 kb).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "ops.hpp"
#include "tc_common.cuh"

namespace znn_gpu {

namespace {

using namespace znn_tc;

constexpr int C1_THREADS = 416;  // warps 0-7 producers, 8-11 epilogue, 12 MMA
constexpr int C1_KB = 4;         // 32-tap K-blocks (taps <= 128)
constexpr uint32_t C1_BBYTES = 128 * 128;  // one K-block of B: 128 rows x 32 floats
constexpr size_t C1_SMEM = 1024 + 2 * C1_KB * size_t(C1_BBYTES) + 2048;  // + barriers, tap offsets, bias

struct c1_params {
    int taps, nkb, f_out, nmma;
    int nx, ny, nz;       // source dims
    int mx, my, mz;       // output dims
    int64_t mvol, nvol;
    int64_t tiles_per_patch, ntiles;
    int act;
    int toff[128];        // tap offsets into the source map (sparse taps of a dilated kernel)
};

__device__ __forceinline__ void tmem_st16_c1(uint32_t addr, const float (&v)[16]) {
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
// 16 TMEM columns of this lane, loaded and waited in one asm statement
__device__ __forceinline__ void tmem_ld16_wait(uint32_t addr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr)
        : "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__global__ void __launch_bounds__(C1_THREADS, 1)
conv1_tc_k(const float* __restrict__ x, const float* __restrict__ w, const float* __restrict__ bias,
           float* __restrict__ y, const __grid_constant__ c1_params p) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* base_ptr = smem_raw + (base - raw);
    const uint32_t bhi = base, blo = base + C1_KB * C1_BBYTES;
    const uint32_t bar_base = base + 2 * C1_KB * C1_BBYTES;
    auto afull = [&](int kb) { return bar_base + 8u * uint32_t(kb); };
    auto aempty = [&](int kb) { return bar_base + 8u * uint32_t(C1_KB + kb); };
    auto accf = [&](int b) { return bar_base + 8u * uint32_t(2 * C1_KB + b); };
    auto acce = [&](int b) { return bar_base + 8u * uint32_t(2 * C1_KB + 2 + b); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base_ptr + (bar_base - base) + 8u * uint32_t(2 * C1_KB + 4));
    int* toff = reinterpret_cast<int*>(base_ptr + (bar_base - base) + 8u * uint32_t(2 * C1_KB + 4) + 16);
    float* sbias = reinterpret_cast<float*>(toff + 128);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // weights -> B hi / lo (128 rows x 128 taps, zero padded), tap offsets, bias
    for (int e = threadIdx.x; e < 128 * 128; e += C1_THREADS) {
        const int n = e >> 7, k = e & 127;
        const float v = (n < p.f_out && k < p.taps) ? __ldg(w + int64_t(n) * p.taps + k) : 0.f;
        const int kb = k >> 5, j = k & 31;
        const uint32_t o = uint32_t(kb) * C1_BBYTES + sw128_off(uint32_t(n), uint32_t(j));
        *reinterpret_cast<float*>(base_ptr + o) = v;
        *reinterpret_cast<float*>(base_ptr + C1_KB * C1_BBYTES + o) = v - tf32_hi(v);
    }
    for (int e = threadIdx.x; e < 128; e += C1_THREADS) {
        toff[e] = e < p.taps ? p.toff[e] : 0;
        sbias[e] = (bias && e < p.f_out) ? bias[e] : 0.f;
    }
    if (threadIdx.x == 0) {
        for (int kb = 0; kb < C1_KB; ++kb) {
            mbar_init(afull(kb), 4);  // the 4 lane-quarter warps filling the slot
            mbar_init(aempty(kb), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(accf(b), 1);
            mbar_init(acce(b), 4);
        }
        fence_barrier_init();
    }
    fence_proxy_async();  // weights written by the generic proxy -> tensor cores
    if (warp == 12) tmem_alloc(smem_u32(tmem_slot), 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < 8) {
        // ---- producers: warp w fills K-blocks kb = w / 4, w / 4 + 2 of its lane quarter ----
        const int q = warp & 3, h = warp >> 2;
        const int row = q * 32 + lane;
        const uint32_t lane_base = uint32_t(q * 32) << 16;
        int it = 0;
        for (int64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++it) {
            const int64_t b = t / p.tiles_per_patch;
            const int64_t v = (t - b * p.tiles_per_patch) * 128 + row;
            const bool ok = v < p.mvol;
            int64_t src = 0;
            if (ok) {
                const int64_t oxy = v / p.mz, oz = v - oxy * p.mz, ox = oxy / p.my, oy = oxy - ox * p.my;
                src = b * p.nvol + (ox * p.ny + oy) * p.nz + oz;
            }
            for (int kb = h; kb < p.nkb; kb += 2) {
                mbar_wait(aempty(kb), uint32_t(it & 1) ^ 1u);
                tc_fence_after();
                float hv[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const int tap = kb * 32 + j;
                    hv[j] = (ok && tap < p.taps) ? __ldg(x + src + toff[tap]) : 0.f;
                }
                const uint32_t a0 = tmem + lane_base + 256u + 64u * uint32_t(kb);
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    float vh[16], vl[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        vh[j] = hv[16 * half + j];
                        vl[j] = vh[j] - tf32_hi(vh[j]);
                    }
                    tmem_st16_c1(a0 + uint32_t(16 * half), vh);
                    tmem_st16_c1(a0 + 32u + uint32_t(16 * half), vl);
                }
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(afull(kb));
            }
        }
    } else if (warp == 12) {
        // ---- MMA issue ----
        const uint32_t idesc = idesc_tf32(128, p.nmma);
        int it = 0;
        for (int64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++it) {
            const int b = it & 1;
            mbar_wait(acce(b), uint32_t((it >> 1) & 1) ^ 1u);
            tc_fence_after();
            const uint32_t d = tmem + uint32_t(b) * 128u;
            for (int kb = 0; kb < p.nkb; ++kb) {
                mbar_wait(afull(kb), uint32_t(it & 1));
                tc_fence_after();
                const uint32_t a0 = tmem + 256u + 64u * uint32_t(kb);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const uint64_t bh = sw128_desc(bhi + uint32_t(kb) * C1_BBYTES + uint32_t(kk) * 32u);
                    const uint64_t bl = sw128_desc(blo + uint32_t(kb) * C1_BBYTES + uint32_t(kk) * 32u);
                    const uint32_t a = a0 + uint32_t(kk) * 8u;
                    const uint32_t acc = (kb == 0 && kk == 0) ? 0u : 1u;
                    mma_tf32_ts_w(d, a, bh, idesc, acc);
                    mma_tf32_ts_w(d, a, bl, idesc, 1u);
                    mma_tf32_ts_w(d, a + 32u, bh, idesc, 1u);
                }
                mma_commit_w(aempty(kb));
            }
            mma_commit_w(accf(b));
        }
    } else {
        // ---- epilogue: warps 8-11, lane = voxel of the tile ----
        const int q = warp & 3;
        const int row = q * 32 + lane;
        const uint32_t lane_base = uint32_t(q * 32) << 16;
        int it = 0;
        for (int64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++it) {
            const int bb = it & 1;
            const int64_t b = t / p.tiles_per_patch;
            const int64_t v = (t - b * p.tiles_per_patch) * 128 + row;
            const bool ok = v < p.mvol;
            mbar_wait(accf(bb), uint32_t((it >> 1) & 1));
            tc_fence_after();
            float* yb = y + b * int64_t(p.f_out) * p.mvol + v;
            for (int c0 = 0; c0 < p.f_out; c0 += 16) {
                float dv[16];
                tmem_ld16_wait(tmem + lane_base + uint32_t(bb) * 128u + uint32_t(c0), dv);
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int o = c0 + j;
                    if (ok && o < p.f_out) __stcs(yb + int64_t(o) * p.mvol, act_value(p.act, dv[j] + sbias[o]));
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acce(bb));
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 12) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

}  // namespace

bool conv1_tc_supported(const conv_shape& c) {
    return c.f_in == 1 && c.f_out >= 16 && c.f_out <= 128 && c.taps() <= 128 && c.n.vol() < (int64_t(1) << 31);
}

void conv1_fwd_tc(cudaStream_t st, const conv_shape& c, const float* x, const float* w, const float* bias, int act,
                  float* y) {
    require(conv1_tc_supported(c), "conv1_fwd_tc: layer unsupported");
    c1_params p{};
    p.taps = int(c.taps());
    p.nkb = int(ceil_div(c.taps(), 32));
    p.f_out = int(c.f_out);
    p.nmma = int(((c.f_out + 15) / 16) * 16);
    p.nx = int(c.n.x), p.ny = int(c.n.y), p.nz = int(c.n.z);
    p.mx = int(c.m.x), p.my = int(c.m.y), p.mz = int(c.m.z);
    p.mvol = c.m.vol(), p.nvol = c.n.vol();
    p.tiles_per_patch = ceil_div(p.mvol, 128);
    p.ntiles = p.tiles_per_patch * c.B;
    p.act = act;
    for (int wx = 0, t = 0; wx < c.k.x; ++wx)
        for (int wy = 0; wy < c.k.y; ++wy)
            for (int wz = 0; wz < c.k.z; ++wz, ++t)
                p.toff[t] = int((c.s.x * wx * c.n.y + c.s.y * wy) * c.n.z + c.s.z * wz);
    int dev = 0, sms = 148;
    ZNN_CUDA_CHECK(cudaGetDevice(&dev));
    ZNN_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const unsigned grid = unsigned(std::min<int64_t>(p.ntiles, sms));
    ZNN_CUDA_CHECK(cudaFuncSetAttribute(conv1_tc_k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C1_SMEM)));
    conv1_tc_k<<<grid, C1_THREADS, C1_SMEM, st>>>(x, w, bias, y, p);
    launch_check("conv1_fwd_tc");
}

}  // namespace znn_gpu
