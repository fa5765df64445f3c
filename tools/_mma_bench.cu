// Microbenchmark (profiling helper, not a test): tcgen05.mma kind::tf32
// issue rate with A in TMEM (TS) vs shared memory (SS), M=128, N in {64,128,256}.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1510_06706_b200/csrc tests/_mma_bench.cu -o /tmp/mma_bench
#include <cstdio>

#include "tc_common.cuh"

using namespace znn_tc;

template <bool TS>
__global__ void __launch_bounds__(384, 1) mma_loop(int iters, int n, float* sink, int mode) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint32_t slot;
    __shared__ uint64_t bar, bar2[4];
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    if (threadIdx.x < 32) tmem_alloc(smem_u32(&slot), 512);
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar), 1);
        for (int i = 0; i < 4; ++i) mbar_init(smem_u32(&bar2[i]), 1);
        fence_barrier_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    volatile __shared__ int stop;
    if (threadIdx.x == 0) stop = 0;
    __syncthreads();
    if (threadIdx.x >= 128 && (mode & 2)) {
        // producers: keep writing TMEM columns [448, 512) of their lane quarter
        const uint32_t lb = uint32_t(((threadIdx.x >> 5) & 3) * 32) << 16;
        float h[8];
        for (int q = 0; q < 8; ++q) h[q] = float(threadIdx.x + q);
        while (!stop) {
            for (int c = 0; c < 8; ++c) tmem_st8(tmem + lb + 448u + 8u * c, h);
            tmem_wait_st();
            if (mode & 8) {
                float v[16];
                for (int c = 0; c < 4; ++c) {
                    tmem_ld16(tmem + lb + 128u + 16u * c, v);
                    tmem_wait_ld();
                    h[c] += v[c];
                }
            }
        }
    }
    if (threadIdx.x < 32 && (mode & 16)) {  // converged warp, elect-predicated issue
        const uint32_t idesc = idesc_tf32(128, n);
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const uint64_t b = sw128_desc(base + 32u * kk);
                mma_tf32_ts_w(tmem, tmem + 256u + 8u * kk, b, idesc, 1u);
                if (mode & 4) {
                    mma_tf32_ts_w(tmem, tmem + 256u + 8u * kk, sw128_desc(base + 32u * kk), idesc, 1u);
                    mma_tf32_ts_w(tmem, tmem + 256u + 8u * kk, sw128_desc(base + 32u * kk), idesc, 1u);
                }
            }
            if (mode & 1) {
                mma_commit_w(smem_u32(&bar2[i & 3]));
                mma_commit_w(smem_u32(&bar2[(i + 1) & 3]));
            }
        }
        mma_commit_w(smem_u32(&bar));
        mbar_wait(smem_u32(&bar), 0);
        if (threadIdx.x == 0) stop = 1;
    } else if (threadIdx.x == 0) {
        const uint32_t idesc = idesc_tf32(128, n);
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const uint64_t b = sw128_desc(base + 32u * kk);
                if (TS) {
                    mma_tf32_ts(tmem, tmem + 256u + 8u * kk, b, idesc, 1u);
                } else {
                    const uint64_t a = sw128_desc(base + 65536u + 32u * kk);
                    mma_tf32(tmem, a, b, idesc, 1u);
                }
                if (mode & 4) {  // 3 MMAs per K-step like the conv kernels
                    mma_tf32_ts(tmem, tmem + 256u + 8u * kk, sw128_desc(base + 32u * kk), idesc, 1u);
                    mma_tf32_ts(tmem, tmem + 256u + 8u * kk, sw128_desc(base + 32u * kk), idesc, 1u);
                }
            }
            if (mode & 1) {
                mma_commit(smem_u32(&bar2[i & 3]));
                mma_commit(smem_u32(&bar2[(i + 1) & 3]));
            }
        }
        mma_commit(smem_u32(&bar));
        mbar_wait(smem_u32(&bar), 0);
        stop = 1;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
    if (threadIdx.x == 0 && iters < 0) sink[0] = 1.f;
}

int main() {
    float* sink;
    cudaMalloc(&sink, 4);
    const int iters = 20000;
    for (int mode : {0, 1, 3, 4, 5, 7, 16, 17, 19, 20, 21, 23})
    for (int ts = 1; ts < 2; ++ts)
        for (int n : {128}) {
            auto k = ts ? mma_loop<true> : mma_loop<false>;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
            k<<<148, 384, 140 * 1024>>>(100, n, sink, mode);
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            k<<<148, 384, 140 * 1024>>>(iters, n, sink, mode);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double macs = 148.0 * iters * 4 * 128.0 * n * 8 * ((mode & 4) ? 3 : 1);
            const double clk = ms * 1e-3 * 1.965e9;
            printf("mode %d %s N=%3d: %.3f ms, %.1f tf32 TFLOP/s, %.1f clk per MMA per SM (floor %d)\n", mode, ts ? "TS" : "SS", n,
                   ms, 2 * macs / (ms * 1e-3) / 1e12, clk / (iters * 4.0 * ((mode & 4) ? 3 : 1)), 128 * n / 256);
        }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
