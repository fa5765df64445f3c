// Issue-rate microbenchmark (profiling helper, not a test): legacy warp MMA
// m16n8k8 TF32 and FP32 FFMA throughput per SM on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void mma_k(float* out, int iters) {
    unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
    float c[8][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void fma_k(float* out, int iters) {
    float x[16];
    for (int j = 0; j < 16; ++j) x[j] = threadIdx.x * 0.001f + j;
    const float m = 0.9999f, a = 0.0001f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 16; ++j) x[j] = fmaf(x[j], m, a);
    }
    float s = 0;
    for (int j = 0; j < 16; ++j) s += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// 3-register FFMA: every operand a distinct live register (the CMAC's form)
__global__ void fma3_k(float* out, const float* __restrict__ in, int iters) {
    float x[16], y[4], z[4];
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = threadIdx.x * 0.001f + j;
#pragma unroll
    for (int j = 0; j < 4; ++j) y[j] = in[j], z[j] = in[4 + j];  // runtime values: no immediate folding
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 16; ++j) x[j] = fmaf(x[j], y[j & 3], z[(j >> 2) & 3]);
    }
    float s = 0;
    for (int j = 0; j < 16; ++j) s += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float* out;
    cudaMalloc(&out, 148 * 8 * 1024 * sizeof(float));
    float* in;
    cudaMalloc(&in, 8 * sizeof(float));
    const float h[8] = {0.9999f, 0.9998f, 0.9997f, 0.9996f, 1e-4f, 2e-4f, 3e-4f, 4e-4f};
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int warps : {4, 8, 16}) {
        const int iters = 20000, blocks = 148 * 4;
        mma_k<<<blocks, warps * 32>>>(out, 10);
        cudaEventRecord(e0);
        mma_k<<<blocks, warps * 32>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = double(blocks) * warps * iters * 8 * (16.0 * 8 * 8 * 2);
        printf("mma.sync m16n8k8 tf32: %d warps/CTA x %d CTAs: %.1f TFLOP/s\n", warps, blocks, flops / ms / 1e9);
    }
    for (int warps : {8, 16, 32}) {
        const int iters = 20000, blocks = 148 * 2;
        fma_k<<<blocks, warps * 32>>>(out, 10);
        cudaEventRecord(e0);
        fma_k<<<blocks, warps * 32>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = double(blocks) * warps * 32 * iters * 16 * 2.0;
        printf("ffma: %d warps/CTA x %d CTAs: %.1f TFLOP/s\n", warps, blocks, flops / ms / 1e9);
    }
    for (int warps : {16, 32}) {
        const int iters = 20000, blocks = 148 * 2;
        fma3_k<<<blocks, warps * 32>>>(out, in, 10);
        cudaEventRecord(e0);
        fma3_k<<<blocks, warps * 32>>>(out, in, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = double(blocks) * warps * 32 * iters * 16 * 2.0;
        printf("ffma 3-register: %d warps/CTA x %d CTAs: %.1f TFLOP/s\n", warps, blocks, flops / ms / 1e9);
    }
    return 0;
}
