// Memory-bound pointwise kernels: transfer edges (transfer.hpp:58-121), the
// loss gradient (taskgraph.hpp:116-126 + cross-entropy extension) and the
// SGD(+momentum) update (engine.hpp:795,800). All HBM-bound: grid-stride
// loops, vectorised where the layout allows, grids sized in multiples of the
// 148 SMs.
#include <algorithm>

#include "ops.hpp"

namespace znn_gpu {

namespace {

constexpr int kThreads = 256;

inline int grid_for(int64_t n, int per_thread = 1) {
    int64_t blocks = ceil_div(n, int64_t(kThreads) * per_thread);
    const int64_t cap = 148 * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    return int(blocks);
}

// grid: x over the voxels of one map, y/z over (patch, map) planes
__global__ void transfer_fwd_k(const float* __restrict__ x, int64_t f, int64_t vox, int64_t planes,
                               const int32_t* __restrict__ kinds, const float* __restrict__ bias,
                               float* __restrict__ y) {
    const int64_t plane = blockIdx.y + int64_t(blockIdx.z) * gridDim.y;
    const int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (plane >= planes || v >= vox) return;
    const int map = int(plane % f);
    const float b = bias ? bias[map] : 0.f;
    const int64_t i = plane * vox + v;
    y[i] = act_value(kinds[map], x[i] + b);
}

// grid (voxel chunks, map, patch): g * phi'(.) written to gx, each thread 4
// voxels strided by the block; per-block partial of the bias gradient written
// to part[(map * B + patch) * chunks + chunk].
constexpr int TB_E = 4;
__global__ void __launch_bounds__(kThreads) transfer_bwd_k(const float* __restrict__ g, const float* __restrict__ xy,
                                                           int from_output, int64_t B, int64_t f, int64_t vox,
                                                           const int32_t* __restrict__ kinds,
                                                           const float* __restrict__ bias, float* gx, float* part) {
    const int64_t map = blockIdx.y, bb = blockIdx.z;
    const int kind = kinds[map];
    const float b = bias ? bias[map] : 0.f;
    const int64_t off = (bb * f + map) * vox;
    float acc = 0.f;
    const int64_t v0 = int64_t(blockIdx.x) * (kThreads * TB_E) + threadIdx.x;
#pragma unroll
    for (int e = 0; e < TB_E; ++e) {
        const int64_t v = v0 + e * kThreads;
        if (v < vox) {
            const int64_t i = off + v;
            if (xy == nullptr) {  // gradient already gated (max-filter codes): bias gradient only
                acc += __ldg(g + i);
                continue;
            }
            const float yv = __ldcs(xy + i), gv = __ldcs(g + i);
            const float d = from_output ? act_deriv_out(kind, yv) : act_deriv_in(kind, yv + b);
            const float r = gv * d;
            __stcs(gx + i, r);
            acc += r;
        }
    }
    if (part) {
        __shared__ float red[kThreads / 32];
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x < 32) {
            float t = threadIdx.x < kThreads / 32 ? red[threadIdx.x] : 0.f;
            for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            if (threadIdx.x == 0) part[(map * B + bb) * gridDim.x + blockIdx.x] = t;
        }
    }
}

// Deterministic fixed-order reduction of per-block partials.
__global__ void reduce_rows_k(const float* __restrict__ part, int64_t rows, int64_t cols,
                              float* __restrict__ out) {
    const int64_t r = blockIdx.x;
    if (r >= rows) return;
    float acc = 0.f;
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) acc += part[r * cols + c];
    __shared__ float red[32];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        float t = threadIdx.x < (blockDim.x + 31) / 32 ? red[threadIdx.x] : 0.f;
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (threadIdx.x == 0) out[r] = t;
    }
}

__global__ void loss_k(int kind, const float* __restrict__ a, const float* __restrict__ d,
                       int64_t count, float scale, float* __restrict__ grad,
                       double* __restrict__ part) {
    double acc = 0.0;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count;
         i += int64_t(gridDim.x) * blockDim.x) {
        const float av = a[i], dv = d[i];
        const float e = av - dv;
        grad[i] = scale * e;
        if (kind == 0) {
            acc += 0.5 * double(e) * double(e);
        } else {
            // clamp keeps log finite for saturated logistic outputs
            const double p = fmin(fmax(double(av), 1e-30), 1.0 - 1e-16);
            acc -= double(dv) * log(p) + (1.0 - double(dv)) * log(1.0 - p);
        }
    }
    __shared__ double red[kThreads / 32];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = threadIdx.x < kThreads / 32 ? red[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (threadIdx.x == 0) part[blockIdx.x] = t;
    }
}

__global__ void sum_doubles_k(const double* __restrict__ part, int n, double* out) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) acc += part[i];
    __shared__ double red[32];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = threadIdx.x < (blockDim.x + 31) / 32 ? red[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (threadIdx.x == 0) *out = t;
    }
}

__global__ void sgd_k(float* __restrict__ w, float* __restrict__ v, const float* __restrict__ g,
                      int64_t count, float lr, float mu) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count;
         i += int64_t(gridDim.x) * blockDim.x) {
        const float nv = mu * v[i] + g[i];
        v[i] = nv;
        w[i] -= lr * nv;
    }
}

__global__ void zero_k(float* p, int64_t count) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count;
         i += int64_t(gridDim.x) * blockDim.x)
        p[i] = 0.f;
}

}  // namespace

void transfer_fwd(cudaStream_t st, const float* x, int64_t B, int64_t f, int64_t vox,
                  const int32_t* kinds_dev, const float* bias, float* y) {
    const int64_t planes = B * f;
    const int64_t gy = planes < 65535 ? (planes < 1 ? 1 : planes) : 65535;
    const dim3 grid(unsigned(ceil_div(vox, kThreads)), unsigned(gy), unsigned(ceil_div(planes, gy)));
    transfer_fwd_k<<<grid, kThreads, 0, st>>>(x, f, vox, planes, kinds_dev, bias, y);
    launch_check("transfer_fwd");
}

void transfer_bwd(cudaStream_t st, const float* g, const float* xy, bool from_output, int64_t B,
                  int64_t f, int64_t vox, const int32_t* kinds_dev, const float* bias,
                  float* gx, float* dbias, scratch& ws) {
    const int64_t chunks = ceil_div(vox, int64_t(kThreads) * TB_E);
    require(f < 65536 && B < 65536, "transfer_bwd: grid exceeds 65535 maps / patches");
    float* part = dbias ? static_cast<float*>(ws.get(sizeof(float) * size_t(f * B * chunks))) : nullptr;
    transfer_bwd_k<<<dim3(unsigned(chunks), unsigned(f), unsigned(B)), kThreads, 0, st>>>(
        g, xy, from_output ? 1 : 0, B, f, vox, kinds_dev, bias, gx, part);
    launch_check("transfer_bwd");
    if (dbias) {
        reduce_rows_k<<<unsigned(f), 128, 0, st>>>(part, f, B * chunks, dbias);
        launch_check("transfer_bwd_reduce");
    }
}

void reduce_rows(cudaStream_t st, const float* part, int64_t rows, int64_t cols, float* out) {
    reduce_rows_k<<<unsigned(rows), 128, 0, st>>>(part, rows, cols, out);
    launch_check("reduce_rows");
}

void loss_grad_async(cudaStream_t st, int kind, const float* a, const float* d, int64_t count,
                     float scale, float* grad, double* loss_dev, scratch& ws) {
    const int blocks = grid_for(count, 4);
    double* part = static_cast<double*>(ws.get(sizeof(double) * size_t(blocks)));
    loss_k<<<blocks, kThreads, 0, st>>>(kind, a, d, count, scale, grad, part);
    launch_check("loss");
    sum_doubles_k<<<1, 256, 0, st>>>(part, blocks, loss_dev);
    launch_check("loss_sum");
}

double loss_grad(cudaStream_t st, int kind, const float* a, const float* d, int64_t count,
                 float scale, float* grad, scratch& ws) {
    const int blocks = grid_for(count, 4);
    char* base = static_cast<char*>(ws.get(sizeof(double) * size_t(blocks + 1)));
    double* loss_dev = reinterpret_cast<double*>(base) + blocks;
    double* part = reinterpret_cast<double*>(base);
    loss_k<<<blocks, kThreads, 0, st>>>(kind, a, d, count, scale, grad, part);
    launch_check("loss");
    sum_doubles_k<<<1, 256, 0, st>>>(part, blocks, loss_dev);
    launch_check("loss_sum");
    double h = 0.0;
    ZNN_CUDA_CHECK(cudaMemcpyAsync(&h, loss_dev, sizeof(double), cudaMemcpyDeviceToHost, st));
    ZNN_CUDA_CHECK(cudaStreamSynchronize(st));
    return h;
}

void sgd_momentum(cudaStream_t st, float* w, float* v, const float* g, int64_t count, float lr,
                  float mu) {
    sgd_k<<<grid_for(count), kThreads, 0, st>>>(w, v, g, count, lr, mu);
    launch_check("sgd_momentum");
}

void fill_zero(cudaStream_t st, float* p, int64_t count) {
    zero_k<<<grid_for(count), kThreads, 0, st>>>(p, count);
    launch_check("fill_zero");
}

scratch::~scratch() {
    if (ptr_) cudaFree(ptr_);
}

void* scratch::get(size_t bytes) {
    if (bytes > cap_) {
        if (frozen_)
            throw cuda_error("scratch arena: " + std::to_string(bytes) + " bytes requested after the arena was "
                             "frozen at " + std::to_string(cap_) + " (steady state must not allocate)");
        if (ptr_) {
            ZNN_CUDA_CHECK(cudaDeviceSynchronize());
            void* old = ptr_;
            ptr_ = nullptr;  // consistent state even if the free or the new allocation fails
            cap_ = 0;
            ZNN_CUDA_CHECK(cudaFree(old));
        }
        const size_t want = bytes + bytes / 4 + 4096;
        dmalloc(&ptr_, want);
        cap_ = want;
        ++grows_;
    }
    return ptr_;
}

namespace {
struct prof_rec {
    std::string name;
    double bytes, flops;
    cudaEvent_t a, b;
};
struct profiler {
    bool on = false;
    std::vector<prof_rec> recs;
    std::vector<cudaEvent_t> spare;
    cudaEvent_t take() {
        if (!spare.empty()) {
            cudaEvent_t e = spare.back();
            spare.pop_back();
            return e;
        }
        cudaEvent_t e;
        ZNN_CUDA_CHECK(cudaEventCreate(&e));
        return e;
    }
};
profiler& prof() {
    static profiler p;
    return p;
}
}  // namespace

void prof_enable(bool on) { prof().on = on; }
bool prof_on() { return prof().on; }

prof_scope::prof_scope(cudaStream_t st, std::string name, double bytes, double flops) : st_(st) {
    profiler& P = prof();
    if (!P.on) return;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
    prof_rec r{std::move(name), bytes, flops, P.take(), P.take()};
    ZNN_CUDA_CHECK(cudaEventRecord(r.a, st));
    P.recs.push_back(std::move(r));
    slot_ = int(P.recs.size()) - 1;
}

prof_scope::~prof_scope() {
    if (slot_ >= 0) cudaEventRecord(prof().recs[size_t(slot_)].b, st_);
}

std::vector<prof_entry> prof_report() {
    profiler& P = prof();
    std::vector<prof_entry> out;
    for (auto& r : P.recs) {
        ZNN_CUDA_CHECK(cudaEventSynchronize(r.b));
        float ms = 0.f;
        ZNN_CUDA_CHECK(cudaEventElapsedTime(&ms, r.a, r.b));
        auto it = std::find_if(out.begin(), out.end(), [&](const prof_entry& e) { return e.name == r.name; });
        if (it == out.end()) {
            out.push_back(prof_entry{r.name, 0, 0, 0, 0});
            it = out.end() - 1;
        }
        it->launches++;
        it->ms += ms;
        it->bytes += r.bytes;
        it->flops += r.flops;
        P.spare.push_back(r.a);
        P.spare.push_back(r.b);
    }
    P.recs.clear();
    return out;
}

launch_stats& stats() {
    static launch_stats s;
    return s;
}

}  // namespace znn_gpu
