// extern "C" entry points beyond the per-op / executor core (capi.cpp):
//   * the FFT engine per layer (conv_fft.hpp:25-192 + fft.hpp:57-192)
//   * the per-layer autotuner (trainer.hpp:181-250)
//   * NCCL data parallelism: communicator, allreduce, and the
//     data-parallel step with a per-layer bucketed allreduce overlapped with
//     the rest of the backward pass
//   * CUDA-graph replay of the training step and library memory counters
//   * ZNNV volume I/O (volume_io.hpp:15-86) and the data provider
//     (trainer.hpp:87-166) with pinned, double-buffered asynchronous H2D
#include <cuda_runtime.h>
#include <dirent.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "capi_internal.hpp"
#include "fft.hpp"

using znn_capi::D;
using znn_capi::guarded;

struct znn_fft_plan_s {
    znn_ctx ctx = nullptr;
    znn_gpu::conv_shape c;
    znn_fft::plan_ptr p;
    bool memo = false;  // a forward has memoised X and K
};

namespace {

// ---------------------------------------------------------------- NCCL --
// libnccl is resolved at run time (dlopen), so the library has no link-time
// NCCL dependency and shares the copy torch already loaded when there is one.
struct nccl_api {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const nccl_api& nccl() {
    static nccl_api api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    });
    if (!api.get_unique_id || !api.comm_init_rank || !api.all_reduce || !api.comm_destroy)
        throw znn_gpu::cuda_error("NCCL (libnccl.so.2) not found");
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw znn_gpu::cuda_error(std::string(what) + ": " +
                                  (nccl().error_string ? nccl().error_string(r) : "nccl error"));
}

}  // namespace

struct znn_comm_s {
    znn_ctx ctx = nullptr;
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0;
    cudaStream_t cs = nullptr;            // communication stream (allreduce overlaps compute)
    std::vector<cudaEvent_t> ready;       // per-bucket "gradient final" events
    cudaEvent_t done = nullptr;
    ~znn_comm_s() {
        for (auto e : ready) cudaEventDestroy(e);
        if (done) cudaEventDestroy(done);
        if (cs) cudaStreamDestroy(cs);
        if (comm) nccl().comm_destroy(comm);
    }
    // in-place sum of [p, p + n) once everything issued so far on `st` has run
    void allreduce_after(cudaStream_t st, float* p, int64_t n, size_t bucket) {
        while (ready.size() <= bucket) {
            cudaEvent_t e;
            ZNN_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            ready.push_back(e);
        }
        ZNN_CUDA_CHECK(cudaEventRecord(ready[bucket], st));
        ZNN_CUDA_CHECK(cudaStreamWaitEvent(cs, ready[bucket], 0));
        nccl_check(nccl().all_reduce(p, p, size_t(n), ncclFloat32, ncclSum, comm, cs), "ncclAllReduce");
    }
    // `st` waits for every allreduce issued so far
    void join(cudaStream_t st) {
        ZNN_CUDA_CHECK(cudaEventRecord(done, cs));
        ZNN_CUDA_CHECK(cudaStreamWaitEvent(st, done, 0));
    }
};

// ------------------------------------------------------- data provider --
namespace {

// ZNNV: magic "ZNNV", u32 version 1, u32 nx, ny, nz, then float32 x-major
// (volume_io.hpp:15-86); all little-endian.
constexpr char kMagic[4] = {'Z', 'N', 'N', 'V'};

void put_u32(std::ofstream& os, uint32_t v) {
    const unsigned char b[4] = {static_cast<unsigned char>(v), static_cast<unsigned char>(v >> 8),
                                static_cast<unsigned char>(v >> 16), static_cast<unsigned char>(v >> 24)};
    os.write(reinterpret_cast<const char*>(b), 4);
}
uint32_t get_u32(std::ifstream& is) {
    unsigned char b[4] = {0, 0, 0, 0};
    is.read(reinterpret_cast<char*>(b), 4);
    return uint32_t(b[0]) | (uint32_t(b[1]) << 8) | (uint32_t(b[2]) << 16) | (uint32_t(b[3]) << 24);
}

// header only (dims), or header + payload into data[0 .. capacity)
void read_znnv(const std::string& path, int64_t dims[3], float* data, int64_t capacity) {
    std::ifstream is(path, std::ios::binary);
    znn_gpu::require(is.good(), "cannot open for reading: " + path);
    char m[4] = {0, 0, 0, 0};
    is.read(m, 4);
    znn_gpu::require(is.good() && std::memcmp(m, kMagic, 4) == 0, "volume file: bad magic bytes");
    const uint32_t ver = get_u32(is);
    znn_gpu::require(ver == 1, "volume file: unsupported version " + std::to_string(ver));
    for (int a = 0; a < 3; ++a) dims[a] = int64_t(get_u32(is));
    znn_gpu::require(is.good() && dims[0] > 0 && dims[1] > 0 && dims[2] > 0, "volume file: non-positive dims");
    if (!data) return;
    const int64_t n = dims[0] * dims[1] * dims[2];
    znn_gpu::require(n <= capacity, "volume file " + path + ": payload larger than the buffer");
    // the payload is little-endian float32: on x86 a straight read
    is.read(reinterpret_cast<char*>(data), std::streamsize(sizeof(float) * size_t(n)));
    znn_gpu::require(is.good(), "volume file: truncated payload");
}

void write_znnv(const std::string& path, const int64_t dims[3], const float* data) {
    std::ofstream os(path, std::ios::binary);
    znn_gpu::require(os.good(), "cannot open for writing: " + path);
    for (int a = 0; a < 3; ++a)
        znn_gpu::require(dims[a] > 0 && dims[a] < (int64_t(1) << 32), "volume file: bad dims");
    os.write(kMagic, 4);
    put_u32(os, 1);
    for (int a = 0; a < 3; ++a) put_u32(os, uint32_t(dims[a]));
    os.write(reinterpret_cast<const char*>(data), std::streamsize(sizeof(float) * size_t(dims[0] * dims[1] * dims[2])));
    znn_gpu::require(os.good(), "volume file: write failed: " + path);
}

std::vector<std::string> sorted_files(const std::string& dir) {
    std::vector<std::string> out;
    DIR* d = opendir(dir.c_str());
    znn_gpu::require(d != nullptr, "data directory missing: " + dir);
    while (dirent* e = readdir(d)) {
        const std::string n = e->d_name;
        if (n == "." || n == "..") continue;
        out.push_back(dir + "/" + n);
    }
    closedir(d);
    std::sort(out.begin(), out.end());
    return out;
}

}  // namespace

// One batch = B patches; patch b of step t is sample (t * stride + offset + b)
// mod size (the reference's source(round) = samples[(round - 1) % size],
// trainer.hpp:152-156, with `stride` = global batch for data parallelism).
// The same volume feeds every input node and the same label every output
// node, as the reference's from_files provider does (trainer.hpp:140-145).
// Two pinned host slots and two device slots: a worker thread reads step
// t + 1's files and issues its H2D on a copy stream while step t computes.
struct znn_loader_s {
    znn_net net = nullptr;
    int64_t B = 1, offset = 0, stride = 1, in_maps = 1, out_maps = 1, in_vol = 1, out_vol = 1;
    // file source, or an in-memory (pinned) source
    std::vector<std::string> in_files, lab_files;
    const float* mem_in = nullptr;
    const float* mem_lab = nullptr;
    int64_t samples = 0;
    float* h_in[2] = {nullptr, nullptr};
    float* h_lab[2] = {nullptr, nullptr};
    float* d_in[2] = {nullptr, nullptr};
    float* d_lab[2] = {nullptr, nullptr};
    cudaStream_t cs = nullptr;
    cudaEvent_t ready[2] = {nullptr, nullptr}, consumed[2] = {nullptr, nullptr};
    int64_t step = 0;           // next step to run
    std::thread worker;
    std::string worker_err;
    bool issued[2] = {false, false};

    ~znn_loader_s() {
        if (worker.joinable()) worker.join();
        for (int i = 0; i < 2; ++i) {
            if (h_in[i]) cudaFreeHost(h_in[i]);
            if (h_lab[i]) cudaFreeHost(h_lab[i]);
            if (d_in[i]) cudaFree(d_in[i]);
            if (d_lab[i]) cudaFree(d_lab[i]);
            if (ready[i]) cudaEventDestroy(ready[i]);
            if (consumed[i]) cudaEventDestroy(consumed[i]);
        }
        if (cs) cudaStreamDestroy(cs);
    }

    int64_t sample_of(int64_t t, int64_t b) const { return (t * stride + offset + b) % samples; }

    // host side of step t into slot t % 2, then its H2D on the copy stream
    void stage(int64_t t) {
        const int slot = int(t & 1);
        const size_t inb = sizeof(float) * size_t(in_vol), lab_b = sizeof(float) * size_t(out_vol);
        ZNN_CUDA_CHECK(cudaStreamWaitEvent(cs, consumed[slot], 0));  // step t - 2 done with the device slot
        if (mem_in) {  // in-memory source: straight from the caller's (pinned) samples
            for (int64_t b = 0; b < B; ++b) {
                const int64_t smp = sample_of(t, b);
                ZNN_CUDA_CHECK(cudaMemcpyAsync(d_in[slot] + b * in_maps * in_vol, mem_in + smp * in_maps * in_vol,
                                               inb * size_t(in_maps), cudaMemcpyHostToDevice, cs));
                ZNN_CUDA_CHECK(cudaMemcpyAsync(d_lab[slot] + b * out_maps * out_vol,
                                               mem_lab + smp * out_maps * out_vol, lab_b * size_t(out_maps),
                                               cudaMemcpyHostToDevice, cs));
            }
        } else {
            // the previous H2D out of this host slot (step t - 2) must be done
            ZNN_CUDA_CHECK(cudaEventSynchronize(ready[slot]));
            int64_t dims[3];
            for (int64_t b = 0; b < B; ++b) {
                const int64_t smp = sample_of(t, b);
                float* hi = h_in[slot] + b * in_maps * in_vol;
                float* hl = h_lab[slot] + b * out_maps * out_vol;
                read_znnv(in_files[size_t(smp)], dims, hi, in_vol);
                znn_gpu::require(dims[0] * dims[1] * dims[2] == in_vol,
                                 "input volume " + in_files[size_t(smp)] + " does not match the net's input dims");
                read_znnv(lab_files[size_t(smp)], dims, hl, out_vol);
                znn_gpu::require(dims[0] * dims[1] * dims[2] == out_vol,
                                 "label volume " + lab_files[size_t(smp)] + " does not match the net's output dims");
                for (int64_t m = 1; m < in_maps; ++m) std::memcpy(hi + m * in_vol, hi, inb);
                for (int64_t m = 1; m < out_maps; ++m) std::memcpy(hl + m * out_vol, hl, lab_b);
            }
            ZNN_CUDA_CHECK(cudaMemcpyAsync(d_in[slot], h_in[slot], inb * size_t(B * in_maps), cudaMemcpyHostToDevice, cs));
            ZNN_CUDA_CHECK(cudaMemcpyAsync(d_lab[slot], h_lab[slot], lab_b * size_t(B * out_maps),
                                           cudaMemcpyHostToDevice, cs));
        }
        ZNN_CUDA_CHECK(cudaEventRecord(ready[slot], cs));
        issued[slot] = true;
    }

    void prefetch(int64_t t, int device) {
        if (worker.joinable()) worker.join();
        worker_err.clear();
        worker = std::thread([this, t, device] {
            try {
                cudaSetDevice(device);
                stage(t);
            } catch (const std::exception& e) {
                worker_err = e.what();
            }
        });
    }

    void wait_worker() {
        if (worker.joinable()) worker.join();
        if (!worker_err.empty()) {
            const std::string e = worker_err;
            worker_err.clear();
            throw znn_gpu::cuda_error("data provider: " + e);
        }
    }
};

namespace {

void loader_alloc(znn_loader_s* L, znn_net net, int64_t offset) {
    L->net = net;
    L->B = 0;
    znn_exec::executor& ex = *net->ex;
    const auto& gi = ex.grp(0);
    const auto& go = ex.grp(ex.num_groups() - 1);
    L->in_maps = gi.maps, L->in_vol = gi.dims.vol();
    L->out_maps = go.maps, L->out_vol = go.dims.vol();
    L->B = ex.batch();
    L->stride = ex.global_batch();
    L->offset = offset;
    for (int i = 0; i < 2; ++i) {
        if (!L->mem_in) {
            ZNN_CUDA_CHECK(cudaHostAlloc(&L->h_in[i], sizeof(float) * size_t(L->B * L->in_maps * L->in_vol), 0));
            ZNN_CUDA_CHECK(cudaHostAlloc(&L->h_lab[i], sizeof(float) * size_t(L->B * L->out_maps * L->out_vol), 0));
        }
        znn_gpu::dmalloc(&L->d_in[i], sizeof(float) * size_t(L->B * L->in_maps * L->in_vol));
        znn_gpu::dmalloc(&L->d_lab[i], sizeof(float) * size_t(L->B * L->out_maps * L->out_vol));
        ZNN_CUDA_CHECK(cudaEventCreateWithFlags(&L->ready[i], cudaEventDisableTiming));
        ZNN_CUDA_CHECK(cudaEventCreateWithFlags(&L->consumed[i], cudaEventDisableTiming));
    }
    ZNN_CUDA_CHECK(cudaStreamCreateWithFlags(&L->cs, cudaStreamNonBlocking));
}

}  // namespace

extern "C" {

// ----------------------------------------------------------- FFT engine --
int znn_fft_plan_create(znn_ctx ctx, int64_t B, int64_t f_in, int64_t f_out, const int64_t n[3], const int64_t k[3],
                        const int64_t s[3], znn_fft_plan* out) {
    return guarded(ctx, [&] {
        if (!out) throw znn_gpu::shape_error("znn_fft_plan_create: null out");
        auto c = znn_gpu::conv_shape::make(B, f_in, f_out, D(n), D(k), D(s));
        auto* p = new znn_fft_plan_s;
        p->ctx = ctx;
        p->c = c;
        try {
            p->p = znn_fft::make_plan(c);
        } catch (...) {
            delete p;
            throw;
        }
        *out = p;
    });
}

int znn_fft_plan_destroy(znn_fft_plan p) {
    if (!p) return ZNN_OK;
    cudaSetDevice(p->ctx->device);
    delete p;
    return ZNN_OK;
}

int znn_fft_plan_info(znn_fft_plan p, int64_t pads[3], int64_t* bins, int64_t* kernel_spectrum_bytes) {
    if (!p) return ZNN_ERR_SHAPE;
    return guarded(p->ctx, [&] {
        int64_t P[3];
        znn_fft::pad_dims(*p->p, P);
        if (pads) pads[0] = P[0], pads[1] = P[1], pads[2] = P[2];
        if (bins) *bins = P[0] * P[1] * (P[2] / 2 + 1);
        if (kernel_spectrum_bytes) *kernel_spectrum_bytes = znn_fft::kernel_spectrum_bytes(p->c);
    });
}

int znn_fft_conv_fwd(znn_fft_plan p, const float* x, const float* w, const float* bias, int act, float* y) {
    if (!p) return ZNN_ERR_SHAPE;
    return guarded(p->ctx, [&] {
        if (act < 0 || act > 3) throw znn_gpu::shape_error("fft conv: unknown transfer kind");
        znn_fft::conv_fwd(p->ctx->stream, *p->p, p->c, x, w, bias, act, y, p->ctx->ws);
        p->memo = true;
    });
}

int znn_fft_conv_bwd(znn_fft_plan p, const float* g, const float* w, float* dw, float* dx) {
    if (!p) return ZNN_ERR_SHAPE;
    return guarded(p->ctx, [&] {
        if (!p->memo) throw znn_gpu::shape_error("fft conv backward: no memoised spectra (run znn_fft_conv_fwd first)");
        if (!dw) throw znn_gpu::shape_error("fft conv backward: dw is required");
        znn_fft::conv_bwd(p->ctx->stream, *p->p, p->c, nullptr, g, w, dw, dx, p->ctx->ws);
        p->memo = false;  // dK reused the kernel-spectrum buffer
    });
}

int znn_fft_plan_counts(znn_fft_plan p, int64_t out[9]) {
    if (!p) return ZNN_ERR_SHAPE;
    return guarded(p->ctx, [&] {
        const auto& t = znn_fft::counts(*p->p);
        const int64_t v[9] = {t.fwd_image, t.fwd_kernel, t.fwd_inverse, t.bwd_image, t.bwd_kernel,
                              t.bwd_inverse, t.upd_image, t.upd_kernel, t.upd_inverse};
        for (int i = 0; i < 9; ++i) out[i] = v[i];
    });
}

// ------------------------------------------------------------ autotune --
int znn_autotune_layer(znn_ctx ctx, int64_t B, int64_t f_in, int64_t f_out, const int64_t n[3], const int64_t k[3],
                       const int64_t s[3], int trials, int* chosen, float ms_out[3]) {
    return guarded(ctx, [&] {
        if (trials < 1) throw znn_gpu::shape_error("autotune: trials must be >= 1");
        const auto c = znn_gpu::conv_shape::make(B, f_in, f_out, D(n), D(k), D(s));
        cudaStream_t st = ctx->stream;
        float *x = nullptr, *w = nullptr, *g = nullptr, *dx = nullptr, *dw = nullptr;
        const size_t nx = size_t(c.B * c.f_in * c.n.vol()), nw = size_t(c.f_out * c.f_in * c.taps()),
                     ng = size_t(c.B * c.f_out * c.m.vol());
        znn_gpu::dmalloc(&x, sizeof(float) * nx);
        znn_gpu::dmalloc(&w, sizeof(float) * nw);
        znn_gpu::dmalloc(&g, sizeof(float) * ng);
        znn_gpu::dmalloc(&dx, sizeof(float) * nx);
        znn_gpu::dmalloc(&dw, sizeof(float) * nw);
        struct freer {
            std::vector<void*> v;
            ~freer() {
                for (void* p : v) cudaFree(p);
            }
        } fr{{x, w, g, dx, dw}};
        // finite synthetic values (0x3c3c3c3c = 0.0115f): the timing is value-independent
        ZNN_CUDA_CHECK(cudaMemsetAsync(x, 0x3c, sizeof(float) * nx, st));
        ZNN_CUDA_CHECK(cudaMemsetAsync(w, 0x3c, sizeof(float) * nw, st));
        ZNN_CUDA_CHECK(cudaMemsetAsync(g, 0x3c, sizeof(float) * ng, st));
        float res[3] = {-1.f, -1.f, -1.f};
        cudaEvent_t a, b;
        ZNN_CUDA_CHECK(cudaEventCreate(&a));
        ZNN_CUDA_CHECK(cudaEventCreate(&b));
        std::unique_ptr<znn_fft::plan, znn_fft::plan_deleter> plan;
        auto run = [&](int e) {
            if (e == ZNN_CONV_FFT) {
                znn_fft::conv_fwd(st, *plan, c, x, w, nullptr, ZNN_ACT_RELU, dx, ctx->ws);
                znn_fft::conv_bwd(st, *plan, c, x, g, w, dw, c.f_in > 1 ? dx : nullptr, ctx->ws);
            } else if (e == ZNN_CONV_DIRECT) {
                znn_gpu::conv_fwd_tc(st, c, x, w, nullptr, ZNN_ACT_RELU, dx, ctx->ws);
                if (c.f_in > 1) znn_gpu::conv_dgrad_tc(st, c, g, w, dx, ctx->ws);
                znn_gpu::conv_wgrad_tc(st, c, x, g, dw, 1.f, ctx->ws);
            } else {
                znn_gpu::conv_fwd_simt(st, c, x, w, nullptr, ZNN_ACT_RELU, dx);
                if (c.f_in > 1) znn_gpu::conv_dgrad_simt(st, c, g, w, dx);
                znn_gpu::conv_wgrad_simt(st, c, x, g, dw, 1.f, ctx->ws);
            }
        };
        std::vector<int> cands;
        if (znn_gpu::conv_tc_supported(c, 0) && znn_gpu::conv_tc_supported(c, 2) &&
            (c.f_in == 1 || znn_gpu::conv_tc_supported(c, 1)))
            cands.push_back(ZNN_CONV_DIRECT);
        if (znn_fft::supported(c)) cands.push_back(ZNN_CONV_FFT);
        if (c.f_in * c.f_out <= 1024 || cands.empty()) cands.push_back(ZNN_CONV_DIRECT_SIMT);
        float best = 1e30f;
        int best_e = cands.front();
        for (int e : cands) {
            try {
                if (e == ZNN_CONV_FFT) plan = znn_fft::make_plan(c);
                std::vector<float> ts;
                for (int t = 0; t <= trials; ++t) {  // run 0 warms plans and scratch
                    ZNN_CUDA_CHECK(cudaEventRecord(a, st));
                    run(e);
                    ZNN_CUDA_CHECK(cudaEventRecord(b, st));
                    ZNN_CUDA_CHECK(cudaEventSynchronize(b));
                    float ms = 0.f;
                    ZNN_CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
                    if (t > 0) ts.push_back(ms);
                    if (t == 1 && ms > 4.f * best) break;  // cannot win
                }
                plan.reset();
                std::sort(ts.begin(), ts.end());
                const float med = ts[ts.size() / 2];
                res[e == ZNN_CONV_DIRECT ? 0 : e == ZNN_CONV_FFT ? 1 : 2] = med;
                if (med < best) best = med, best_e = e;
            } catch (const std::exception&) {
                plan.reset();
                cudaGetLastError();
                cudaStreamSynchronize(st);
            }
        }
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        if (chosen) *chosen = best_e;
        if (ms_out)
            for (int i = 0; i < 3; ++i) ms_out[i] = res[i];
    });
}

// ---------------------------------------------------------------- NCCL --
int znn_comm_unique_id(void* id) {
    return guarded(nullptr, [&] {
        if (!id) throw znn_gpu::shape_error("znn_comm_unique_id: null buffer");
        ncclUniqueId u;
        nccl_check(nccl().get_unique_id(&u), "ncclGetUniqueId");
        std::memcpy(id, &u, sizeof(u));
    });
}

int znn_comm_create(znn_ctx ctx, const void* id, int nranks, int rank, znn_comm* out) {
    return guarded(ctx, [&] {
        if (!id || !out) throw znn_gpu::shape_error("znn_comm_create: null argument");
        if (nranks < 1 || rank < 0 || rank >= nranks) throw znn_gpu::shape_error("znn_comm_create: bad rank");
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        auto* c = new znn_comm_s;
        c->ctx = ctx;
        c->nranks = nranks;
        c->rank = rank;
        try {
            nccl_check(nccl().comm_init_rank(&c->comm, nranks, u, rank), "ncclCommInitRank");
            ZNN_CUDA_CHECK(cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking));
            ZNN_CUDA_CHECK(cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming));
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

int znn_comm_destroy(znn_comm comm) {
    if (!comm) return ZNN_OK;
    cudaSetDevice(comm->ctx->device);
    delete comm;
    return ZNN_OK;
}

int znn_allreduce(znn_comm comm, float* buf, int64_t count) {
    if (!comm) return ZNN_ERR_SHAPE;
    return guarded(comm->ctx, [&] {
        cudaStream_t st = comm->ctx->stream;
        comm->allreduce_after(st, buf, count, 0);
        comm->join(st);
    });
}

int znn_net_train_step_dp(znn_net net, znn_comm comm, const float* inputs_dev, const float* labels_dev,
                          double* loss) {
    if (!net || !comm) return ZNN_ERR_SHAPE;
    return guarded(net->ctx, [&] {
        znn_exec::executor& ex = *net->ex;
        cudaStream_t st = net->ctx->stream;
        ex.set_stream(st);
        float* gbuf = ex.grad_buffer();
        size_t bucket = 0;
        // one bucket per layer, issued in backward order as soon as the
        // layer's gradient slice is final: the allreduce of layer l runs on
        // the communication stream under the backward of layers < l
        ex.set_grad_hook([&](int64_t off, int64_t cnt) { comm->allreduce_after(st, gbuf + off, cnt, bucket++); });
        double l = 0.0;
        try {
            l = ex.forward_backward(inputs_dev, labels_dev, false, false);
        } catch (...) {
            ex.set_grad_hook(nullptr);
            throw;
        }
        ex.set_grad_hook(nullptr);
        comm->join(st);
        ex.apply_update();
        if (loss) *loss = ex.last_loss_device();
        (void)l;
    });
}

// ------------------------------------------------ graph / memory counters --
int znn_net_set_graph(znn_net net, int on) {
    if (!net) return ZNN_ERR_SHAPE;
    return guarded(net->ctx, [&] { net->ex->set_graph_mode(on != 0); });
}

int znn_net_graph_captured(znn_net net, int* yes) {
    if (!net) return ZNN_ERR_SHAPE;
    return guarded(net->ctx, [&] {
        if (yes) *yes = net->ex->graph_captured() ? 1 : 0;
    });
}

int znn_mem_stats(znn_ctx ctx, int64_t out[4]) {
    return guarded(ctx, [&] {
        size_t fr = 0, tot = 0;
        ZNN_CUDA_CHECK(cudaMemGetInfo(&fr, &tot));
        out[0] = int64_t(fr);
        out[1] = int64_t(tot);
        out[2] = znn_gpu::stats().allocs;
        out[3] = znn_gpu::stats().alloc_bytes;
    });
}

int znn_profile_enable(znn_ctx ctx, int on) {
    return guarded(ctx, [&] { znn_gpu::prof_enable(on != 0); });
}

int znn_profile_report(znn_ctx ctx, char* buf, int64_t len) {
    return guarded(ctx, [&] {
        std::string j = "[";
        bool first = true;
        for (const auto& e : znn_gpu::prof_report()) {
            char tmp[160];
            std::snprintf(tmp, sizeof(tmp), "\", \"launches\": %lld, \"ms\": %.6f, \"bytes\": %.6e, \"flops\": %.6e}",
                          (long long)e.launches, e.ms, e.bytes, e.flops);
            j += std::string(first ? "" : ", ") + "{\"kernel\": \"" + e.name + tmp;
            first = false;
        }
        j += "]";
        if (!buf || len < int64_t(j.size()) + 1) throw znn_gpu::shape_error("profile report: buffer too small");
        std::memcpy(buf, j.c_str(), j.size() + 1);
    });
}

// ----------------------------------------------------- volumes / loader --
int znn_volume_write(const char* path, const int64_t dims[3], const float* data) {
    return guarded(nullptr, [&] {
        if (!path || !dims || !data) throw znn_gpu::shape_error("znn_volume_write: null argument");
        write_znnv(path, dims, data);
    });
}

int znn_volume_read(const char* path, int64_t dims[3], float* data, int64_t capacity) {
    return guarded(nullptr, [&] {
        if (!path || !dims) throw znn_gpu::shape_error("znn_volume_read: null argument");
        read_znnv(path, dims, data, capacity);
    });
}

int znn_loader_open_dir(znn_net net, const char* dir, int64_t shard_offset, znn_loader* out) {
    if (!net) return ZNN_ERR_SHAPE;
    return guarded(net->ctx, [&] {
        if (!dir || !out) throw znn_gpu::shape_error("znn_loader_open_dir: null argument");
        auto ins = sorted_files(std::string(dir) + "/inputs");
        auto labs = sorted_files(std::string(dir) + "/labels");
        if (ins.empty() || ins.size() != labs.size())
            throw znn_gpu::shape_error("data directory needs matching inputs/ and labels/ files");
        auto* L = new znn_loader_s;
        L->in_files = std::move(ins);
        L->lab_files = std::move(labs);
        L->samples = int64_t(L->in_files.size());
        try {
            loader_alloc(L, net, shard_offset);
            // validate the first pair's dims against the net (trainer.hpp:132-139)
            int64_t d[3];
            read_znnv(L->in_files[0], d, nullptr, 0);
            const auto& gi = net->ex->grp(0);
            const auto& go = net->ex->grp(net->ex->num_groups() - 1);
            if (d[0] != gi.dims.x || d[1] != gi.dims.y || d[2] != gi.dims.z)
                throw znn_gpu::shape_error("input volume " + L->in_files[0] + " does not match the net's input dims");
            read_znnv(L->lab_files[0], d, nullptr, 0);
            if (d[0] != go.dims.x || d[1] != go.dims.y || d[2] != go.dims.z)
                throw znn_gpu::shape_error("label volume " + L->lab_files[0] + " does not match the net's output dims");
        } catch (...) {
            delete L;
            throw;
        }
        *out = L;
    });
}

int znn_loader_open_host(znn_net net, const float* inputs, const float* labels, int64_t samples,
                         int64_t shard_offset, znn_loader* out) {
    if (!net) return ZNN_ERR_SHAPE;
    return guarded(net->ctx, [&] {
        if (!inputs || !labels || !out || samples < 1) throw znn_gpu::shape_error("znn_loader_open_host: bad argument");
        auto* L = new znn_loader_s;
        L->mem_in = inputs;
        L->mem_lab = labels;
        L->samples = samples;
        try {
            loader_alloc(L, net, shard_offset);
        } catch (...) {
            delete L;
            throw;
        }
        *out = L;
    });
}

int znn_loader_size(znn_loader ld, int64_t* samples) {
    if (!ld) return ZNN_ERR_SHAPE;
    *samples = ld->samples;
    return ZNN_OK;
}

int znn_loader_destroy(znn_loader ld) {
    if (!ld) return ZNN_OK;
    cudaSetDevice(ld->net->ctx->device);
    delete ld;
    return ZNN_OK;
}

int znn_net_step_loader(znn_net net, znn_loader ld, double* loss) {
    if (!net || !ld || ld->net != net) return ZNN_ERR_SHAPE;
    return guarded(net->ctx, [&] {
        znn_exec::executor& ex = *net->ex;
        cudaStream_t st = net->ctx->stream;
        ex.set_stream(st);
        const int64_t t = ld->step;
        const int slot = int(t & 1);
        if (t == 0) ld->prefetch(0, net->ctx->device);
        ld->wait_worker();  // step t's H2D is issued
        ZNN_CUDA_CHECK(cudaStreamWaitEvent(st, ld->ready[slot], 0));
        // step t + 1's files and H2D overlap this step's compute
        ld->prefetch(t + 1, net->ctx->device);
        const double l = ex.train_step(ld->d_in[slot], ld->d_lab[slot], false);
        (void)l;
        ZNN_CUDA_CHECK(cudaEventRecord(ld->consumed[slot], st));
        ld->step = t + 1;
        if (loss) *loss = ex.last_loss_device();
    });
}

}  // extern "C"
