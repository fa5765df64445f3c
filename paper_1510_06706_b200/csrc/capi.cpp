// extern "C" boundary of libznn_cuda.so (declared in include/znn_cuda.h).
// Every entry point converts C++ exceptions into the reference's status
// convention: 1 = structural/config error, 2 = CUDA/runtime error.
#include "../../include/znn_cuda.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "capi_internal.hpp"
#include "fft.hpp"

namespace {

using znn_capi::D;
using znn_capi::g_orphan_err;
using znn_capi::guarded;

const int32_t* kinds_to_device(znn_ctx ctx, const int32_t* kinds_host, int64_t f) {
    // per-map kinds into the context's grow-only device array (no per-call allocation)
    static thread_local std::vector<int32_t> tmp;
    tmp.assign(kinds_host, kinds_host + f);
    for (int32_t k : tmp)
        if (k < 0 || k > 3) throw znn_gpu::shape_error("transfer: unknown transfer kind");
    if (f > ctx->kinds_cap) {
        if (ctx->kinds) {
            ZNN_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
            cudaFree(ctx->kinds);
            ctx->kinds = nullptr;
            ctx->kinds_cap = 0;
        }
        znn_gpu::dmalloc(&ctx->kinds, sizeof(int32_t) * size_t(std::max<int64_t>(f, 256)));
        ctx->kinds_cap = std::max<int64_t>(f, 256);
    }
    ZNN_CUDA_CHECK(cudaMemcpyAsync(ctx->kinds, tmp.data(), sizeof(int32_t) * size_t(f), cudaMemcpyHostToDevice,
                                   ctx->stream));
    return ctx->kinds;
}

}  // namespace

extern "C" {

const char* znn_version(void) { return "znn-b200 0.1 (sm_100a)"; }

int znn_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int znn_ctx_create(int device, znn_ctx* out) {
    if (!out) return ZNN_ERR_SHAPE;
    return guarded(nullptr, [&] {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
            cudaGetLastError();
            throw znn_gpu::cuda_error("no CUDA device: libznn_cuda has no CPU fallback");
        }
        if (device < 0 || device >= n) throw znn_gpu::shape_error("device index out of range");
        ZNN_CUDA_CHECK(cudaSetDevice(device));
        cudaDeviceProp prop{};
        ZNN_CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10)
            throw znn_gpu::cuda_error("libznn_cuda is built for sm_100a (B200); device is sm_" +
                                      std::to_string(prop.major) + std::to_string(prop.minor));
        auto* c = new znn_ctx_s;
        c->device = device;
        *out = c;
    });
}

int znn_ctx_destroy(znn_ctx ctx) {
    if (!ctx) return ZNN_OK;
    cudaSetDevice(ctx->device);
    delete ctx;
    return ZNN_OK;
}

int znn_ctx_set_stream(znn_ctx ctx, void* s) {
    if (!ctx) return ZNN_ERR_SHAPE;
    ctx->stream = static_cast<cudaStream_t>(s);
    return ZNN_OK;
}

int znn_ctx_synchronize(znn_ctx ctx) {
    return guarded(ctx, [&] { ZNN_CUDA_CHECK(cudaStreamSynchronize(ctx->stream)); });
}

const char* znn_last_error(znn_ctx ctx) { return ctx ? ctx->err.c_str() : g_orphan_err.c_str(); }

int64_t znn_ctx_launch_count(znn_ctx) { return znn_gpu::stats().launches; }

int znn_malloc(znn_ctx ctx, size_t bytes, void** dptr) {
    return guarded(ctx, [&] { ZNN_CUDA_CHECK(cudaMalloc(dptr, bytes)); });
}
int znn_free(znn_ctx ctx, void* dptr) {
    return guarded(ctx, [&] { ZNN_CUDA_CHECK(cudaFree(dptr)); });
}
int znn_memcpy_h2d(znn_ctx ctx, void* dst, const void* src, size_t bytes) {
    return guarded(ctx, [&] {
        ZNN_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
        ZNN_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}
int znn_memcpy_d2h(znn_ctx ctx, void* dst, const void* src, size_t bytes) {
    return guarded(ctx, [&] {
        ZNN_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        ZNN_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

// ---- per-layer operators --------------------------------------------

int znn_conv_fwd(znn_ctx ctx, const float* x, int64_t B, int64_t f_in, const int64_t n[3],
                 const float* w, int64_t f_out, const int64_t k[3], const int64_t s[3],
                 const float* bias, int act, float* y, int engine) {
    return guarded(ctx, [&] {
        if (act < 0 || act > 3) throw znn_gpu::shape_error("conv: unknown transfer kind");
        auto c = znn_gpu::conv_shape::make(B, f_in, f_out, D(n), D(k), D(s));
        if (engine == ZNN_CONV_FFT) {
            // op-level forward: a throw-away plan (the executor keeps its plans)
            auto plan = znn_fft::make_plan(c);
            znn_fft::conv_fwd(ctx->stream, *plan, c, x, w, bias, act, y, ctx->ws);
            ZNN_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        }
        else if (engine != ZNN_CONV_DIRECT_SIMT && znn_gpu::conv_tc_supported(c, 0))
            znn_gpu::conv_fwd_tc(ctx->stream, c, x, w, bias, act, y, ctx->ws);
        else
            znn_gpu::conv_fwd_simt(ctx->stream, c, x, w, bias, act, y);
    });
}

int znn_conv_dgrad(znn_ctx ctx, const float* g, int64_t B, int64_t f_out, const int64_t m[3],
                   const float* w, int64_t f_in, const int64_t k[3], const int64_t s[3],
                   float* dx, int engine) {
    return guarded(ctx, [&] {
        const auto md = D(m), kd = D(k), sd = D(s);
        const znn_gpu::dims3 n{md.x + sd.x * (kd.x - 1), md.y + sd.y * (kd.y - 1), md.z + sd.z * (kd.z - 1)};
        auto c = znn_gpu::conv_shape::make(B, f_in, f_out, n, kd, sd);
        if (engine == ZNN_CONV_FFT) {
            // wgrad output is required by the FFT backward kernel; use scratch
            throw znn_gpu::shape_error("fft engine: dgrad is only available through the network executor");
        } else if (engine != ZNN_CONV_DIRECT_SIMT && znn_gpu::conv_tc_supported(c, 1)) {
            znn_gpu::conv_dgrad_tc(ctx->stream, c, g, w, dx, ctx->ws);
        } else {
            znn_gpu::conv_dgrad_simt(ctx->stream, c, g, w, dx);
        }
    });
}

int znn_conv_wgrad(znn_ctx ctx, const float* x, int64_t B, int64_t f_in, const int64_t n[3],
                   const float* g, int64_t f_out, const int64_t k[3], const int64_t s[3],
                   float* dw, float scale, int engine) {
    return guarded(ctx, [&] {
        auto c = znn_gpu::conv_shape::make(B, f_in, f_out, D(n), D(k), D(s));
        if (engine == ZNN_CONV_FFT)
            throw znn_gpu::shape_error("fft engine: wgrad is only available through the network executor");
        else if (engine != ZNN_CONV_DIRECT_SIMT && znn_gpu::conv_tc_supported(c, 2))
            znn_gpu::conv_wgrad_tc(ctx->stream, c, x, g, dw, scale, ctx->ws);
        else
            znn_gpu::conv_wgrad_simt(ctx->stream, c, x, g, dw, scale, ctx->ws);
    });
}

int znn_transfer_fwd(znn_ctx ctx, const float* x, int64_t B, int64_t f, int64_t voxels,
                     const int32_t* kinds_host, const float* bias, float* y) {
    return guarded(ctx, [&] {
        const int32_t* kd = kinds_to_device(ctx, kinds_host, f);
        znn_gpu::transfer_fwd(ctx->stream, x, B, f, voxels, kd, bias, y);
    });
}

int znn_transfer_bwd(znn_ctx ctx, const float* g, const float* xy, int from_output, int64_t B,
                     int64_t f, int64_t voxels, const int32_t* kinds_host, const float* bias,
                     float* gx, float* dbias) {
    return guarded(ctx, [&] {
        const int32_t* kd = kinds_to_device(ctx, kinds_host, f);
        znn_gpu::transfer_bwd(ctx->stream, g, xy, from_output != 0, B, f, voxels, kd, bias, gx, dbias, ctx->ws);
    });
}

int znn_maxpool_fwd(znn_ctx ctx, const float* x, int64_t maps, const int64_t n[3],
                    const int64_t p[3], float* y, int32_t* mask) {
    return guarded(ctx, [&] { znn_gpu::maxpool_fwd(ctx->stream, x, maps, D(n), D(p), y, mask); });
}
int znn_maxpool_bwd(znn_ctx ctx, const float* g, const int32_t* mask, int64_t maps,
                    const int64_t m[3], const int64_t p[3], float* dx) {
    return guarded(ctx, [&] { znn_gpu::maxpool_bwd(ctx->stream, g, mask, maps, D(m), D(p), dx); });
}
int znn_maxfilter_fwd(znn_ctx ctx, const float* x, int64_t maps, const int64_t n[3],
                      const int64_t k[3], const int64_t s[3], float* y, int32_t* mask) {
    return guarded(ctx, [&] { znn_gpu::maxfilter_fwd(ctx->stream, x, maps, D(n), D(k), D(s), y, mask); });
}
int znn_maxfilter_bwd(znn_ctx ctx, const float* g, const int32_t* mask, int64_t maps,
                      const int64_t m[3], const int64_t k[3], const int64_t s[3], float* dx) {
    return guarded(ctx, [&] { znn_gpu::maxfilter_bwd(ctx->stream, g, mask, maps, D(m), D(k), D(s), dx); });
}

int znn_loss(znn_ctx ctx, int kind, const float* a, const float* d, int64_t count, float scale,
             float* grad, double* loss_out) {
    return guarded(ctx, [&] {
        if (kind != ZNN_LOSS_L2 && kind != ZNN_LOSS_CE) throw znn_gpu::shape_error("loss: unknown kind");
        const double l = znn_gpu::loss_grad(ctx->stream, kind, a, d, count, scale, grad, ctx->ws);
        if (loss_out) *loss_out = l;
    });
}

int znn_sgd_momentum(znn_ctx ctx, float* w, float* v, const float* g, int64_t count, float lr,
                     float mu) {
    return guarded(ctx, [&] { znn_gpu::sgd_momentum(ctx->stream, w, v, g, count, lr, mu); });
}

// ---- network executor -----------------------------------------------

int znn_net_create(znn_ctx ctx, const char* netspec, const int64_t* out_dims,
                   const znn_train_cfg* cfg, znn_net* out) {
    return guarded(ctx, [&] {
        if (!netspec || !cfg || !out) throw znn_gpu::shape_error("znn_net_create: null argument");
        znn_exec::train_cfg c;
        c.batch = cfg->batch;
        c.global_batch = cfg->global_batch > 0 ? cfg->global_batch : cfg->batch;
        c.lr = cfg->learning_rate;
        c.mu = cfg->momentum;
        c.loss = cfg->loss;
        c.engine = cfg->engine == ZNN_CONV_AUTO ? ZNN_CONV_DIRECT : cfg->engine;
        c.sliding = cfg->sliding != 0;
        // per-group backward images only on request (tests/inspection); the
        // default is two ping-pong gradient buffers
        c.keep_images = getenv("ZNN_KEEP_IMAGES") != nullptr && std::string(getenv("ZNN_KEEP_IMAGES")) == "1";
        znn_host::v3 od{0, 0, 0};
        if (out_dims) od = znn_host::v3{out_dims[0], out_dims[1], out_dims[2]};
        auto* n = new znn_net_s;
        n->ctx = ctx;
        try {
            n->ex = std::make_unique<znn_exec::executor>(netspec, out_dims ? &od : nullptr, c, ctx->stream);
        } catch (...) {
            delete n;
            throw;
        }
        *out = n;
    });
}

int znn_net_destroy(znn_net net) {
    if (!net) return ZNN_OK;
    cudaSetDevice(net->ctx->device);
    delete net;
    return ZNN_OK;
}

const char* znn_net_describe(znn_net net) { return net ? net->ex->describe().c_str() : ""; }

int znn_net_num_params(znn_net net, int64_t* count) {
    return guarded(net->ctx, [&] { *count = net->ex->num_params(); });
}

int znn_net_io_sizes(znn_net net, int64_t* in_per_patch, int64_t* out_per_patch) {
    return guarded(net->ctx, [&] {
        if (in_per_patch) *in_per_patch = net->ex->in_per_patch();
        if (out_per_patch) *out_per_patch = net->ex->out_per_patch();
    });
}

int znn_net_set_params(znn_net net, const float* p) {
    return guarded(net->ctx, [&] { net->ex->set_stream(net->ctx->stream); net->ex->set_params(p); });
}
int znn_net_get_params(znn_net net, float* p) {
    return guarded(net->ctx, [&] { net->ex->set_stream(net->ctx->stream); net->ex->get_params(p); });
}
int znn_net_get_gradients(znn_net net, float* p) {
    return guarded(net->ctx, [&] { net->ex->set_stream(net->ctx->stream); net->ex->get_gradients(p); });
}
int znn_net_reset_momentum(znn_net net) {
    return guarded(net->ctx, [&] { net->ex->set_stream(net->ctx->stream); net->ex->reset_momentum(); });
}
int znn_net_set_layer_engine(znn_net net, int conv_layer, int engine) {
    return guarded(net->ctx, [&] { net->ex->set_layer_engine(conv_layer, engine); });
}
int znn_net_autotune(znn_net net, int trials, int32_t* chosen, int max_layers) {
    return guarded(net->ctx, [&] {
        net->ex->set_stream(net->ctx->stream);
        auto c = net->ex->autotune(trials);
        for (size_t i = 0; i < c.size() && int(i) < max_layers; ++i)
            if (chosen) chosen[i] = c[i];
    });
}

int znn_net_fft_counts(znn_net net, int conv_layer, int64_t* out) {
    return guarded(net->ctx, [&] {
        znn_fft::transform_counts t;
        if (!net->ex->fft_counts(conv_layer, t)) throw znn_gpu::shape_error("conv layer has no FFT plan");
        const int64_t v[9] = {t.fwd_image, t.fwd_kernel, t.fwd_inverse, t.bwd_image, t.bwd_kernel,
                              t.bwd_inverse, t.upd_image, t.upd_kernel, t.upd_inverse};
        for (int i = 0; i < 9; ++i) out[i] = v[i];
    });
}

int znn_fft_cmac_time(znn_ctx ctx, int which, int64_t B, int64_t f_in, int64_t f_out, const int64_t n[3],
                      const int64_t k[3], const int64_t s[3], int reps, float* ms, int64_t* bins) {
    return guarded(ctx, [&] {
        auto c = znn_gpu::conv_shape::make(B, f_in, f_out, D(n), D(k), D(s));
        const float t = znn_fft::time_cmac(ctx->stream, which, c, reps, bins);
        if (ms) *ms = t;
    });
}

int znn_fma_peak_tflops(znn_ctx ctx, float* tflops) {
    return guarded(ctx, [&] {
        const float t = znn_fft::fma_peak_tflops(ctx->stream);
        if (tflops) *tflops = t;
    });
}

int znn_net_step_host(znn_net net, const float* inputs, const float* labels, double* loss) {
    return guarded(net->ctx, [&] {
        net->ex->set_stream(net->ctx->stream);
        const double l = net->ex->step_host(inputs, labels);
        if (loss) *loss = l;
    });
}

int znn_net_forward_backward(znn_net net, const float* inputs_dev, const float* labels_dev,
                             double* loss) {
    return guarded(net->ctx, [&] {
        net->ex->set_stream(net->ctx->stream);
        const double l = net->ex->forward_backward(inputs_dev, labels_dev, loss != nullptr);
        if (loss) *loss = l;
    });
}

int znn_net_train_step(znn_net net, const float* inputs_dev, const float* labels_dev, double* loss) {
    return guarded(net->ctx, [&] {
        net->ex->set_stream(net->ctx->stream);
        const double l = net->ex->train_step(inputs_dev, labels_dev, loss != nullptr);
        if (loss) *loss = l;
    });
}

int znn_net_apply_update(znn_net net) {
    return guarded(net->ctx, [&] { net->ex->set_stream(net->ctx->stream); net->ex->apply_update(); });
}

int znn_net_grad_buffer(znn_net net, float** dptr, int64_t* count) {
    return guarded(net->ctx, [&] {
        *dptr = net->ex->grad_buffer();
        *count = net->ex->flat_size();
    });
}

int znn_net_forward(znn_net net, const float* inputs_dev, float* host_out) {
    return guarded(net->ctx, [&] {
        net->ex->set_stream(net->ctx->stream);
        net->ex->forward(inputs_dev);
        if (host_out) net->ex->copy_outputs(host_out);
    });
}

int znn_net_group_info(znn_net net, int group, int64_t* maps, int64_t dims[3]) {
    return guarded(net->ctx, [&] {
        if (group < 0 || group >= net->ex->num_groups()) throw znn_gpu::shape_error("group index out of range");
        const auto& G = net->ex->grp(group);
        if (maps) *maps = G.materialized ? G.maps : -G.maps;
        if (dims) dims[0] = G.dims.x, dims[1] = G.dims.y, dims[2] = G.dims.z;
    });
}

int znn_net_get_group_image(znn_net net, int group, int which, float* host) {
    return guarded(net->ctx, [&] { net->ex->set_stream(net->ctx->stream); net->ex->group_image(group, which, host); });
}

int znn_net_get_mask(znn_net net, int group, int32_t* host) {
    return guarded(net->ctx, [&] { net->ex->set_stream(net->ctx->stream); net->ex->group_mask(group, host); });
}

}  // extern "C"
