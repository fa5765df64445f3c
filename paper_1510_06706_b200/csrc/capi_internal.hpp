// Shared internals of the C-ABI translation units (capi.cpp, capi_ext.cpp).
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <string>

#include "../../include/znn_cuda.h"
#include "net.hpp"
#include "ops.hpp"

struct znn_ctx_s {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    znn_gpu::scratch ws;
    int32_t* kinds = nullptr;  // per-map transfer kinds of the op-level calls (grow-only)
    int64_t kinds_cap = 0;
    ~znn_ctx_s() {
        if (kinds) cudaFree(kinds);
    }
};

struct znn_net_s {
    znn_ctx ctx = nullptr;
    std::unique_ptr<znn_exec::executor> ex;
};

namespace znn_capi {

inline thread_local std::string g_orphan_err;

template <typename F>
int guarded(znn_ctx ctx, F&& body) {
    std::string* err = ctx ? &ctx->err : &g_orphan_err;
    try {
        if (ctx) {
            cudaError_t e = cudaSetDevice(ctx->device);
            if (e != cudaSuccess) throw znn_gpu::cuda_error(cudaGetErrorString(e));
        }
        body();
        return ZNN_OK;
    } catch (const znn_gpu::shape_error& e) {
        *err = e.what();
        return ZNN_ERR_SHAPE;
    } catch (const std::exception& e) {
        *err = e.what();
        return ZNN_ERR_RUNTIME;
    }
}

inline znn_gpu::dims3 D(const int64_t* p) {
    if (!p) throw znn_gpu::shape_error("null dims pointer");
    return znn_gpu::dims3{p[0], p[1], p[2]};
}

}  // namespace znn_capi
