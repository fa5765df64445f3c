/*
 * znn_gpu_engine.hpp — reference-side drop-in for engine<float> on one B200.
 *
 * Header-only C++ over the C ABI (znn_cuda.h, libznn_cuda.so). Include it
 * AFTER the reference's headers (it uses znn::net_graph, conv_op,
 * transfer_op and engine<float>::sample / sample_source / round_stats from
 * /root/reference/proj/include/znn) and link -lznn_cuda. It replaces
 *
 *   engine<float> eng(g, compute_priorities(g), cfg);       // engine.hpp:65
 *   auto stats = eng.run(rounds, source);                    // engine.hpp:200-254
 *
 * with
 *
 *   znn::gpu_engine eng(g, netspec_text, gcfg);
 *   auto stats = eng.run(rounds, source);
 *
 * Same net_graph, same netspec text (netspec.hpp:13-27), same sample source
 * (one sample per round, inputs / desired in node-id order), same per-round
 * loss (half-L2, taskgraph.hpp:116-126, or CE), same parameter order
 * (edges by id: conv kernel volume, transfer bias; test_engine.cpp:57-67).
 * After run() the updated parameters are written back into the graph's
 * conv_op / transfer_op edges, as the reference's in-place updates leave
 * them (engine.hpp:775-801). Errors: status 1 -> structural_error,
 * status 2 -> std::runtime_error (types.hpp:57-74, tools/znn.cpp:182-191).
 *
 * Data parallelism: give each rank a communicator (znn_comm_create over an
 * id rank 0 made with znn_comm_unique_id) and the global batch; run() then
 * sums the weight gradients over ranks with one NCCL allreduce per layer,
 * overlapped with the backward pass (znn_net_train_step_dp).
 */
#pragma once

#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "znn_cuda.h"

namespace znn {

struct gpu_engine_config {
    int device = 0;
    float learning_rate = 0.01f;  // engine<T>::config::learning_rate (engine.hpp:70)
    float momentum = 0.f;         // 0 = the reference's plain SGD
    int loss = ZNN_LOSS_L2;       // the reference's half-L2
    int conv = ZNN_CONV_AUTO;     // conv_mode_policy: direct / fft / autotune (trainer.hpp:22)
    int autotune_trials = 3;      // train_config::autotune_trials
    int64_t batch = 1;            // samples per step on this rank (the reference: 1 per round)
    int64_t global_batch = 0;     // 0 = batch (data parallel: the sum over ranks)
    znn_comm comm = nullptr;      // data-parallel communicator (optional)
};

class gpu_engine {
public:
    using sample = typename engine<float>::sample;
    using sample_source = typename engine<float>::sample_source;
    using round_stats = typename engine<float>::round_stats;

    gpu_engine(net_graph<float>& g, const std::string& netspec_text, const gpu_engine_config& cfg = {})
        : g_(g), cfg_(cfg) {
        check_ctx(znn_ctx_create(cfg.device, &ctx_));
        znn_train_cfg tc{cfg.batch, cfg.global_batch > 0 ? cfg.global_batch : cfg.batch, cfg.learning_rate,
                         cfg.momentum, cfg.loss, cfg.conv == ZNN_CONV_AUTO ? ZNN_CONV_DIRECT : cfg.conv, 0};
        vec3i od{0, 0, 0};
        for (const auto& n : g.nodes)
            if (n.role == node_role::output) od = n.dims;
        const int64_t odims[3] = {od.x, od.y, od.z};
        check(znn_net_create(ctx_, netspec_text.c_str(), odims, &tc, &net_));
        int64_t np = 0, in_pp = 0, out_pp = 0;
        check(znn_net_num_params(net_, &np));
        check(znn_net_io_sizes(net_, &in_pp, &out_pp));
        params_.resize(size_t(np));
        in_.resize(size_t(in_pp * cfg.batch));
        out_.resize(size_t(out_pp * cfg.batch));
        collect(g_, params_);
        check(znn_net_set_params(net_, params_.data()));
        if (cfg.conv == ZNN_CONV_AUTO) {
            std::vector<int32_t> chosen(256);
            check(znn_net_autotune(net_, cfg.autotune_trials, chosen.data(), int(chosen.size())));
        }
        if (cfg.comm) {
            check(znn_malloc(ctx_, sizeof(float) * in_.size(), reinterpret_cast<void**>(&d_in_)));
            check(znn_malloc(ctx_, sizeof(float) * out_.size(), reinterpret_cast<void**>(&d_out_)));
        }
    }

    ~gpu_engine() {
        if (d_in_) znn_free(ctx_, d_in_);
        if (d_out_) znn_free(ctx_, d_out_);
        znn_net_destroy(net_);
        znn_ctx_destroy(ctx_);
    }
    gpu_engine(const gpu_engine&) = delete;
    gpu_engine& operator=(const gpu_engine&) = delete;

    // engine<float>::run: `rounds` SGD steps; each step consumes `batch`
    // consecutive samples of the source (round numbers start at 1). The
    // returned seconds are device-synchronous wall times per step; loss is
    // the mean per-sample loss of the step.
    std::vector<round_stats> run(std::int64_t rounds, const sample_source& source) {
        std::vector<round_stats> stats;
        std::int64_t r = next_round_;
        for (std::int64_t t = 0; t < rounds; ++t) {
            const auto t0 = std::chrono::steady_clock::now();
            size_t io = 0, oo = 0;
            for (int64_t b = 0; b < cfg_.batch; ++b) {
                const sample& s = source(r++);
                io += pack(s.inputs, in_.data() + io);
                oo += pack(s.desired, out_.data() + oo);
            }
            double loss = 0;
            if (cfg_.comm) {
                check(znn_memcpy_h2d(ctx_, d_in_, in_.data(), sizeof(float) * in_.size()));
                check(znn_memcpy_h2d(ctx_, d_out_, out_.data(), sizeof(float) * out_.size()));
                check(znn_net_train_step_dp(net_, cfg_.comm, d_in_, d_out_, &loss));
            } else {
                check(znn_net_step_host(net_, in_.data(), out_.data(), &loss));
            }
            round_stats rs;
            rs.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            rs.loss = loss;
            stats.push_back(rs);
        }
        next_round_ = r;
        check(znn_net_get_params(net_, params_.data()));
        scatter(params_, g_);
        return stats;
    }

    znn_net handle() const { return net_; }
    znn_ctx context() const { return ctx_; }
    const char* describe() const { return znn_net_describe(net_); }

private:
    void check_ctx(int st) {
        if (st == ZNN_ERR_SHAPE) throw structural_error(znn_last_error(nullptr));
        if (st != ZNN_OK) throw std::runtime_error(znn_last_error(nullptr));
    }
    void check(int st) {
        if (st == ZNN_ERR_SHAPE) throw structural_error(znn_last_error(ctx_));
        if (st != ZNN_OK) throw std::runtime_error(znn_last_error(ctx_));
    }
    static size_t pack(const std::vector<vol_p<float>>& vols, float* dst) {
        size_t off = 0;
        for (const auto& v : vols) {
            std::memcpy(dst + off, v->data(), sizeof(float) * size_t(v->size()));
            off += size_t(v->size());
        }
        return off;
    }
    static void collect(const net_graph<float>& g, std::vector<float>& p) {
        size_t off = 0;
        for (const auto& e : g.edges) {
            if (auto* c = std::get_if<conv_op<float>>(&e.op)) {
                for (std::int64_t i = 0; i < c->k.weights.size(); ++i) p.at(off++) = c->k.weights[i];
            } else if (auto* t = std::get_if<transfer_op<float>>(&e.op)) {
                p.at(off++) = t->fn.bias;
            }
        }
        if (off != p.size()) throw structural_error("gpu_engine: parameter count differs from the net_graph");
    }
    static void scatter(const std::vector<float>& p, net_graph<float>& g) {
        size_t off = 0;
        for (auto& e : g.edges) {
            if (auto* c = std::get_if<conv_op<float>>(&e.op)) {
                for (std::int64_t i = 0; i < c->k.weights.size(); ++i) c->k.weights[i] = p[off++];
            } else if (auto* t = std::get_if<transfer_op<float>>(&e.op)) {
                t->fn.bias = p[off++];
            }
        }
    }

    net_graph<float>& g_;
    gpu_engine_config cfg_;
    znn_ctx ctx_ = nullptr;
    znn_net net_ = nullptr;
    float* d_in_ = nullptr;
    float* d_out_ = nullptr;
    std::vector<float> params_, in_, out_;
    std::int64_t next_round_ = 1;
};

}  // namespace znn
