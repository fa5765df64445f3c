// Layer-wave GPU executor: replaces the reference's per-edge task engine
// (engine.hpp:45-901) for one data-parallel rank. Nodes of the reference
// graph are grouped by depth into node groups (one device tensor
// [B][maps][x][y][z] per group); each group-to-group transition is one layer
// call covering every edge between the two groups and every patch.
#pragma once

#include <cuda_runtime.h>

#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "fft.hpp"
#include "netgraph.hpp"
#include "ops.hpp"

namespace znn_exec {

using znn_gpu::conv_shape;
using znn_gpu::dims3;
using znn_host::v3;

struct group {
    std::vector<int> nodes;  // graph node ids in map order
    int64_t maps = 0;
    dims3 dims{1, 1, 1};
    float* act = nullptr;    // forward image [B][maps][vol] (null when fused away)
    float* grad = nullptr;   // backward image (kept per group only with keep_images)
    int32_t* mask = nullptr; // argmax record (flat index) when produced by a pool
    uint8_t* code = nullptr; // argmax record (window code) when produced by a max-filter
    bool materialized = true;
    // phase-major order [B s^3][maps][dims / s] (phase r = (rx sy + ry) sz + rz holds
    // the voxels s q + r) instead of [B][maps][dims]: between two FFT layers
    // of the same sparsity (executor::plan_layouts)
    bool pm = false;
    dims3 pm_s{1, 1, 1};
};

enum class lkind { conv, transfer, pool, filter };

struct layer {
    lkind kind = lkind::conv;
    int in = -1, out = -1;  // group indices
    // conv
    conv_shape shape;
    int64_t w_off = -1;     // offset of [f_out][f_in][T] in the flat parameter buffer
    int engine = 0;         // ZNN_CONV_*
    std::shared_ptr<znn_fft::plan> fft;  // memoised spectra when engine == FFT
    bool fused = false;     // transfer edge fused into the conv epilogue
    int fused_act = 3;
    int64_t b_off = -1;     // bias offset (fused transfer or transfer layer)
    // transfer
    std::vector<int32_t> kinds;
    int32_t* kinds_dev = nullptr;
    int32_t* none_dev = nullptr;  // identity kinds (CE: loss already gave a - d)
    // pool / filter
    dims3 k{1, 1, 1}, s{1, 1, 1};
    bool relu_gate = false;     // filter: its codes carry the ReLU backward of the conv feeding it
    bool pregated = false;      // conv with fused ReLU: the gradient arrives gated (by a relu_gate filter)
    bool bias_summed = false;   // this backward pass: the filter above already left the bias gradient
    std::vector<int> edge_ids;  // reference edges covered (map order)
    std::vector<int> transfer_edge_ids;
};

struct train_cfg {
    int64_t batch = 1, global_batch = 1;
    float lr = 0.01f, mu = 0.f;
    int loss = 0, engine = 0;
    bool sliding = false;
    bool keep_images = true;
};

class executor {
public:
    executor(const std::string& netspec, const v3* out_dims, const train_cfg& cfg,
             cudaStream_t stream);
    ~executor();
    executor(const executor&) = delete;
    executor& operator=(const executor&) = delete;

    void set_stream(cudaStream_t s) { st_ = s; }
    const std::string& describe() const { return desc_; }
    int64_t num_params() const { return int64_t(canon_.size()); }
    int64_t in_per_patch() const;
    int64_t out_per_patch() const;
    void set_params(const float* host);
    void get_params(float* host);
    void get_gradients(float* host);
    void reset_momentum();
    void set_layer_engine(int conv_layer, int engine);
    std::vector<int> autotune(int trials);

    // inputs/labels are device pointers [B][maps][vol] in input/output-node id order
    // update: apply SGD+momentum layer by layer as each gradient becomes final
    // (fused into the tensor-core weight-gradient epilogue); single-process
    // training only — data parallelism needs the summed gradient first
    double forward_backward(const float* in_dev, const float* labels_dev, bool sync_loss = true,
                            bool update = false);
    // single-process SGD step (forward_backward with the fused update); with
    // graph mode on, the second call onwards replays one captured CUDA graph
    // of the whole step (the scratch arena is frozen: no allocation)
    double train_step(const float* in_dev, const float* labels_dev, bool sync_loss);
    void set_graph_mode(bool on);
    bool graph_captured() const { return !graphs_.empty(); }
    int64_t batch() const { return cfg_.batch; }
    int64_t global_batch() const { return cfg_.global_batch; }
    // called at issue time, in backward order, once a layer's slice of the
    // flat gradient buffer [off, off + count) is final on the stream
    // (data-parallel bucketed allreduce)
    void set_grad_hook(std::function<void(int64_t, int64_t)> h) { grad_hook_ = std::move(h); }
    // bytes of device memory the kernel spectra of all FFT layers may use
    // (pool + resident), from cudaMemGetInfo at first use
    double fft_kernel_budget() const { return fft_budget_; }
    void apply_update();
    void forward(const float* in_dev);
    double step_host(const float* in_host, const float* labels_host);
    void copy_outputs(float* host);
    float* grad_buffer() { return grads_; }
    int64_t flat_size() const { return flat_; }
    int num_groups() const { return int(groups_.size()); }
    const group& grp(int i) const { return groups_.at(size_t(i)); }
    void group_image(int g, int which, float* host);
    void group_mask(int g, int32_t* host);
    const std::vector<layer>& layers() const { return layers_; }
    // transform counts of conv layer `conv_layer` (FFT engine), test hook
    bool fft_counts(int conv_layer, znn_fft::transform_counts& out) const;
    double last_loss_device();

private:
    void build(const znn_host::graph& g);
    void allocate();
    void run_forward(const float* in_dev);
    void run_conv_fwd(layer& L);
    void run_conv_bwd(layer& L, float* g_out, float* g_in, bool need_dgrad, bool update,
                      const float* relu_y = nullptr, float* dbias = nullptr);
    znn_fft::plan& fft_plan(layer& L);
    bool fft_pooled(const layer& L);
    void plan_fft_memory();
    void plan_layouts();
    void drop_fft_plans();
    void drop_graph();
    bool fft_decided_ = false;
    double fft_budget_ = -1.0;
    std::vector<const layer*> fft_pool_members_;
    std::function<void(int64_t, int64_t)> grad_hook_;
    bool graph_mode_ = false;
    int graph_warm_ = 0;
    struct step_graph {
        const float* in;
        const float* lab;
        cudaGraphExec_t exec;
    };
    std::vector<step_graph> graphs_;  // one per (input, label) buffer pair (double-buffered loaders: 2)
    std::shared_ptr<znn_fft::kpool> kpool_;  // kernel spectra shared by the largest FFT layers
    std::shared_ptr<znn_gpu::scratch> phase_ws_;  // phase-split tensors of the dilated FFT layers

    train_cfg cfg_;
    cudaStream_t st_ = nullptr;
    znn_host::graph g_;
    std::vector<group> groups_;
    std::vector<layer> layers_;
    std::string desc_;
    std::string layout_note_;  // phase-major groups currently planned
    int64_t flat_ = 0;
    float* params_ = nullptr;
    float* grads_ = nullptr;
    float* vel_ = nullptr;
    float* gbuf_[2] = {nullptr, nullptr};
    float* labels_perm_ = nullptr;
    float* in_stage_ = nullptr;
    float* lab_stage_ = nullptr;
    double* loss_dev_ = nullptr;
    std::vector<int> out_perm_;  // group-position -> output ordinal
    bool out_identity_ = true;
    std::vector<int64_t> canon_;  // canonical param index -> flat index
    znn_gpu::scratch ws_;
    std::vector<void*> owned_;
    void* dalloc(size_t bytes);
};

}  // namespace znn_exec
