#include "net.hpp"

#include <algorithm>
#include <cstring>
#include <map>
#include <sstream>

#include "fft.hpp"

namespace znn_exec {

using znn_gpu::require;
using znn_host::op;
using znn_host::role;
using znn_host::gedge;

namespace {
dims3 to_d3(v3 v) { return dims3{v.x, v.y, v.z}; }
const char* kname(lkind k) {
    switch (k) {
        case lkind::conv: return "conv";
        case lkind::transfer: return "transfer";
        case lkind::pool: return "pool";
        default: return "filter";
    }
}
const char* ename(int e) {
    switch (e) {
        case 0: return "direct";
        case 1: return "fft";
        case 2: return "auto";
        default: return "direct-simt";
    }
}
}  // namespace

executor::executor(const std::string& netspec, const v3* out_dims, const train_cfg& cfg,
                   cudaStream_t stream)
    : cfg_(cfg), st_(stream) {
    require(cfg.batch >= 1 && cfg.global_batch >= cfg.batch, "train config: bad batch sizes");
    require(cfg.loss == 0 || cfg.loss == 1, "train config: unknown loss");
    v3 od = out_dims ? *out_dims : v3{0, 0, 0};
    znn_host::graph g = znn_host::parse_netspec(netspec, od);
    if (cfg.sliding) {
        v3 outd{0, 0, 0};
        for (const auto& n : g.nodes)
            if (n.r == role::output) outd = n.dims;
        g = znn_host::sliding_equivalent(g);
        znn_host::infer_shapes(g, outd);
    }
    g_ = std::move(g);
    build(g_);
    allocate();
}

executor::~executor() {
    for (auto& g : graphs_) cudaGraphExecDestroy(g.exec);
    for (auto& L : layers_) L.fft.reset();
    kpool_.reset();
    phase_ws_.reset();
    for (void* p : owned_) cudaFree(p);
}

void* executor::dalloc(size_t bytes) {
    void* p = nullptr;
    znn_gpu::dmalloc(&p, bytes < 16 ? 16 : bytes);
    owned_.push_back(p);
    return p;
}

void executor::build(const znn_host::graph& g) {
    const auto order = g.topo();
    std::vector<int> depth(g.nodes.size(), 0);
    for (int v : order)
        for (int eid : g.nodes[size_t(v)].outs) {
            const int t = g.edges[size_t(eid)].to;
            depth[size_t(t)] = std::max(depth[size_t(t)], depth[size_t(v)] + 1);
        }
    int D = 0;
    for (int d : depth) D = std::max(D, d);
    std::vector<std::vector<int>> byd(size_t(D) + 1);
    for (size_t v = 0; v < g.nodes.size(); ++v) byd[size_t(depth[v])].push_back(int(v));
    for (const auto& e : g.edges)
        require(depth[size_t(e.to)] == depth[size_t(e.from)] + 1,
                "GPU executor: edge " + e.name + " skips a layer (node groups must be layered)");
    for (int v : byd[0]) require(g.nodes[size_t(v)].r == role::input, "GPU executor: depth-0 node " + g.nodes[size_t(v)].name + " is not an input");
    for (size_t v = 0; v < g.nodes.size(); ++v)
        require((g.nodes[v].r == role::output) == (depth[v] == D),
                "GPU executor: outputs must be exactly the deepest node group (node " + g.nodes[v].name + ")");

    groups_.resize(size_t(D) + 1);
    groups_[0].nodes = byd[0];
    std::vector<int> pos(g.nodes.size(), -1);
    auto set_group = [&](int d, const std::vector<int>& nodes) {
        group& G = groups_[size_t(d)];
        G.nodes = nodes;
        G.maps = int64_t(nodes.size());
        const v3 dm = g.nodes[size_t(nodes[0])].dims;
        for (size_t i = 0; i < nodes.size(); ++i) {
            require(g.nodes[size_t(nodes[i])].dims == dm, "GPU executor: node group " + std::to_string(d) + " has unequal image dims");
            pos[size_t(nodes[i])] = int(i);
        }
        G.dims = to_d3(dm);
    };
    set_group(0, byd[0]);

    for (int d = 0; d < D; ++d) {
        const auto& heads = byd[size_t(d) + 1];
        const op kind = g.edges[size_t(g.nodes[size_t(heads[0])].ins[0])].kind;
        layer L;
        L.in = d, L.out = d + 1;
        const group& I = groups_[size_t(d)];
        if (kind == op::conv) {
            const gedge& e0 = g.edges[size_t(g.nodes[size_t(heads[0])].ins[0])];
            for (int h : heads)
                for (int eid : g.nodes[size_t(h)].ins) {
                    const auto& e = g.edges[size_t(eid)];
                    require(e.kind == op::conv && e.k == e0.k && e.s == e0.s,
                            "GPU executor: conv layer " + std::to_string(d) + " mixes kernels/sparsities/edge types");
                }
            std::vector<int> hs = heads;
            std::sort(hs.begin(), hs.end());
            set_group(d + 1, hs);
            // full connectivity: exactly one edge per (head, tail) pair
            std::vector<int> seen(size_t(I.maps) * hs.size(), -1);
            for (int h : hs)
                for (int eid : g.nodes[size_t(h)].ins) {
                    const auto& e = g.edges[size_t(eid)];
                    const size_t slot = size_t(pos[size_t(h)]) * size_t(I.maps) + size_t(pos[size_t(e.from)]);
                    require(seen[slot] < 0, "GPU executor: duplicate conv edge " + e.name);
                    seen[slot] = eid;
                }
            for (int s : seen) require(s >= 0, "GPU executor: conv layer " + std::to_string(d) + " is not fully connected");
            L.kind = lkind::conv;
            L.edge_ids = seen;  // [o][i]
            L.shape = conv_shape::make(cfg_.batch, I.maps, int64_t(hs.size()), I.dims, to_d3(e0.k), to_d3(e0.s));
            L.engine = cfg_.engine;
        } else {
            // element-wise layer: one in-edge per head, one out-edge per tail
            require(heads.size() == size_t(I.maps), "GPU executor: layer " + std::to_string(d) + " must map tails to heads one-to-one");
            std::vector<int> hs(heads.size(), -1);
            std::vector<int> eids(heads.size(), -1);
            const gedge& e0 = g.edges[size_t(g.nodes[size_t(heads[0])].ins[0])];
            for (int h : heads) {
                require(g.nodes[size_t(h)].ins.size() == 1, "GPU executor: node " + g.nodes[size_t(h)].name + " mixes convergent edges with a non-conv layer");
                const auto& e = g.edges[size_t(g.nodes[size_t(h)].ins[0])];
                require(e.kind == kind, "GPU executor: layer " + std::to_string(d) + " mixes edge types");
                if (kind != op::transfer)
                    require(e.k == e0.k && e.s == e0.s, "GPU executor: layer " + std::to_string(d) + " mixes windows");
                const int p = pos[size_t(e.from)];
                require(p >= 0 && hs[size_t(p)] < 0, "GPU executor: layer " + std::to_string(d) + " is not one-to-one");
                hs[size_t(p)] = h;
                eids[size_t(p)] = g.nodes[size_t(h)].ins[0];
            }
            for (int v : byd[size_t(d)])
                require(g.nodes[size_t(v)].outs.size() == 1, "GPU executor: node " + g.nodes[size_t(v)].name + " fans out into an element-wise layer");
            set_group(d + 1, hs);
            L.edge_ids = eids;
            if (kind == op::transfer) {
                L.kind = lkind::transfer;
                for (int eid : eids) L.kinds.push_back(g.edges[size_t(eid)].fn);
            } else {
                L.kind = kind == op::pool ? lkind::pool : lkind::filter;
                L.k = to_d3(e0.k);
                L.s = to_d3(e0.s);
            }
        }
        layers_.push_back(std::move(L));
    }

    // fuse conv -> transfer (uniform kind) into the conv epilogue
    std::vector<layer> fused;
    for (size_t i = 0; i < layers_.size(); ++i) {
        layer L = layers_[i];
        if (L.kind == lkind::conv && i + 1 < layers_.size() && layers_[i + 1].kind == lkind::transfer) {
            const layer& T = layers_[i + 1];
            bool uniform = std::all_of(T.kinds.begin(), T.kinds.end(), [&](int k) { return k == T.kinds[0]; });
            if (uniform) {
                L.fused = true;
                L.fused_act = T.kinds[0];
                L.kinds = T.kinds;
                L.transfer_edge_ids = T.edge_ids;
                groups_[size_t(L.out)].materialized = false;
                L.out = T.out;
                ++i;
            }
        }
        fused.push_back(std::move(L));
    }
    layers_ = std::move(fused);

    // flat parameter layout and the canonical (reference edge-id) order map
    std::vector<std::pair<int64_t, int64_t>> edge_slot(g.edges.size(), {-1, 0});
    flat_ = 0;
    for (auto& L : layers_) {
        if (L.kind == lkind::conv) {
            const int64_t T = L.shape.taps();
            L.w_off = flat_;
            for (int64_t o = 0; o < L.shape.f_out; ++o)
                for (int64_t i = 0; i < L.shape.f_in; ++i)
                    edge_slot[size_t(L.edge_ids[size_t(o * L.shape.f_in + i)])] = {L.w_off + (o * L.shape.f_in + i) * T, T};
            flat_ += L.shape.f_out * L.shape.f_in * T;
            if (L.fused) {
                L.b_off = flat_;
                for (size_t o = 0; o < L.transfer_edge_ids.size(); ++o)
                    edge_slot[size_t(L.transfer_edge_ids[o])] = {L.b_off + int64_t(o), 1};
                flat_ += L.shape.f_out;
            }
        } else if (L.kind == lkind::transfer) {
            L.b_off = flat_;
            for (size_t o = 0; o < L.edge_ids.size(); ++o) edge_slot[size_t(L.edge_ids[o])] = {L.b_off + int64_t(o), 1};
            flat_ += int64_t(L.edge_ids.size());
        }
    }
    canon_.clear();
    for (size_t eid = 0; eid < g.edges.size(); ++eid) {
        const auto& e = g.edges[eid];
        if (e.kind != op::conv && e.kind != op::transfer) continue;
        for (int64_t t = 0; t < edge_slot[eid].second; ++t) canon_.push_back(edge_slot[eid].first + t);
    }

    // output ordering: group position -> ordinal among output nodes by id
    const group& G = groups_.back();
    std::vector<int> outs;
    for (size_t v = 0; v < g.nodes.size(); ++v)
        if (g.nodes[v].r == role::output) outs.push_back(int(v));
    out_perm_.assign(size_t(G.maps), 0);
    out_identity_ = true;
    for (size_t p = 0; p < G.nodes.size(); ++p) {
        out_perm_[p] = int(std::find(outs.begin(), outs.end(), G.nodes[p]) - outs.begin());
        if (out_perm_[p] != int(p)) out_identity_ = false;
    }
    if (cfg_.loss == 1) {
        const layer& last = layers_.back();
        const bool ok = (last.kind == lkind::conv && last.fused && last.fused_act == 0) ||
                        (last.kind == lkind::transfer &&
                         std::all_of(last.kinds.begin(), last.kinds.end(), [](int k) { return k == 0; }));
        require(ok, "cross-entropy loss needs a logistic transfer edge into every output node");
    }

    std::ostringstream os;
    for (size_t i = 0; i < groups_.size(); ++i)
        os << "group " << i << ": maps=" << groups_[i].maps << " dims=" << groups_[i].dims.x << ","
           << groups_[i].dims.y << "," << groups_[i].dims.z << (groups_[i].materialized ? "" : " (fused)") << "\n";
    int ci = 0;
    for (const auto& L : layers_) {
        os << "layer " << kname(L.kind) << " " << L.in << "->" << L.out;
        if (L.kind == lkind::conv) {
            os << " conv#" << ci++ << " f=" << L.shape.f_in << "->" << L.shape.f_out << " k=" << L.shape.k.x << ","
               << L.shape.k.y << "," << L.shape.k.z << " s=" << L.shape.s.x << "," << L.shape.s.y << "," << L.shape.s.z
               << " engine=" << ename(L.engine);
            if (L.fused) os << " +transfer(kind=" << L.fused_act << ")";
        } else if (L.kind == lkind::pool || L.kind == lkind::filter) {
            os << " k=" << L.k.x << "," << L.k.y << "," << L.k.z << " s=" << L.s.x << "," << L.s.y << "," << L.s.z;
        }
        os << "\n";
    }
    desc_ = os.str();
}

void executor::allocate() {
    const int64_t B = cfg_.batch;
    int64_t maxsz = 0;
    for (size_t j = 0; j < groups_.size(); ++j) {
        group& G = groups_[j];
        const int64_t n = B * G.maps * G.dims.vol();
        maxsz = std::max(maxsz, n);
        if (j > 0 && G.materialized) G.act = static_cast<float*>(dalloc(sizeof(float) * size_t(n)));
        if (cfg_.keep_images && G.materialized) G.grad = static_cast<float*>(dalloc(sizeof(float) * size_t(n)));
    }
    for (const auto& L : layers_) {
        group& G = groups_[size_t(L.out)];
        const size_t nv = size_t(B * G.maps * G.dims.vol());
        if (L.kind == lkind::pool) G.mask = static_cast<int32_t*>(dalloc(sizeof(int32_t) * nv));
        if (L.kind == lkind::filter) {
            require(L.k.vol() <= 256, "max-filter window exceeds 256 taps");
            G.code = static_cast<uint8_t*>(dalloc(nv));
        }
    }
    // a max-filter whose input is the ReLU output of a fused conv layer (and
    // its only consumer) folds that ReLU backward into its window codes; the
    // conv's backward then skips its own gate (ZNN_NO_RELU_FUSION=1: off)
    if (!std::getenv("ZNN_NO_RELU_FUSION")) {
        for (auto& F : layers_) {
            if (F.kind != lkind::filter || F.k.vol() > 128) continue;
            int consumers = 0;
            for (const auto& L2 : layers_) consumers += L2.in == F.in;
            for (auto& C : layers_)
                if (C.kind == lkind::conv && C.out == F.in && C.fused && C.fused_act == 2 &&
                    consumers == 1) {
                    F.relu_gate = true;
                    C.pregated = true;
                }
        }
    }
    if (!cfg_.keep_images) {
        gbuf_[0] = static_cast<float*>(dalloc(sizeof(float) * size_t(maxsz)));
        gbuf_[1] = static_cast<float*>(dalloc(sizeof(float) * size_t(maxsz)));
    }
    params_ = static_cast<float*>(dalloc(sizeof(float) * size_t(flat_)));
    grads_ = static_cast<float*>(dalloc(sizeof(float) * size_t(flat_)));
    vel_ = static_cast<float*>(dalloc(sizeof(float) * size_t(flat_)));
    ZNN_CUDA_CHECK(cudaMemsetAsync(params_, 0, sizeof(float) * size_t(flat_), st_));
    ZNN_CUDA_CHECK(cudaMemsetAsync(grads_, 0, sizeof(float) * size_t(flat_), st_));
    ZNN_CUDA_CHECK(cudaMemsetAsync(vel_, 0, sizeof(float) * size_t(flat_), st_));
    for (auto& L : layers_)
        if (!L.kinds.empty()) {
            L.kinds_dev = static_cast<int32_t*>(dalloc(sizeof(int32_t) * L.kinds.size()));
            ZNN_CUDA_CHECK(cudaMemcpy(L.kinds_dev, L.kinds.data(), sizeof(int32_t) * L.kinds.size(),
                                      cudaMemcpyHostToDevice));
            const std::vector<int32_t> none(L.kinds.size(), 3);
            L.none_dev = static_cast<int32_t*>(dalloc(sizeof(int32_t) * none.size()));
            ZNN_CUDA_CHECK(cudaMemcpy(L.none_dev, none.data(), sizeof(int32_t) * none.size(),
                                      cudaMemcpyHostToDevice));
        }
    const group& G = groups_.back();
    labels_perm_ = static_cast<float*>(dalloc(sizeof(float) * size_t(B * G.maps * G.dims.vol())));
    in_stage_ = static_cast<float*>(dalloc(sizeof(float) * size_t(in_per_patch() * B)));
    lab_stage_ = static_cast<float*>(dalloc(sizeof(float) * size_t(out_per_patch() * B)));
    loss_dev_ = static_cast<double*>(dalloc(sizeof(double)));
    groups_[0].act = in_stage_;
    // grad pointers for the ping-pong scheme: alternate by materialized ordinal
    if (!cfg_.keep_images) {
        int q = 0;
        for (size_t j = 0; j < groups_.size(); ++j)
            if (groups_[j].materialized) groups_[j].grad = gbuf_[(q++) & 1];
    }
    ZNN_CUDA_CHECK(cudaStreamSynchronize(st_));
}

int64_t executor::in_per_patch() const { return groups_.front().maps * groups_.front().dims.vol(); }
int64_t executor::out_per_patch() const { return groups_.back().maps * groups_.back().dims.vol(); }

void executor::set_params(const float* host) {
    std::vector<float> flat(size_t(flat_), 0.f);
    for (size_t c = 0; c < canon_.size(); ++c) flat[size_t(canon_[c])] = host[c];
    ZNN_CUDA_CHECK(cudaMemcpyAsync(params_, flat.data(), sizeof(float) * size_t(flat_), cudaMemcpyHostToDevice, st_));
    ZNN_CUDA_CHECK(cudaStreamSynchronize(st_));
}

void executor::get_params(float* host) {
    std::vector<float> flat(static_cast<size_t>(flat_));
    ZNN_CUDA_CHECK(cudaMemcpyAsync(flat.data(), params_, sizeof(float) * size_t(flat_), cudaMemcpyDeviceToHost, st_));
    ZNN_CUDA_CHECK(cudaStreamSynchronize(st_));
    for (size_t c = 0; c < canon_.size(); ++c) host[c] = flat[size_t(canon_[c])];
}

void executor::get_gradients(float* host) {
    std::vector<float> flat(static_cast<size_t>(flat_));
    ZNN_CUDA_CHECK(cudaMemcpyAsync(flat.data(), grads_, sizeof(float) * size_t(flat_), cudaMemcpyDeviceToHost, st_));
    ZNN_CUDA_CHECK(cudaStreamSynchronize(st_));
    for (size_t c = 0; c < canon_.size(); ++c) host[c] = flat[size_t(canon_[c])];
}

void executor::reset_momentum() {
    ZNN_CUDA_CHECK(cudaMemsetAsync(vel_, 0, sizeof(float) * size_t(flat_), st_));
}

void executor::set_layer_engine(int conv_layer, int engine) {
    int ci = 0;
    for (auto& L : layers_)
        if (L.kind == lkind::conv) {
            if (ci == conv_layer) {
                require(engine == 0 || engine == 1 || engine == 3, "set_layer_engine: unknown engine");
                if (L.engine != engine) drop_fft_plans();  // the spectra memory plan depends on the engines
                L.engine = engine;
                return;
            }
            ++ci;
        }
    throw znn_gpu::shape_error("set_layer_engine: no conv layer " + std::to_string(conv_layer));
}

// Memory plan of the FFT layers' kernel spectra (the big per-layer object,
// f*f'*bins complex: 52 GB for c5 conv2). At the first FFT plan the budget
// for all kernel spectra (shared buffer + resident) is taken from
// cudaMemGetInfo: free memory minus every FFT layer's memoised image spectra,
// the largest FFT scratch need and a headroom (ZNN_MEM_HEADROOM_GB, 20).
// Layers keep their own spectra (the reference's memo) unless the sum does
// not fit; then the largest layers share one buffer (kpool) and a layer whose
// spectra were overwritten since its forward recomputes them in the backward
// pass. ZNN_FFT_RESIDENT_GB overrides the budget (0 = all layers share).
void executor::plan_fft_memory() {
    fft_decided_ = true;
    fft_pool_members_.clear();
    std::vector<std::pair<int64_t, const layer*>> sz;
    int64_t total = 0, xspec = 0, wsmax = 0, phmax = 0;
    for (const auto& M : layers_)
        if (M.kind == lkind::conv && M.engine == 1 && znn_fft::supported(M.shape)) {
            sz.emplace_back(znn_fft::kernel_spectrum_bytes(M.shape), &M);
            total += sz.back().first;
            xspec += znn_fft::image_spectrum_bytes(M.shape);
            wsmax = std::max(wsmax, znn_fft::workspace_bytes(M.shape));
            phmax = std::max(phmax, znn_fft::phase_bytes(M.shape));
        }
    if (sz.empty()) return;
    std::sort(sz.begin(), sz.end(), [](const auto& a, const auto& b) { return a.first > b.first; });
    if (const char* e = std::getenv("ZNN_FFT_RESIDENT_GB")) {
        fft_budget_ = std::atof(e) * double(int64_t(1) << 30);
    } else {
        size_t fr = 0, tot = 0;
        ZNN_CUDA_CHECK(cudaMemGetInfo(&fr, &tot));
        double head = 20.0;
        if (const char* h = std::getenv("ZNN_MEM_HEADROOM_GB")) head = std::atof(h);
        const double have = double(fr) + double(ws_.capacity());  // the arena is re-grown to wsmax
        fft_budget_ = have - double(xspec) - double(wsmax) * 1.25 - double(phmax) -
                      head * double(int64_t(1) << 30);
    }
    // smallest j: the j largest layers share one buffer (its size = the
    // largest), the others stay resident; j = 1 saves nothing over j = 0
    const size_t n = sz.size();
    size_t j = 0;
    double rest = double(total);
    for (; j <= n; ++j) {
        const double mem = (j == 0 ? 0.0 : double(sz[0].first)) + rest;
        if (j != 1 && mem <= fft_budget_) break;
        if (j < n) rest -= double(sz[j].first);
    }
    if (j > n) j = n;  // nothing fits: every FFT layer shares the buffer
    for (size_t q = 0; q < j; ++q) fft_pool_members_.push_back(sz[q].second);
}

bool executor::fft_pooled(const layer& L) {
    const bool member = &L >= layers_.data() && &L < layers_.data() + layers_.size();
    if (!member) return false;  // autotune trial copies own their spectra
    if (!fft_decided_) plan_fft_memory();
    return std::find(fft_pool_members_.begin(), fft_pool_members_.end(), &L) != fft_pool_members_.end();
}

void executor::drop_fft_plans() {
    drop_graph();
    for (auto& L : layers_) L.fft.reset();
    kpool_.reset();
    phase_ws_.reset();
    fft_decided_ = false;
}

void executor::drop_graph() {
    for (auto& g : graphs_) cudaGraphExecDestroy(g.exec);
    graphs_.clear();
    graph_warm_ = 0;
    ws_.freeze(false);
}

void executor::set_graph_mode(bool on) {
    if (!on) drop_graph();
    graph_mode_ = on;
}

double executor::train_step(const float* in, const float* lab, bool sync_loss) {
    if (!graph_mode_ || st_ == nullptr)  // the legacy default stream cannot be captured
        return forward_backward(in, lab, sync_loss, true);
    if (graph_warm_ < 1) {  // first step eager: plans, spectra buffers and the arena reach full size
        ++graph_warm_;
        return forward_backward(in, lab, sync_loss, true);
    }
    cudaGraphExec_t exec = nullptr;
    for (const auto& g : graphs_)
        if (g.in == in && g.lab == lab) exec = g.exec;
    if (!exec) {
        if (graphs_.size() >= 4) {  // bounded cache: start over
            for (auto& g : graphs_) cudaGraphExecDestroy(g.exec);
            graphs_.clear();
        }
        ws_.freeze(true);
        cudaGraph_t g = nullptr;
        ZNN_CUDA_CHECK(cudaStreamBeginCapture(st_, cudaStreamCaptureModeRelaxed));
        try {
            forward_backward(in, lab, false, true);
        } catch (...) {
            cudaStreamEndCapture(st_, &g);
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
            ws_.freeze(false);
            throw;
        }
        ZNN_CUDA_CHECK(cudaStreamEndCapture(st_, &g));
        const cudaError_t ie = cudaGraphInstantiate(&exec, g, 0);
        cudaGraphDestroy(g);
        if (ie != cudaSuccess) {
            ws_.freeze(false);
            throw znn_gpu::cuda_error(std::string("cudaGraphInstantiate: ") + cudaGetErrorString(ie));
        }
        graphs_.push_back(step_graph{in, lab, exec});
    }
    ZNN_CUDA_CHECK(cudaGraphLaunch(exec, st_));
    return sync_loss ? last_loss_device() : 0.0;
}

znn_fft::plan& executor::fft_plan(layer& L) {
    if (!L.fft) {
        std::shared_ptr<znn_fft::kpool> pool;
        if (fft_pooled(L)) {
            if (!kpool_) kpool_ = std::make_shared<znn_fft::kpool>();
            pool = kpool_;
        }
        if (!phase_ws_) phase_ws_ = std::make_shared<znn_gpu::scratch>();
        L.fft = std::shared_ptr<znn_fft::plan>(znn_fft::make_plan(L.shape, pool, phase_ws_).release(),
                                               znn_fft::plan_deleter());
    }
    return *L.fft;
}

bool executor::fft_counts(int conv_layer, znn_fft::transform_counts& out) const {
    int ci = 0;
    for (const auto& L : layers_)
        if (L.kind == lkind::conv) {
            if (ci++ == conv_layer) {
                if (!L.fft) return false;
                out = znn_fft::counts(*L.fft);
                return true;
            }
        }
    return false;
}

void executor::run_conv_fwd(layer& L) {
    const float* x = groups_[size_t(L.in)].act;
    float* y = groups_[size_t(L.out)].act;
    const float* w = params_ + L.w_off;
    const float* bias = L.fused ? params_ + L.b_off : nullptr;
    const int act = L.fused ? L.fused_act : 3;
    if (L.engine == 1) {
        znn_fft::conv_fwd(st_, fft_plan(L), L.shape, x, w, bias, act, y, ws_, groups_[size_t(L.in)].pm,
                          groups_[size_t(L.out)].pm);
    } else if (L.engine == 0 && znn_gpu::conv_tc_supported(L.shape, 0)) {
        znn_gpu::conv_fwd_tc(st_, L.shape, x, w, bias, act, y, ws_);
    } else {
        znn_gpu::conv_fwd_simt(st_, L.shape, x, w, bias, act, y);
    }
}

void executor::run_conv_bwd(layer& L, float* g_out, float* g_in, bool need_dgrad, bool update, const float* relu_y,
                            float* dbias) {
    const float* x = groups_[size_t(L.in)].act;
    float* w = params_ + L.w_off;
    float* gw = grads_ + L.w_off;
    const int64_t wcount = L.shape.f_out * L.shape.f_in * L.shape.taps();
    if (L.engine == 1) {
        znn_fft::conv_bwd(st_, fft_plan(L), L.shape, x, g_out, w, gw, need_dgrad ? g_in : nullptr, ws_, relu_y, dbias,
                          groups_[size_t(L.in)].pm, groups_[size_t(L.out)].pm);
        if (update) znn_gpu::sgd_momentum(st_, w, vel_ + L.w_off, gw, wcount, cfg_.lr, cfg_.mu);
        return;
    }
    const bool tc = L.engine == 0;
    auto dgrad = [&] {
        if (tc && znn_gpu::conv_tc_supported(L.shape, 1))
            znn_gpu::conv_dgrad_tc(st_, L.shape, g_out, w, g_in, ws_);
        else
            znn_gpu::conv_dgrad_simt(st_, L.shape, g_out, w, g_in);
    };
    // with the update fused, the data gradient must read the weights first
    if (need_dgrad && update) dgrad();
    if (tc && znn_gpu::conv_tc_supported(L.shape, 2)) {
        znn_gpu::sgd_fuse upd{w, vel_ + L.w_off, cfg_.lr, cfg_.mu};
        znn_gpu::conv_wgrad_tc(st_, L.shape, x, g_out, gw, 1.f, ws_, update ? &upd : nullptr);
    } else {
        znn_gpu::conv_wgrad_simt(st_, L.shape, x, g_out, gw, 1.f, ws_);
        if (update) znn_gpu::sgd_momentum(st_, w, vel_ + L.w_off, gw, wcount, cfg_.lr, cfg_.mu);
    }
    if (need_dgrad && !update) dgrad();
}

// Tensor order of the groups between FFT layers. A convolution with sparsity
// s maps phase r of its input (voxels s q + r) to phase r of its output, so a
// group written by one polyphase FFT layer and read by another of the same
// sparsity (c5: conv3 -> conv4 -> conv5, s = 4) stays phase-major: both
// layers' transforms then read / write dense phase images with whole-sector
// vector accesses instead of every s-th float of the interleaved tensor, and
// so do the gradient of that group and the fused ReLU gate. Nothing else may
// touch the group: the producer's transfer is fused (ReLU gate inside the
// gradient transform) or absent. A 2^3 max-filter feeding an FFT layer writes
// its output (and reads its gradient) in that layer's phase order too
// (ZNN_PHASE_MAJOR_FILTER=0: not). ZNN_PHASE_MAJOR=0: natural order everywhere.
void executor::plan_layouts() {
    const char* env = std::getenv("ZNN_PHASE_MAJOR");
    const bool on = !(env && std::string(env) == "0") && !cfg_.keep_images;
    const bool relu_fusion = !std::getenv("ZNN_NO_RELU_FUSION");
    const char* fenv = std::getenv("ZNN_PHASE_MAJOR_FILTER");
    const bool filter_pm = !(fenv && std::string(fenv) == "0");
    std::string note;
    for (size_t j = 1; j + 1 < groups_.size(); ++j) {
        group& G = groups_[j];
        const layer *A = nullptr, *C = nullptr;
        int np = 0, nc = 0;
        for (const auto& L : layers_) {
            if (L.out == int(j)) A = &L, ++np;
            if (L.in == int(j)) C = &L, ++nc;
        }
        const bool consumer_ok = on && G.materialized && np == 1 && nc == 1 && C->kind == lkind::conv &&
                                 C->engine == 1 && znn_fft::supported(C->shape) && znn_fft::phase_major_ok(C->shape);
        bool pm = false;
        if (consumer_ok && A->kind == lkind::conv) {
            pm = A->engine == 1 && znn_fft::supported(A->shape) && znn_fft::phase_major_ok(A->shape) &&
                 A->shape.s.x == C->shape.s.x && A->shape.s.y == C->shape.s.y && A->shape.s.z == C->shape.s.z &&
                 (!A->fused || (A->fused_act == 2 && relu_fusion && !A->pregated));
        } else if (consumer_ok && A->kind == lkind::filter && filter_pm) {
            // a 2^3 max-filter writes its output / reads its gradient in the consumer's phase order
            const int64_t sz = C->shape.s.z;
            pm = znn_fft::phase_major_pays(C->shape) && A->k.x == 2 && A->k.y == 2 && A->k.z == 2 &&
                 (A->s.x == 1 || A->s.x == 2) && G.code != nullptr && 32 % sz == 0 &&
                 cfg_.batch * G.maps < 65536 && (sz & (sz - 1)) == 0;
        }
        if (pm != G.pm) drop_graph();
        G.pm = pm;
        G.pm_s = pm ? C->shape.s : dims3{1, 1, 1};
        if (pm) note += " " + std::to_string(j);
    }
    if (note != layout_note_) {
        layout_note_ = note;
        if (!note.empty()) desc_ += "phase-major groups:" + note + "\n";
    }
}

void executor::run_forward(const float* in_dev) {
    plan_layouts();
    groups_[0].act = const_cast<float*>(in_dev);
    const int64_t B = cfg_.batch;
    for (auto& L : layers_) {
        const group& I = groups_[size_t(L.in)];
        group& O = groups_[size_t(L.out)];
        switch (L.kind) {
            case lkind::conv: run_conv_fwd(L); break;
            case lkind::transfer:
                znn_gpu::transfer_fwd(st_, I.act, B, I.maps, I.dims.vol(), L.kinds_dev, params_ + L.b_off, O.act);
                break;
            case lkind::pool: znn_gpu::maxpool_fwd(st_, I.act, B * I.maps, I.dims, L.k, O.act, O.mask); break;
            case lkind::filter:
                znn_gpu::maxfilter_fwd(st_, I.act, B * I.maps, I.dims, L.k, L.s, O.act, O.code, L.relu_gate,
                                       znn_gpu::pm_order{O.pm ? 1 : 0, int(O.maps), O.pm_s});
                break;
        }
    }
}

void executor::forward(const float* in_dev) { run_forward(in_dev); }

double executor::forward_backward(const float* in_dev, const float* labels_dev, bool sync_loss, bool update) {
    const int64_t B = cfg_.batch;
    run_forward(in_dev);
    group& G = groups_.back();
    const int64_t vol = G.dims.vol();
    const float* lab = labels_dev;
    if (!out_identity_) {
        for (int64_t b = 0; b < B; ++b)
            for (int64_t p = 0; p < G.maps; ++p)
                ZNN_CUDA_CHECK(cudaMemcpyAsync(labels_perm_ + (b * G.maps + p) * vol,
                                               labels_dev + (b * G.maps + out_perm_[size_t(p)]) * vol,
                                               sizeof(float) * size_t(vol), cudaMemcpyDeviceToDevice, st_));
        lab = labels_perm_;
    }
    znn_gpu::loss_grad_async(st_, cfg_.loss, G.act, lab, B * G.maps * vol, 1.f / float(cfg_.global_batch),
                             G.grad, loss_dev_, ws_);
    // parameters of a layer are contiguous in the flat buffer: conv weights
    // [f_out][f_in][T] then the fused transfer's biases; a transfer layer's biases
    auto grad_ready = [&](const layer& L) {
        if (!grad_hook_) return;
        if (L.kind == lkind::conv)
            grad_hook_(L.w_off, L.shape.f_out * L.shape.f_in * L.shape.taps() + (L.fused ? L.shape.f_out : 0));
        else if (L.kind == lkind::transfer)
            grad_hook_(L.b_off, int64_t(L.edge_ids.size()));
    };
    // backward in reverse layer order
    for (size_t li = layers_.size(); li-- > 0;) {
        layer& L = layers_[li];
        group& I = groups_[size_t(L.in)];
        group& O = groups_[size_t(L.out)];
        const bool last = li + 1 == layers_.size();
        const bool ce_here = last && cfg_.loss == 1;
        switch (L.kind) {
            case lkind::conv: {
                // FFT layers with a fused ReLU gate the gradient inside their
                // spectrum pass and take the bias gradient from its DC term
                // (no separate transfer-backward pass over the activations)
                const bool fuse_relu = L.fused && L.engine == 1 && !ce_here && L.fused_act == 2 &&
                                       !std::getenv("ZNN_NO_RELU_FUSION");
                if (fuse_relu) {
                    // (bias_summed: the max-filter backward above already left this layer's bias gradient)
                    run_conv_bwd(L, O.grad, I.grad, L.in != 0, update, L.pregated ? nullptr : O.act,
                                 L.bias_summed ? nullptr : grads_ + L.b_off);
                    L.bias_summed = false;
                    if (update)
                        znn_gpu::sgd_momentum(st_, params_ + L.b_off, vel_ + L.b_off, grads_ + L.b_off,
                                              L.shape.f_out, cfg_.lr, cfg_.mu);
                    grad_ready(L);
                    break;
                }
                if (L.fused) {
                    // ce: loss already produced the pre-activation gradient a - d
                    if (ce_here) {
                        znn_gpu::transfer_bwd(st_, O.grad, O.act, true, B, L.shape.f_out, O.dims.vol(),
                                              L.none_dev, params_ + L.b_off, O.grad, grads_ + L.b_off, ws_);
                    } else if (L.bias_summed) {
                        L.bias_summed = false;  // the max-filter backward above left the bias gradient
                    } else {
                        // pregated (the max-filter's codes applied this ReLU's backward): the
                        // gradient is final, only its per-map sums (the bias gradient) remain
                        const bool sum_only = L.pregated && L.fused_act == 2;
                        znn_gpu::transfer_bwd(st_, O.grad, sum_only ? nullptr : O.act, true, B, L.shape.f_out,
                                              O.dims.vol(), L.kinds_dev, params_ + L.b_off, O.grad,
                                              grads_ + L.b_off, ws_);
                    }
                }
                // the bias gradient is final here (transfer_bwd above): update it
                if (update && L.fused)
                    znn_gpu::sgd_momentum(st_, params_ + L.b_off, vel_ + L.b_off, grads_ + L.b_off,
                                          L.shape.f_out, cfg_.lr, cfg_.mu);
                run_conv_bwd(L, O.grad, I.grad, L.in != 0, update);
                grad_ready(L);
                break;
            }
            case lkind::transfer:
                znn_gpu::transfer_bwd(st_, O.grad, I.act, false, B, I.maps, I.dims.vol(),
                                      ce_here ? L.none_dev : L.kinds_dev, params_ + L.b_off,
                                      I.grad ? I.grad : O.grad, grads_ + L.b_off, ws_);
                if (update)
                    znn_gpu::sgd_momentum(st_, params_ + L.b_off, vel_ + L.b_off, grads_ + L.b_off, I.maps,
                                          cfg_.lr, cfg_.mu);
                grad_ready(L);
                break;
            case lkind::pool:
                if (L.in != 0) znn_gpu::maxpool_bwd(st_, O.grad, O.mask, B * I.maps, O.dims, L.k, I.grad);
                break;
            case lkind::filter:
                if (L.in != 0) {
                    // the conv layer below with a fused ReLU whose backward this filter's codes
                    // carry: its bias gradient is the per-map sum of the gradient written here,
                    // taken from the kernel's per-block partial sums (no extra pass over it)
                    layer* below = nullptr;
                    const int64_t cols = znn_gpu::maxfilter_bwd_sum_cols(O.dims, L.k, L.s);
                    // (the phase-major variant keeps its registers; the inspection mode keeps the
                    // plain sum-only pass, whose summation order does not depend on the tensor order)
                    if (L.relu_gate && cols > 0 && B * I.maps < 65536 && !O.pm && !cfg_.keep_images)
                        for (auto& C : layers_)
                            // (an FFT layer takes its bias gradient from the DC bins of the
                            // gradient spectra it forms anyway, in double)
                            if (C.kind == lkind::conv && C.out == L.in && C.pregated && C.fused && C.fused_act == 2 &&
                                C.engine != 1)
                                below = &C;
                    float* part = below ? static_cast<float*>(ws_.get(sizeof(float) * size_t(B * I.maps * cols)))
                                        : nullptr;
                    znn_gpu::maxfilter_bwd(st_, O.grad, O.code, B * I.maps, O.dims, L.k, L.s, I.grad,
                                           znn_gpu::pm_order{O.pm ? 1 : 0, int(O.maps), O.pm_s}, part, int(I.maps));
                    if (below) {
                        znn_gpu::reduce_rows(st_, part, I.maps, B * cols, grads_ + below->b_off);
                        below->bias_summed = true;
                    }
                }
                break;
        }
    }
    if (!sync_loss) return 0.0;
    return last_loss_device();
}

double executor::last_loss_device() {
    double h = 0.0;
    ZNN_CUDA_CHECK(cudaMemcpyAsync(&h, loss_dev_, sizeof(double), cudaMemcpyDeviceToHost, st_));
    ZNN_CUDA_CHECK(cudaStreamSynchronize(st_));
    return h / double(cfg_.batch);
}

void executor::apply_update() { znn_gpu::sgd_momentum(st_, params_, vel_, grads_, flat_, cfg_.lr, cfg_.mu); }

double executor::step_host(const float* in_host, const float* labels_host) {
    const int64_t B = cfg_.batch;
    ZNN_CUDA_CHECK(cudaMemcpyAsync(in_stage_, in_host, sizeof(float) * size_t(B * in_per_patch()), cudaMemcpyHostToDevice, st_));
    ZNN_CUDA_CHECK(cudaMemcpyAsync(lab_stage_, labels_host, sizeof(float) * size_t(B * out_per_patch()), cudaMemcpyHostToDevice, st_));
    train_step(in_stage_, lab_stage_, false);
    return last_loss_device();
}

void executor::copy_outputs(float* host) {
    const group& G = groups_.back();
    const int64_t vol = G.dims.vol();
    std::vector<float> tmp(size_t(cfg_.batch * G.maps * vol));
    ZNN_CUDA_CHECK(cudaMemcpyAsync(tmp.data(), G.act, sizeof(float) * tmp.size(), cudaMemcpyDeviceToHost, st_));
    ZNN_CUDA_CHECK(cudaStreamSynchronize(st_));
    for (int64_t b = 0; b < cfg_.batch; ++b)
        for (int64_t p = 0; p < G.maps; ++p)
            std::memcpy(host + (b * G.maps + out_perm_[size_t(p)]) * vol, tmp.data() + (b * G.maps + p) * vol,
                        sizeof(float) * size_t(vol));
}

void executor::group_image(int gi, int which, float* host) {
    const group& G = groups_.at(size_t(gi));
    require(G.materialized, "group image: group " + std::to_string(gi) + " is fused away");
    const float* src = which == 0 ? G.act : G.grad;
    require(src != nullptr, "group image: image not available");
    const int64_t total = cfg_.batch * G.maps * G.dims.vol();
    if (!G.pm) {
        ZNN_CUDA_CHECK(cudaMemcpyAsync(host, src, sizeof(float) * size_t(total), cudaMemcpyDeviceToHost, st_));
        ZNN_CUDA_CHECK(cudaStreamSynchronize(st_));
        return;
    }
    // phase-major group: back to [B][maps][x][y][z] on the host
    std::vector<float> pmv(static_cast<size_t>(total));
    ZNN_CUDA_CHECK(cudaMemcpyAsync(pmv.data(), src, sizeof(float) * size_t(total), cudaMemcpyDeviceToHost, st_));
    ZNN_CUDA_CHECK(cudaStreamSynchronize(st_));
    const dims3 s = G.pm_s, n = G.dims, q{n.x / s.x, n.y / s.y, n.z / s.z};
    const int64_t S = s.vol();
    for (int64_t b = 0; b < cfg_.batch; ++b)
        for (int64_t m = 0; m < G.maps; ++m)
            for (int64_t x = 0; x < n.x; ++x)
                for (int64_t y = 0; y < n.y; ++y)
                    for (int64_t z = 0; z < n.z; ++z) {
                        const int64_t r = ((x % s.x) * s.y + (y % s.y)) * s.z + (z % s.z);
                        const int64_t img = (b * S + r) * G.maps + m;
                        host[((b * G.maps + m) * n.x + x) * n.y * n.z + y * n.z + z] =
                            pmv[size_t(((img * q.x + x / s.x) * q.y + y / s.y) * q.z + z / s.z)];
                    }
}

void executor::group_mask(int gi, int32_t* host) {
    const group& G = groups_.at(size_t(gi));
    require(G.mask != nullptr || G.code != nullptr,
            "group mask: group " + std::to_string(gi) + " has no argmax record");
    const int64_t n = cfg_.batch * G.maps * G.dims.vol();
    if (G.mask) {
        ZNN_CUDA_CHECK(cudaMemcpyAsync(host, G.mask, sizeof(int32_t) * size_t(n), cudaMemcpyDeviceToHost, st_));
        ZNN_CUDA_CHECK(cudaStreamSynchronize(st_));
        return;
    }
    // max-filter window codes -> the reference's flat input index per output voxel
    std::vector<uint8_t> code(static_cast<size_t>(n));
    ZNN_CUDA_CHECK(cudaMemcpyAsync(code.data(), G.code, size_t(n), cudaMemcpyDeviceToHost, st_));
    ZNN_CUDA_CHECK(cudaStreamSynchronize(st_));
    const layer* P = nullptr;
    for (const auto& L : layers_)
        if (L.kind == lkind::filter && L.out == gi) P = &L;
    require(P != nullptr, "group mask: no max-filter produces group " + std::to_string(gi));
    const dims3 in = groups_[size_t(P->in)].dims, m = G.dims, k = P->k, s = P->s;
    const int64_t mv = m.vol();
    for (int64_t e = 0; e < n; ++e) {
        const int64_t v = e % mv;
        const int64_t i = v / (m.y * m.z), j = (v / m.z) % m.y, l = v % m.z;
        const int c = code[size_t(e)] & 0x7F;  // (bit 7: the ReLU gate, not part of the argmax)
        const int64_t a = c / (k.y * k.z), b = (c / k.z) % k.y, cz = c % k.z;
        host[e] = int32_t(((i + s.x * a) * in.y + (j + s.y * b)) * in.z + (l + s.z * cz));
    }
}

std::vector<int> executor::autotune(int trials) {
    require(trials >= 1, "autotune: trials must be >= 1");
    std::vector<int> chosen;
    cudaEvent_t a, b;
    ZNN_CUDA_CHECK(cudaEventCreate(&a));
    ZNN_CUDA_CHECK(cudaEventCreate(&b));
    std::ostringstream report;  // appended to describe(): per-layer median fwd+bwd+upd times
    for (auto& G : groups_) G.pm = false;  // candidates are timed on natural-order tensors
    int ci = 0;
    for (auto& L : layers_) {
        if (L.kind != lkind::conv) continue;
        report << "autotune conv#" << ci++ << " (median of " << trials << "):";
        // candidate engines: tensor-core direct, SIMT direct, FFT
        std::vector<int> cands{0};
        if (znn_fft::supported(L.shape)) cands.push_back(1);
        // the SIMT engine is for thin layers; on wide ones it is 10-40x off the
        // tensor-core engine (c5 conv2: 6.8 s vs 0.44 s) and only costs time
        if (L.shape.f_in * L.shape.f_out <= 1024) cands.push_back(3);
        // scratch inputs for the bwd pass: reuse the layer's own buffers
        float* gout = groups_[size_t(L.out)].grad;
        float* gin = groups_[size_t(L.in)].grad;
        float best = 1e30f;
        int best_e = L.engine;
        for (int e : cands) {
            layer T = L;
            T.engine = e;
            std::vector<float> ts;
            try {
                for (int t = 0; t <= trials; ++t) {
                    ZNN_CUDA_CHECK(cudaEventRecord(a, st_));
                    run_conv_fwd(T);
                    run_conv_bwd(T, gout, gin, L.in != 0, false);
                    ZNN_CUDA_CHECK(cudaEventRecord(b, st_));
                    ZNN_CUDA_CHECK(cudaEventSynchronize(b));
                    float ms = 0.f;
                    ZNN_CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
                    if (t > 0) ts.push_back(ms);  // first run warms plans and scratch
                    // a candidate whose first timed run is already 4x the best so far
                    // cannot win: skip its other trials (SIMT on a 120->120 layer
                    // takes seconds; the warm-up run also pays plan allocation)
                    if (t == 1 && ms > 4.f * best) break;
                }
            } catch (const std::exception& ex) {
                // a candidate that cannot run this layer (launch limits, memory)
                // drops out instead of failing the whole autotune
                cudaGetLastError();
                cudaStreamSynchronize(st_);
                report << " " << ename(e) << " failed(" << ex.what() << ")";
                continue;
            }
            std::sort(ts.begin(), ts.end());
            const float med = ts[ts.size() / 2];
            report << (e == 0 ? " direct " : e == 1 ? " fft " : " direct-simt ") << med << "ms"
                   << (ts.size() == 1 && trials > 1 ? "(pruned)" : "");
            if (med < best) best = med, best_e = e;
        }
        report << " -> " << ename(best_e) << "\n";
        if (L.engine != best_e) drop_fft_plans();
        L.engine = best_e;
        chosen.push_back(best_e);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    desc_ += report.str();
    // the timing runs overwrote activations/gradients: not a training step
    return chosen;
}

}  // namespace znn_exec
