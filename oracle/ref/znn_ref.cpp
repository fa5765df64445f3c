// Driver around the REFERENCE implementation (compiled from /root/reference
// with the Eigen-subset shim; see build.sh). TEST / BASELINE INFRASTRUCTURE
// ONLY — never linked into the product.
//
//   znn_ref bench <spec> <x,y,z> <threads> <warmup> <rounds> <direct|auto|fft> [budget_s]
//       times the reference task engine (engine<float>, engine.hpp:65-254) on
//       one patch per round: <warmup> rounds in one run(), then <rounds>
//       measured rounds (one run() each, wall time around each; stops early
//       once budget_s would be exceeded); prints {"rounds","warmup","seconds",
//       "round_seconds",...} JSON
//   znn_ref tune <spec> <x,y,z> <trials>
//       the reference's autotune_modes (trainer.hpp:181-250): per-signature
//       direct / FFT times and choices
//   znn_ref estimate <spec> <x,y,z> <threads>
//       per-edge task-body timing of one round, extrapolated (see estimate())
//   znn_ref round <spec> <x,y,z> <params.f64> <inputs.f64> <labels.f64> <eta> <out.f64>
//       one straight-line training round of the reference's own oracle
//       (tests/oracles.hpp:155-252) in double; writes [loss, params...]
//   znn_ref maxfilter <in.f64> <nx,ny,nz> <k> <s> <out.f64> <rec.i32>
//       maxfilter_forward (maxops.hpp:111-164): values + argmax record
//   znn_ref conv <x.f64> <n> <w.f64> <k> <s> <out.f64>
//       conv_valid_direct (conv_direct.hpp:39-68)
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "oracles.hpp"
#include "znn/engine.hpp"
#include "znn/netspec.hpp"
#include "znn/trainer.hpp"

using namespace znn;

namespace {

std::string read_file(const std::string& p) {
    std::ifstream is(p);
    std::stringstream ss;
    ss << is.rdbuf();
    return ss.str();
}

vec3i v3(const std::string& s) {
    vec3i v;
    char c1, c2;
    std::istringstream is(s);
    is >> v.x >> c1 >> v.y >> c2 >> v.z;
    return v;
}

template <typename T>
std::vector<T> read_bin(const std::string& p) {
    std::ifstream is(p, std::ios::binary);
    is.seekg(0, std::ios::end);
    const auto bytes = is.tellg();
    is.seekg(0);
    std::vector<T> v(size_t(bytes) / sizeof(T));
    is.read(reinterpret_cast<char*>(v.data()), bytes);
    return v;
}

template <typename T>
void write_bin(const std::string& p, const std::vector<T>& v) {
    std::ofstream os(p, std::ios::binary);
    os.write(reinterpret_cast<const char*>(v.data()), std::streamsize(v.size() * sizeof(T)));
}

template <typename T>
void set_params(net_graph<T>& g, const std::vector<double>& p) {
    size_t off = 0;
    for (auto& e : g.edges) {
        if (auto* c = std::get_if<conv_op<T>>(&e.op))
            for (std::int64_t i = 0; i < c->k.weights.size(); ++i) c->k.weights[i] = T(p.at(off++));
        else if (auto* t = std::get_if<transfer_op<T>>(&e.op))
            t->fn.bias = T(p.at(off++));
    }
}

template <typename T>
std::vector<double> get_params(const net_graph<T>& g) {
    std::vector<double> out;
    for (const auto& e : g.edges) {
        if (auto* c = std::get_if<conv_op<T>>(&e.op))
            for (std::int64_t i = 0; i < c->k.weights.size(); ++i) out.push_back(double(c->k.weights[i]));
        else if (auto* t = std::get_if<transfer_op<T>>(&e.op))
            out.push_back(double(t->fn.bias));
    }
    return out;
}

int bench(int argc, char** argv) {
    const std::string spec = read_file(argv[2]);
    const vec3i od = v3(argv[3]);
    const int threads = std::atoi(argv[4]);
    const int warmup = std::atoi(argv[5]);
    const int rounds = std::atoi(argv[6]);
    const std::string mode = argv[7];
    const double budget = argc > 8 ? std::atof(argv[8]) : 1e30;
    auto g = parse_netspec<float>(spec, od);
    init_weights(g, 1);

    // one synthetic sample: inputs uniform[0,1), desired Bernoulli(0.5) (the
    // data content does not affect the cost of a round)
    std::mt19937 rng(7);
    typename engine<float>::sample smp;
    for (const auto& n : g.nodes) {
        if (n.role == node_role::input) {
            auto v = make_volume<float>(n.dims);
            fill_uniform(*v, rng, 0.f, 1.f);
            smp.inputs.push_back(std::move(v));
        }
    }
    std::bernoulli_distribution coin(0.5);
    for (const auto& n : g.nodes)
        if (n.role == node_role::output) {
            auto v = make_volume<float>(n.dims);
            for (std::int64_t i = 0; i < v->size(); ++i) (*v)[i] = coin(rng) ? 1.f : 0.f;
            smp.desired.push_back(std::move(v));
        }
    typename engine<float>::sample_source src = [&](std::int64_t) -> const typename engine<float>::sample& {
        return smp;
    };

    typename engine<float>::config cfg;
    cfg.threads = threads;
    cfg.memoize = true;
    cfg.learning_rate = 0.01f;
    std::string chosen = "direct";
    using clk = std::chrono::steady_clock;
    double tune_s = 0;
    if (mode == "fft") {
        cfg.edge_modes.assign(g.edges.size(), conv_engine::fft);
        chosen = "fft";
    } else if (mode == "auto") {
        const auto t0 = clk::now();
        cfg.edge_modes = autotune_modes(g, 3);  // the reference's default policy (trainer.hpp:41)
        tune_s = std::chrono::duration<double>(clk::now() - t0).count();
        int nf = 0;
        for (auto m : cfg.edge_modes) nf += m == conv_engine::fft;
        chosen = "auto(" + std::to_string(nf) + " fft edges)";
    }
    engine<float> eng(g, compute_priorities(g), cfg);
    // warm-up rounds (pools, plans) in one pipelined run, as train() runs them
    auto t0 = clk::now();
    if (warmup > 0) eng.run(warmup, src);
    const double warm = std::chrono::duration<double>(clk::now() - t0).count();
    // measured rounds one run() call each (no overlap with the warm-up or
    // each other), wall time around each; stop early past the budget
    std::vector<double> per;
    t0 = clk::now();
    for (int r = 0; r < rounds; ++r) {
        const auto a = clk::now();
        eng.run(1, src);
        per.push_back(std::chrono::duration<double>(clk::now() - a).count());
        if (std::chrono::duration<double>(clk::now() - t0).count() + warm + per.back() > budget) break;
    }
    const double sec = std::chrono::duration<double>(clk::now() - t0).count();
    std::printf("{\"rounds\": %zu, \"warmup\": %d, \"seconds\": %.6f, \"warmup_seconds\": %.6f, "
                "\"autotune_seconds\": %.3f, \"threads\": %d, \"mode\": \"%s\", \"round_seconds\": [",
                per.size(), warmup, sec, warm, tune_s, threads, chosen.c_str());
    for (size_t i = 0; i < per.size(); ++i) std::printf("%s%.4f", i ? ", " : "", per[i]);
    std::printf("]}\n");
    return 0;
}

// The reference's own layerwise autotuner (autotune_modes, trainer.hpp:
// 181-250) on a netspec: per signature the direct and FFT fwd+bwd+upd
// times and the choice, without running a round.
int tune(int argc, char** argv) {
    const std::string spec = read_file(argv[2]);
    auto g = parse_netspec<float>(spec, v3(argv[3]));
    init_weights(g, 1);
    std::vector<autotune_choice<float>> rep;
    auto modes = autotune_modes(g, std::atoi(argv[4]), &rep);
    int nf = 0;
    for (auto m : modes) nf += m == conv_engine::fft;
    std::printf("{\"fft_edges\": %d, \"signatures\": [", nf);
    for (size_t i = 0; i < rep.size(); ++i)
        std::printf("%s{\"in\": \"%s\", \"k\": \"%s\", \"s\": \"%s\", \"direct_s\": %.5f, \"fft_s\": %.5f, "
                    "\"chosen\": \"%s\"}",
                    i ? ", " : "", rep[i].image_dims.str().c_str(), rep[i].kernel_dims.str().c_str(),
                    rep[i].sparsity.str().c_str(), rep[i].direct_seconds, rep[i].fft_seconds,
                    rep[i].chosen == conv_engine::fft ? "fft" : "direct");
    std::printf("]}\n");
    return 0;
}

// Per-edge cost estimate of one reference round: for every distinct edge
// signature, time the exact per-edge task bodies the engine runs
// (do_forward, run_backward, run_update_body: engine.hpp:582-829) on one
// thread (median of 3), multiply by the number of such edges and divide by
// the worker count, i.e. assume the paper's linear speedup.
// This favours the CPU (no scheduling or memory-bandwidth losses).
int estimate(int argc, char** argv) {
    const std::string spec = read_file(argv[2]);
    const vec3i od = v3(argv[3]);
    const int threads = std::atoi(argv[4]);
    auto g = parse_netspec<float>(spec, od);
    init_weights(g, 1);
    std::mt19937 rng(3);
    using clk = std::chrono::steady_clock;
    std::map<std::string, std::pair<double, std::int64_t>> sig;  // signature -> (seconds, count)
    for (const auto& e : g.edges) {
        const vec3i in = g.nodes[size_t(e.from)].dims;
        std::string key = std::to_string(int(e.kind())) + ":" + in.str();
        if (auto* c = std::get_if<conv_op<float>>(&e.op)) key += ":" + c->k.dims().str() + ":" + c->k.sparsity.str();
        if (auto* p = std::get_if<pool_op>(&e.op)) key += ":" + p->spec.p.str();
        if (auto* f = std::get_if<filter_op>(&e.op)) key += ":" + f->spec.k.str() + ":" + f->spec.s.str();
        auto it = sig.find(key);
        if (it != sig.end()) {
            it->second.second++;
            continue;
        }
        volume<float> x(in);
        fill_uniform(x, rng, 0.f, 1.f);
        const vec3i outd = g.nodes[size_t(e.to)].dims;
        volume<float> gout(outd);
        fill_uniform(gout, rng, -1.f, 1.f);
        auto body = [&]() {
            if (auto* c = std::get_if<conv_op<float>>(&e.op)) {
                auto y = conv_valid_direct(x, c->k);
                auto gx = conv_full_direct(gout, reflect(c->k.weights), c->k.sparsity);
                auto gw = kernel_gradient_direct(x, gout, c->k.weights.dims(), c->k.sparsity);
            } else if (auto* t = std::get_if<transfer_op<float>>(&e.op)) {
                auto y = transfer_forward(x, t->fn);
                auto gx = transfer_backward(gout, x, t->fn);
                volatile float gb = transfer_bias_gradient(x, gout, t->fn);
                (void)gb;
            } else if (auto* p = std::get_if<pool_op>(&e.op)) {
                auto [y, rec] = maxpool_forward(x, p->spec);
                auto gx = maxpool_backward(gout, rec, p->spec);
            } else {
                const auto& f = std::get<filter_op>(e.op);
                auto [y, rec] = maxfilter_forward(x, f.spec);
                auto gx = maxfilter_backward(gout, rec, f.spec, in);
            }
        };
        body();  // warm pools
        std::vector<double> ts;
        for (int t = 0; t < 3; ++t) {
            const auto t0 = clk::now();
            body();
            ts.push_back(std::chrono::duration<double>(clk::now() - t0).count());
        }
        std::sort(ts.begin(), ts.end());
        sig[key] = {ts[1], 1};
    }
    double serial = 0;
    for (const auto& [k, v] : sig) serial += v.first * double(v.second);
    std::printf("{\"serial_seconds\": %.6f, \"round_seconds\": %.6f, \"threads\": %d, \"signatures\": %zu}\n", serial,
                serial / threads, threads, sig.size());
    return 0;
}

int round_(int argc, char** argv) {
    const std::string spec = read_file(argv[2]);
    auto g = parse_netspec<double>(spec, v3(argv[3]));
    set_params(g, read_bin<double>(argv[4]));
    const auto in = read_bin<double>(argv[5]);
    const auto lab = read_bin<double>(argv[6]);
    const double eta = std::atof(argv[7]);
    volume<double> input(g.nodes[0].dims);
    for (std::int64_t i = 0; i < input.size(); ++i) input[i] = in.at(size_t(i));
    std::vector<volume<double>> desired;
    size_t off = 0;
    for (const auto& n : g.nodes)
        if (n.role == node_role::output) {
            volume<double> d(n.dims);
            for (std::int64_t i = 0; i < d.size(); ++i) d[i] = lab.at(off++);
            desired.push_back(std::move(d));
        }
    const double loss = oracle::net_train_round(g, input, desired, eta);
    std::vector<double> out{loss};
    for (double p : get_params(g)) out.push_back(p);
    write_bin(argv[8], out);
    return 0;
}

int maxfilter(int argc, char** argv) {
    const auto in = read_bin<double>(argv[2]);
    const vec3i n = v3(argv[3]);
    volume<double> x(n);
    for (std::int64_t i = 0; i < x.size(); ++i) x[i] = in.at(size_t(i));
    auto [out, rec] = maxfilter_forward(x, filter_spec{v3(argv[4]), v3(argv[5])});
    std::vector<double> o(size_t(out.size()));
    std::vector<std::int32_t> r(size_t(out.size()));
    for (std::int64_t i = 0; i < out.size(); ++i) o[size_t(i)] = out[i], r[size_t(i)] = rec[i];
    write_bin(argv[6], o);
    write_bin(argv[7], r);
    return 0;
}

int conv(int argc, char** argv) {
    const auto xin = read_bin<double>(argv[2]);
    const auto win = read_bin<double>(argv[4]);
    volume<double> x(v3(argv[3])), w(v3(argv[5]));
    for (std::int64_t i = 0; i < x.size(); ++i) x[i] = xin.at(size_t(i));
    for (std::int64_t i = 0; i < w.size(); ++i) w[i] = win.at(size_t(i));
    auto y = conv_valid_direct(x, w, v3(argv[6]));
    std::vector<double> o(y.data(), y.data() + y.size());
    write_bin(argv[7], o);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const std::string cmd = argc > 1 ? argv[1] : "";
        if (cmd == "bench" && (argc == 8 || argc == 9)) return bench(argc, argv);
        if (cmd == "tune" && argc == 5) return tune(argc, argv);
        if (cmd == "round" && argc == 9) return round_(argc, argv);
        if (cmd == "estimate" && argc == 5) return estimate(argc, argv);
        if (cmd == "maxfilter" && argc == 8) return maxfilter(argc, argv);
        if (cmd == "conv" && argc == 8) return conv(argc, argv);
        std::fprintf(stderr, "usage: see znn_ref.cpp header\n");
        return 1;
    } catch (const structural_error& e) {
        std::fprintf(stderr, "structural error: %s\n", e.what());
        return 1;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "runtime error: %s\n", e.what());
        return 2;
    }
}
