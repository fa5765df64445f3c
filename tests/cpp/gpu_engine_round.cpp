// TEST INFRASTRUCTURE: the reference-side drop-in (include/znn_gpu_engine.hpp)
// compiled against the reference's own headers (/root/reference/proj/include,
// Eigen-subset shim) and linked with libznn_cuda.so. Built by
// tests/cpp/build.sh into oracle/_ref/ (git-ignored; travels to the GPU box).
//
//   gpu_engine_round <netspec> <x,y,z out dims> <seed>
//
// 1. one round of znn::gpu_engine vs the reference's straight-line oracle
//    round in double (tests/oracles.hpp:155-252, net_train_round) on the same
//    weights, input and desired volumes: loss within 1e-4, every updated
//    parameter (scattered back into net_graph<float>) within 1e-3
//    (max_rel_error, volume.hpp:170-176);
// 2. three more rounds vs the reference engine<float> (engine.hpp:65-254,
//    direct mode, 1 thread) from the same state: per-round losses within 1e-3.
// Prints one JSON line; exit 0 = pass.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <random>
#include <sstream>

#include "oracles.hpp"
#include "znn/engine.hpp"
#include "znn/netspec.hpp"
#include "znn/trainer.hpp"
#include "znn_gpu_engine.hpp"

using namespace znn;

static std::string read_file(const char* p) {
    std::ifstream is(p);
    std::stringstream ss;
    ss << is.rdbuf();
    return ss.str();
}

template <typename A, typename B>
static void copy_params(const net_graph<A>& src, net_graph<B>& dst) {
    for (size_t e = 0; e < src.edges.size(); ++e) {
        if (auto* c = std::get_if<conv_op<A>>(&src.edges[e].op)) {
            auto& d = std::get<conv_op<B>>(dst.edges[e].op);
            for (std::int64_t i = 0; i < c->k.weights.size(); ++i) d.k.weights[i] = B(c->k.weights[i]);
        } else if (auto* t = std::get_if<transfer_op<A>>(&src.edges[e].op)) {
            std::get<transfer_op<B>>(dst.edges[e].op).fn.bias = B(t->fn.bias);
        }
    }
}

template <typename T>
static std::vector<double> params_of(const net_graph<T>& g) {
    std::vector<double> p;
    for (const auto& e : g.edges) {
        if (auto* c = std::get_if<conv_op<T>>(&e.op))
            for (std::int64_t i = 0; i < c->k.weights.size(); ++i) p.push_back(double(c->k.weights[i]));
        else if (auto* t = std::get_if<transfer_op<T>>(&e.op))
            p.push_back(double(t->fn.bias));
    }
    return p;
}

int main(int argc, char** argv) {
    if (argc != 4) {
        std::fprintf(stderr, "usage: gpu_engine_round <netspec> <x,y,z> <seed>\n");
        return 2;
    }
    try {
        const std::string spec = read_file(argv[1]);
        vec3i od;
        char c1, c2;
        std::istringstream(argv[2]) >> od.x >> c1 >> od.y >> c2 >> od.z;
        const unsigned seed = unsigned(std::atoi(argv[3]));
        auto g = parse_netspec<float>(spec, od);
        init_weights(g, seed);
        auto gd = parse_netspec<double>(spec, od);
        copy_params(g, gd);
        auto ge = parse_netspec<float>(spec, od);  // for engine<float>
        copy_params(g, ge);

        // one sample: inputs uniform[0,1), desired uniform[0,1) (half-L2)
        std::mt19937 rng(seed);
        typename engine<float>::sample smp;
        volume<double> in_d({1, 1, 1});
        std::vector<volume<double>> des_d;
        for (const auto& n : g.nodes)
            if (n.role == node_role::input) {
                auto v = make_volume<float>(n.dims);
                fill_uniform(*v, rng, 0.f, 1.f);
                in_d = volume<double>(n.dims);
                for (std::int64_t i = 0; i < v->size(); ++i) in_d[i] = double((*v)[i]);
                smp.inputs.push_back(std::move(v));
            }
        for (const auto& n : g.nodes)
            if (n.role == node_role::output) {
                auto v = make_volume<float>(n.dims);
                fill_uniform(*v, rng, 0.f, 1.f);
                volume<double> d(n.dims);
                for (std::int64_t i = 0; i < v->size(); ++i) d[i] = double((*v)[i]);
                des_d.push_back(std::move(d));
                smp.desired.push_back(std::move(v));
            }
        typename engine<float>::sample_source src = [&](std::int64_t) -> const typename engine<float>::sample& {
            return smp;
        };
        const float eta = 0.01f;

        // 1. gpu_engine round vs the double oracle round
        gpu_engine_config gc;
        gc.learning_rate = eta;
        gc.conv = ZNN_CONV_DIRECT;
        gpu_engine eng(g, spec, gc);
        const auto s1 = eng.run(1, src);
        const double ref_loss = oracle::net_train_round(gd, in_d, des_d, double(eta));
        const auto pg = params_of(g), pr = params_of(gd);
        double perr = 0, pmax = 0;
        for (size_t i = 0; i < pg.size(); ++i) perr = std::max(perr, std::fabs(pg[i] - pr[i])), pmax = std::max(pmax, std::fabs(pr[i]));
        perr /= (pmax + 1.0);
        const double lerr = std::fabs(s1[0].loss - ref_loss) / (std::fabs(ref_loss) + 1.0);

        // 2. three more rounds vs engine<float> from the same (updated) state
        copy_params(gd, ge);
        typename engine<float>::config ec;
        ec.threads = 1;
        ec.learning_rate = eta;
        engine<float> ref(ge, compute_priorities(ge), ec);
        const auto s2 = eng.run(3, src);
        const auto s3 = ref.run(3, src);
        double traj = 0;
        for (size_t r = 0; r < 3; ++r)
            traj = std::max(traj, std::fabs(s2[r].loss - s3[r].loss) / (std::fabs(s3[r].loss) + 1e-30));
        const bool ok = lerr < 1e-4 && perr < 1e-3 && traj < 1e-3;
        std::printf("{\"ok\": %s, \"loss\": %.9g, \"oracle_loss\": %.9g, \"loss_err\": %.3e, \"param_err\": %.3e, "
                    "\"params\": %zu, \"engine_traj_rel_err\": %.3e, \"gpu_losses\": [%.9g, %.9g, %.9g], "
                    "\"engine_float_losses\": [%.9g, %.9g, %.9g]}\n",
                    ok ? "true" : "false", s1[0].loss, ref_loss, lerr, perr, pg.size(), traj, s2[0].loss,
                    s2[1].loss, s2[2].loss, s3[0].loss, s3[1].loss, s3[2].loss);
        return ok ? 0 : 1;
    } catch (const structural_error& e) {
        std::fprintf(stderr, "structural error: %s\n", e.what());
        return 3;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "runtime error: %s\n", e.what());
        return 4;
    }
}
