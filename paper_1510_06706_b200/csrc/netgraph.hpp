// Host-side network description: the reference's node/edge graph and netspec
// text format, kept as the drop-in user API (the
// netspec format and the shape rules are reproduced as host API so the same
// text builds the same graph). This is a restatement of the reference's
// parser and rules, following their control flow and error messages so that
// structural errors read the same: parse_netspec / expand_layered
// (netspec.hpp:67-223), the graph and its validation (netgraph.hpp:21-156),
// shape inference (netgraph.hpp:161-254) and the sliding-window rewrite
// (netgraph.hpp:321-354). Host code, off the hot path.
#pragma once

#include <cstdint>
#include <string>
#include <unordered_map>
#include <vector>

namespace znn_host {

struct v3 {
    int64_t x = 0, y = 0, z = 0;
    int64_t vol() const { return x * y * z; }
    bool operator==(const v3&) const = default;
    bool positive() const { return x > 0 && y > 0 && z > 0; }
    std::string str() const;
};

inline v3 window(v3 k, v3 s) {  // types.hpp:51-53 effective window
    return {s.x * (k.x - 1) + 1, s.y * (k.y - 1) + 1, s.z * (k.z - 1) + 1};
}

enum class role { input, internal, output };
enum class op { conv, transfer, pool, filter };

struct gnode {
    std::string name;
    role r = role::internal;
    v3 dims;
    std::vector<int> ins, outs;
};

struct gedge {
    std::string name;
    int from = -1, to = -1;
    op kind = op::conv;
    v3 k{1, 1, 1};  // conv kernel / filter window / pool window
    v3 s{1, 1, 1};  // conv / filter sparsity
    int fn = 2;     // transfer kind (ZNN_ACT_*)
};

struct graph {
    std::vector<gnode> nodes;
    std::vector<gedge> edges;
    std::unordered_map<std::string, int> index;

    int find(const std::string& name) const;
    int add_node(const std::string& name, role r);
    int add_edge(gedge e);
    std::vector<int> topo() const;  // throws on cycles
    void validate() const;          // netgraph.hpp:134-155 rules
};

// netspec.hpp:158-223; out_override (if positive) beats dims given in the text
graph parse_netspec(const std::string& text, v3 out_override);
void infer_shapes(graph& g, v3 out_dims);
graph sliding_equivalent(const graph& g);

}  // namespace znn_host
