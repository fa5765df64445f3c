#include "netgraph.hpp"

#include <algorithm>
#include <cctype>
#include <map>
#include <sstream>

#include "common.cuh"

namespace znn_host {

using znn_gpu::require;

std::string v3::str() const {
    return std::to_string(x) + "," + std::to_string(y) + "," + std::to_string(z);
}

int graph::find(const std::string& name) const {
    auto it = index.find(name);
    return it == index.end() ? -1 : it->second;
}

int graph::add_node(const std::string& name, role r) {
    require(find(name) < 0, "duplicate node '" + name + "'");
    gnode n;
    n.name = name;
    n.r = r;
    index[name] = int(nodes.size());
    nodes.push_back(std::move(n));
    return int(nodes.size()) - 1;
}

int graph::add_edge(gedge e) {
    require(e.from >= 0 && e.from < int(nodes.size()) && e.to >= 0 && e.to < int(nodes.size()),
            "edge " + e.name + ": unknown endpoint");
    const int id = int(edges.size());
    nodes[size_t(e.from)].outs.push_back(id);
    nodes[size_t(e.to)].ins.push_back(id);
    edges.push_back(std::move(e));
    return id;
}

std::vector<int> graph::topo() const {
    std::vector<int> indeg(nodes.size(), 0), order;
    for (const auto& e : edges) indeg[size_t(e.to)]++;
    for (size_t i = 0; i < nodes.size(); ++i)
        if (!indeg[i]) order.push_back(int(i));
    for (size_t h = 0; h < order.size(); ++h)
        for (int eid : nodes[size_t(order[h])].outs)
            if (--indeg[size_t(edges[size_t(eid)].to)] == 0)
                order.push_back(edges[size_t(eid)].to);
    if (order.size() != nodes.size())
        for (size_t i = 0; i < nodes.size(); ++i)
            if (indeg[i] > 0) throw znn_gpu::shape_error("graph has a cycle through node " +
                                                         nodes[i].name);
    return order;
}

void graph::validate() const {
    require(!nodes.empty() && !edges.empty(), "graph must have nodes and edges");
    (void)topo();
    for (const auto& v : nodes) {
        if (v.ins.size() >= 2)
            for (int eid : v.ins)
                require(edges[size_t(eid)].kind == op::conv,
                        "node " + v.name + ": convergent edges must all be convolutions (edge " +
                            edges[size_t(eid)].name + " is not)");
        if (v.r == role::input) require(v.ins.empty(), "input node " + v.name + " has incoming edges");
        if (v.r == role::output) require(v.outs.empty(), "output node " + v.name + " has outgoing edges");
        if (v.ins.empty()) require(v.r == role::input, "node " + v.name + " has no incoming edges but is not an input");
        if (v.outs.empty()) require(v.r == role::output, "node " + v.name + " has no outgoing edges but is not an output");
    }
}

namespace {

std::string strip(const std::string& s) {
    const auto a = s.find_first_not_of(" \t\r\n");
    if (a == std::string::npos) return "";
    const auto b = s.find_last_not_of(" \t\r\n");
    return s.substr(a, b - a + 1);
}

v3 parse_v3(const std::string& s, const std::string& what) {
    v3 v;
    char c1 = 0, c2 = 0;
    std::istringstream is(s);
    is >> v.x >> c1 >> v.y >> c2 >> v.z;
    require(!is.fail() && c1 == ',' && c2 == ',',
            what + ": expected three comma-separated integers, got '" + s + "'");
    return v;
}

int parse_fn(const std::string& s) {
    if (s == "logistic" || s == "sigmoid") return 0;
    if (s == "tanh") return 1;
    if (s == "relu" || s == "rectified_linear") return 2;
    throw znn_gpu::shape_error("unknown transfer function '" + s + "'");
}

struct section {
    std::string kind, name;
    std::map<std::string, std::string> kv;
    std::string get(const std::string& k, const std::string& dflt = "") const {
        auto it = kv.find(k);
        return it == kv.end() ? dflt : it->second;
    }
    bool has(const std::string& k) const { return kv.count(k) != 0; }
};

std::vector<section> split_sections(const std::string& text) {
    std::vector<section> out;
    std::istringstream is(text);
    std::string line;
    while (std::getline(is, line)) {
        if (auto h = line.find('#'); h != std::string::npos) line.resize(h);
        line = strip(line);
        if (line.empty()) continue;
        if (line.front() == '[') {
            const auto close = line.find(']');
            require(close != std::string::npos, "netspec: unterminated section '" + line + "'");
            std::istringstream hs(strip(line.substr(1, close - 1)));
            section sec;
            hs >> sec.kind >> sec.name;
            require(sec.kind == "node" || sec.kind == "edge" || sec.kind == "layered",
                    "netspec: unknown section kind '" + sec.kind + "'");
            require(sec.kind == "layered" || !sec.name.empty(),
                    "netspec: [" + sec.kind + "] needs a name");
            out.push_back(std::move(sec));
            line = strip(line.substr(close + 1));
            if (line.empty()) continue;
        }
        require(!out.empty(), "netspec: key outside any section: '" + line + "'");
        std::istringstream ls(line);
        std::string tok;
        while (ls >> tok) {
            const auto eq = tok.find('=');
            require(eq != std::string::npos && eq > 0, "netspec: expected key=value, got '" + tok + "'");
            out.back().kv[tok.substr(0, eq)] = tok.substr(eq + 1);
        }
    }
    return out;
}

// [layered] shorthand (netspec.hpp:103-151): C conv, T transfer, M filter, P pool.
v3 expand_layered(graph& g, const section& sec) {
    const std::string seq = sec.get("seq");
    require(!seq.empty(), "[layered]: missing seq=");
    const int width = std::stoi(sec.get("width", "1"));
    require(width >= 1, "[layered]: width must be >= 1");
    const v3 kd = parse_v3(sec.get("kernel", "3,3,3"), "[layered] kernel");
    const v3 pd = parse_v3(sec.get("pool", "2,2,2"), "[layered] pool");
    const int fn = parse_fn(sec.get("fn", "relu"));
    require(sec.has("output"), "[layered]: missing output=");
    const v3 od = parse_v3(sec.get("output"), "[layered] output");
    std::vector<int> prev{g.add_node("in", role::input)};
    for (size_t li = 0; li < seq.size(); ++li) {
        const char c = seq[li];
        const role r = li + 1 == seq.size() ? role::output : role::internal;
        const std::string ln = "L" + std::to_string(li + 1);
        std::vector<int> cur;
        if (c == 'C') {
            for (int j = 0; j < width; ++j) cur.push_back(g.add_node(ln + "_" + std::to_string(j), r));
            for (int u : prev)
                for (size_t j = 0; j < cur.size(); ++j) {
                    gedge e;
                    e.name = "c" + std::to_string(li + 1) + "_" + g.nodes[size_t(u)].name + "_" + std::to_string(j);
                    e.from = u, e.to = cur[j], e.kind = op::conv, e.k = kd;
                    g.add_edge(e);
                }
        } else {
            for (size_t j = 0; j < prev.size(); ++j) {
                cur.push_back(g.add_node(ln + "_" + std::to_string(j), r));
                gedge e;
                e.name = std::string(1, char(std::tolower(c))) + std::to_string(li + 1) + "_" + std::to_string(j);
                e.from = prev[j], e.to = cur.back();
                if (c == 'T') e.kind = op::transfer, e.fn = fn;
                else if (c == 'M') e.kind = op::filter, e.k = pd;
                else if (c == 'P') e.kind = op::pool, e.k = pd;
                else throw znn_gpu::shape_error("[layered]: unknown layer letter '" + std::string(1, c) + "'");
                g.add_edge(e);
            }
        }
        prev = std::move(cur);
    }
    return od;
}

v3 tail_of(const gedge& e, v3 head) {
    switch (e.kind) {
        case op::conv:
        case op::filter: {
            const v3 w = window(e.k, e.s);
            return {head.x + w.x - 1, head.y + w.y - 1, head.z + w.z - 1};
        }
        case op::pool: return {head.x * e.k.x, head.y * e.k.y, head.z * e.k.z};
        default: return head;
    }
}

v3 head_of(const gedge& e, v3 tail) {
    switch (e.kind) {
        case op::conv:
        case op::filter: {
            const v3 w = window(e.k, e.s);
            require(w.x <= tail.x && w.y <= tail.y && w.z <= tail.z,
                    "edge " + e.name + ": effective window " + w.str() + " exceeds image " + tail.str());
            return {tail.x - w.x + 1, tail.y - w.y + 1, tail.z - w.z + 1};
        }
        case op::pool:
            require(tail.x % e.k.x == 0 && tail.y % e.k.y == 0 && tail.z % e.k.z == 0,
                    "edge " + e.name + ": image " + tail.str() + " not divisible by pool window " + e.k.str());
            return {tail.x / e.k.x, tail.y / e.k.y, tail.z / e.k.z};
        default: return tail;
    }
}

}  // namespace

graph parse_netspec(const std::string& text, v3 out_override) {
    graph g;
    v3 out_dims = out_override;
    for (const section& sec : split_sections(text)) {
        if (sec.kind == "layered") {
            const v3 od = expand_layered(g, sec);
            if (!out_dims.positive()) out_dims = od;
        } else if (sec.kind == "node") {
            const std::string r = sec.get("role", "internal");
            role rr = role::internal;
            if (r == "input") rr = role::input;
            else if (r == "output") rr = role::output;
            else require(r == "internal", "node " + sec.name + ": unknown role '" + r + "'");
            g.add_node(sec.name, rr);
            if (sec.has("dims") && rr == role::output && !out_dims.positive())
                out_dims = parse_v3(sec.get("dims"), "node " + sec.name + " dims");
        } else {
            gedge e;
            e.name = sec.name;
            e.from = g.find(sec.get("from"));
            e.to = g.find(sec.get("to"));
            require(e.from >= 0, "edge " + sec.name + ": unknown node '" + sec.get("from") + "'");
            require(e.to >= 0, "edge " + sec.name + ": unknown node '" + sec.get("to") + "'");
            const std::string type = sec.get("type");
            if (type == "conv") {
                e.kind = op::conv;
                e.k = parse_v3(sec.get("kernel", "1,1,1"), "edge " + sec.name);
                if (sec.has("sparsity")) e.s = parse_v3(sec.get("sparsity"), "edge " + sec.name);
                require(e.k.positive() && e.s.positive(), "edge " + sec.name + ": kernel and sparsity must be positive");
            } else if (type == "transfer") {
                e.kind = op::transfer;
                e.fn = parse_fn(sec.get("fn", "relu"));
            } else if (type == "pool") {
                e.kind = op::pool;
                e.k = parse_v3(sec.get("p", "2,2,2"), "edge " + sec.name);
            } else if (type == "filter") {
                e.kind = op::filter;
                e.k = parse_v3(sec.get("k", "2,2,2"), "edge " + sec.name);
                if (sec.has("sparsity")) e.s = parse_v3(sec.get("sparsity"), "edge " + sec.name);
            } else {
                throw znn_gpu::shape_error("edge " + sec.name + ": unknown type '" + type +
                                           "' (want conv|transfer|pool|filter)");
            }
            g.add_edge(e);
        }
    }
    g.validate();
    require(out_dims.positive(), "netspec: no output dims given ([layered] output=, node dims=, or override)");
    infer_shapes(g, out_dims);
    return g;
}

void infer_shapes(graph& g, v3 out_dims) {
    const auto order = g.topo();
    std::vector<v3> dims(g.nodes.size());
    for (size_t i = 0; i < g.nodes.size(); ++i)
        if (g.nodes[i].r == role::output) dims[i] = out_dims;
    for (auto it = order.rbegin(); it != order.rend(); ++it) {
        const int v = *it;
        require(dims[size_t(v)].positive(), "shape inference: node " + g.nodes[size_t(v)].name + " unreachable from outputs");
        for (int eid : g.nodes[size_t(v)].ins) {
            const gedge& e = g.edges[size_t(eid)];
            const v3 t = tail_of(e, dims[size_t(v)]);
            if (dims[size_t(e.from)].positive())
                require(dims[size_t(e.from)] == t, "shape inference: node " + g.nodes[size_t(e.from)].name +
                                                       " implied " + t.str() + " via edge " + e.name +
                                                       " but already " + dims[size_t(e.from)].str());
            else
                dims[size_t(e.from)] = t;
        }
    }
    for (int v : order)
        for (int eid : g.nodes[size_t(v)].outs) {
            const gedge& e = g.edges[size_t(eid)];
            const v3 h = head_of(e, dims[size_t(v)]);
            require(h == dims[size_t(e.to)], "shape inference: edge " + e.name + " maps " + dims[size_t(v)].str() +
                                                 " to " + h.str() + " but node " + g.nodes[size_t(e.to)].name +
                                                 " has " + dims[size_t(e.to)].str());
        }
    for (size_t i = 0; i < g.nodes.size(); ++i) g.nodes[i].dims = dims[i];
}

graph sliding_equivalent(const graph& src) {
    graph g = src;
    std::vector<v3> mult(g.nodes.size());
    for (size_t i = 0; i < g.nodes.size(); ++i)
        if (g.nodes[i].r == role::input) mult[i] = {1, 1, 1};
    for (int v : g.topo()) {
        require(mult[size_t(v)].positive(), "to_sliding_equivalent: node " + g.nodes[size_t(v)].name + " unreachable");
        for (int eid : g.nodes[size_t(v)].outs) {
            gedge& e = g.edges[size_t(eid)];
            const v3 m = mult[size_t(v)];
            v3 hm = m;
            if (e.kind == op::conv || e.kind == op::filter) {
                e.s = {e.s.x * m.x, e.s.y * m.y, e.s.z * m.z};
            } else if (e.kind == op::pool) {
                const v3 win = e.k;
                e.kind = op::filter;
                e.s = m;
                hm = {m.x * win.x, m.y * win.y, m.z * win.z};
            }
            if (mult[size_t(e.to)].positive())
                require(mult[size_t(e.to)] == hm, "to_sliding_equivalent: inconsistent pooling factors at node " +
                                                      g.nodes[size_t(e.to)].name);
            else
                mult[size_t(e.to)] = hm;
        }
    }
    return g;
}

}  // namespace znn_host
