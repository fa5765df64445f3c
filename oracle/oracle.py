"""CPU oracle for the ZNN training hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module; the product package
(paper_1510_06706_b200) never does.

Layers:
  * ctypes bindings to liboracle.so (plain-C double restatement of the
    per-map operators, oracle/znn_oracle.c);
  * an independent netspec parser + shape inference restating
    netspec.hpp:158-223 and netgraph.hpp:161-254, 321-372;
  * ``train_step``: one straight-line SGD step restating
    tests/oracles.hpp:155-252 (forward in topological order with convergent
    sums in edge-id order, loss gradient, reverse-topological backward,
    parameter updates), extended for the BASELINE configs with a batch of
    patches (mean gradient), momentum (v = mu*v + g; w -= lr*v) and binomial
    cross-entropy on a logistic output (pre-activation gradient a - d).
"""
from __future__ import annotations

import ctypes
import os
import re
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

LOGISTIC, TANH, RELU = 0, 1, 2
_FN = {"logistic": LOGISTIC, "sigmoid": LOGISTIC, "tanh": TANH, "relu": RELU,
       "rectified_linear": RELU}


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            import subprocess
            subprocess.check_call(["make", "-s", "-C", _HERE])
        _LIB = ctypes.CDLL(path)
        d = ctypes.POINTER(ctypes.c_double)
        i64 = ctypes.POINTER(ctypes.c_int64)
        i32 = ctypes.POINTER(ctypes.c_int32)
        L = _LIB
        L.zo_conv_valid.argtypes = [d, i64, d, i64, i64, d]
        L.zo_conv_valid_at.argtypes = [d, i64, d, i64, i64, i64, ctypes.c_int64, d]
        L.zo_conv_full.argtypes = [d, i64, d, i64, i64, d]
        L.zo_conv_full_at.argtypes = [d, i64, d, i64, i64, i64, ctypes.c_int64, d]
        L.zo_kernel_grad.argtypes = [d, i64, d, i64, i64, i64, d]
        L.zo_reflect.argtypes = [d, i64, d]
        L.zo_dilate.argtypes = [d, i64, i64, d]
        L.zo_sliding_max_1d.argtypes = [d, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_int64, d, ctypes.c_int64, i32]
        L.zo_maxpool_fwd.argtypes = [d, i64, i64, d, i32]
        L.zo_maxpool_bwd.argtypes = [d, i32, i64, i64, d]
        L.zo_maxfilter_fwd.argtypes = [d, i64, i64, i64, d, i32]
        L.zo_maxfilter_bwd.argtypes = [d, i32, i64, i64, d]
        L.zo_transfer_value.argtypes = [ctypes.c_int, ctypes.c_double]
        L.zo_transfer_value.restype = ctypes.c_double
        L.zo_transfer_derivative.argtypes = [ctypes.c_int, ctypes.c_double]
        L.zo_transfer_derivative.restype = ctypes.c_double
        L.zo_transfer_fwd.argtypes = [d, ctypes.c_int64, ctypes.c_int, ctypes.c_double, d]
        L.zo_transfer_bwd.argtypes = [d, d, ctypes.c_int64, ctypes.c_int, ctypes.c_double, d]
        L.zo_transfer_bias_grad.argtypes = [d, d, ctypes.c_int64, ctypes.c_int, ctypes.c_double]
        L.zo_transfer_bias_grad.restype = ctypes.c_double
        L.zo_loss_l2.argtypes = [d, d, ctypes.c_int64, d]
        L.zo_loss_l2.restype = ctypes.c_double
        L.zo_loss_ce.argtypes = [d, d, ctypes.c_int64, d]
        L.zo_loss_ce.restype = ctypes.c_double
        L.zo_max_rel_error.argtypes = [d, d, ctypes.c_int64]
        L.zo_max_rel_error.restype = ctypes.c_double
    return _LIB


def _d(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _i32(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def _v3(t):
    a = np.ascontiguousarray(np.asarray(t, dtype=np.int64).reshape(3))
    return a


def _i64(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def _f64(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def eff(k, s):
    """types.hpp:51-53 effective window s*(k-1)+1."""
    return tuple(int(si) * (int(ki) - 1) + 1 for ki, si in zip(k, s))


# --------------------------------------------------------------------------
# per-map operators (thin numpy wrappers over liboracle.so)
# --------------------------------------------------------------------------

def conv_valid(x, k, s=(1, 1, 1)):
    x, k = _f64(x), _f64(k)
    n, kd, sv = _v3(x.shape), _v3(k.shape), _v3(s)
    m = tuple(int(n[a] - sv[a] * (kd[a] - 1)) for a in range(3))
    out = np.empty(m, dtype=np.float64)
    lib().zo_conv_valid(_d(x), _i64(n), _d(k), _i64(kd), _i64(sv), _d(out))
    return out


def conv_valid_at(x, k, s, flat_idx):
    x, k = _f64(x), _f64(k)
    idx = np.ascontiguousarray(np.asarray(flat_idx, dtype=np.int64))
    n, kd, sv = _v3(x.shape), _v3(k.shape), _v3(s)
    out = np.empty(idx.size, dtype=np.float64)
    lib().zo_conv_valid_at(_d(x), _i64(n), _d(k), _i64(kd), _i64(sv), _i64(idx), idx.size,
                           _d(out))
    return out


def conv_full(g, k, s=(1, 1, 1)):
    g, k = _f64(g), _f64(k)
    m, kd, sv = _v3(g.shape), _v3(k.shape), _v3(s)
    od = tuple(int(m[a] + sv[a] * (kd[a] - 1)) for a in range(3))
    out = np.empty(od, dtype=np.float64)
    lib().zo_conv_full(_d(g), _i64(m), _d(k), _i64(kd), _i64(sv), _d(out))
    return out


def conv_full_at(g, k, s, flat_idx):
    g, k = _f64(g), _f64(k)
    idx = np.ascontiguousarray(np.asarray(flat_idx, dtype=np.int64))
    m, kd, sv = _v3(g.shape), _v3(k.shape), _v3(s)
    out = np.empty(idx.size, dtype=np.float64)
    lib().zo_conv_full_at(_d(g), _i64(m), _d(k), _i64(kd), _i64(sv), _i64(idx), idx.size, _d(out))
    return out


def kernel_grad(x, g, kd, s=(1, 1, 1)):
    x, g = _f64(x), _f64(g)
    n, m, kv, sv = _v3(x.shape), _v3(g.shape), _v3(kd), _v3(s)
    out = np.empty(tuple(int(v) for v in kv), dtype=np.float64)
    lib().zo_kernel_grad(_d(x), _i64(n), _d(g), _i64(m), _i64(kv), _i64(sv), _d(out))
    return out


def reflect(x):
    x = _f64(x)
    out = np.empty_like(x)
    lib().zo_reflect(_d(x), _i64(_v3(x.shape)), _d(out))
    return out


def dilate(k, s):
    k = _f64(k)
    e = eff(k.shape, s)
    out = np.empty(e, dtype=np.float64)
    lib().zo_dilate(_d(k), _i64(_v3(k.shape)), _i64(_v3(s)), _d(out))
    return out


def sliding_max_1d(v, k, s):
    v = _f64(v).reshape(-1)
    n = v.size
    m = n - s * (k - 1)
    out = np.empty(m, dtype=np.float64)
    arg = np.empty(m, dtype=np.int32)
    lib().zo_sliding_max_1d(_d(v), n, 1, k, s, _d(out), 1, _i32(arg))
    return out, arg


def maxpool_fwd(x, p):
    x = _f64(x)
    m = tuple(x.shape[a] // p[a] for a in range(3))
    out = np.empty(m, dtype=np.float64)
    rec = np.empty(m, dtype=np.int32)
    lib().zo_maxpool_fwd(_d(x), _i64(_v3(x.shape)), _i64(_v3(p)), _d(out), _i32(rec))
    return out, rec


def maxpool_bwd(g, rec, p):
    g = _f64(g)
    rec = np.ascontiguousarray(rec, dtype=np.int32)
    out = np.empty(tuple(g.shape[a] * p[a] for a in range(3)), dtype=np.float64)
    lib().zo_maxpool_bwd(_d(g), _i32(rec), _i64(_v3(g.shape)), _i64(_v3(p)), _d(out))
    return out


def maxfilter_fwd(x, k, s):
    x = _f64(x)
    e = eff(k, s)
    m = tuple(x.shape[a] - e[a] + 1 for a in range(3))
    out = np.empty(m, dtype=np.float64)
    rec = np.empty(m, dtype=np.int32)
    lib().zo_maxfilter_fwd(_d(x), _i64(_v3(x.shape)), _i64(_v3(k)), _i64(_v3(s)), _d(out),
                           _i32(rec))
    return out, rec


def maxfilter_bwd(g, rec, in_dims):
    g = _f64(g)
    rec = np.ascontiguousarray(rec, dtype=np.int32)
    out = np.empty(tuple(int(v) for v in in_dims), dtype=np.float64)
    lib().zo_maxfilter_bwd(_d(g), _i32(rec), _i64(_v3(g.shape)), _i64(_v3(in_dims)), _d(out))
    return out


def transfer_value(kind, x):
    return lib().zo_transfer_value(kind, float(x))


def transfer_derivative(kind, x):
    return lib().zo_transfer_derivative(kind, float(x))


def transfer_fwd(x, kind, bias):
    x = _f64(x)
    out = np.empty_like(x)
    lib().zo_transfer_fwd(_d(x), x.size, kind, float(bias), _d(out))
    return out


def transfer_bwd(g, x, kind, bias):
    g, x = _f64(g), _f64(x)
    out = np.empty_like(x)
    lib().zo_transfer_bwd(_d(g), _d(x), x.size, kind, float(bias), _d(out))
    return out


def transfer_bias_grad(x, g, kind, bias):
    g, x = _f64(g), _f64(x)
    return lib().zo_transfer_bias_grad(_d(x), _d(g), x.size, kind, float(bias))


def loss_l2(a, d):
    a, d = _f64(a), _f64(d)
    grad = np.empty_like(a)
    loss = lib().zo_loss_l2(_d(a), _d(d), a.size, _d(grad))
    return loss, grad


def loss_ce(a, d):
    a, d = _f64(a), _f64(d)
    grad = np.empty_like(a)
    loss = lib().zo_loss_ce(_d(a), _d(d), a.size, _d(grad))
    return loss, grad


def max_rel_error(a, b):
    a, b = _f64(a).reshape(-1), _f64(b).reshape(-1)
    assert a.size == b.size
    return lib().zo_max_rel_error(_d(a), _d(b), a.size)


# --------------------------------------------------------------------------
# network description: netspec.hpp text format, restated independently
# --------------------------------------------------------------------------

@dataclass
class Node:
    name: str
    role: str = "internal"  # input | internal | output
    dims: tuple = (0, 0, 0)
    in_edges: list = field(default_factory=list)
    out_edges: list = field(default_factory=list)


@dataclass
class Edge:
    name: str
    src: int
    dst: int
    kind: str  # conv | transfer | pool | filter
    k: tuple = (1, 1, 1)  # conv kernel dims / filter window / pool window
    s: tuple = (1, 1, 1)  # sparsity (conv, filter)
    fn: int = RELU  # transfer kind


class Graph:
    def __init__(self):
        self.nodes: list[Node] = []
        self.edges: list[Edge] = []

    def node_id(self, name):
        for i, n in enumerate(self.nodes):
            if n.name == name:
                return i
        return -1

    def add_node(self, name, role="internal"):
        self.nodes.append(Node(name, role))
        return len(self.nodes) - 1

    def add_edge(self, e: Edge):
        self.edges.append(e)
        eid = len(self.edges) - 1
        self.nodes[e.src].out_edges.append(eid)
        self.nodes[e.dst].in_edges.append(eid)
        return eid

    def topo(self):
        indeg = [0] * len(self.nodes)
        for e in self.edges:
            indeg[e.dst] += 1
        order = [i for i in range(len(self.nodes)) if indeg[i] == 0]
        h = 0
        while h < len(order):
            for eid in self.nodes[order[h]].out_edges:
                t = self.edges[eid].dst
                indeg[t] -= 1
                if indeg[t] == 0:
                    order.append(t)
            h += 1
        if len(order) != len(self.nodes):
            raise ValueError("graph has a cycle")
        return order

    def inputs(self):
        return [i for i, n in enumerate(self.nodes) if n.role == "input"]

    def outputs(self):
        return [i for i, n in enumerate(self.nodes) if n.role == "output"]

    def param_layout(self):
        """Flat parameter order: edges by id; a conv edge contributes its
        k-volume (x-major), a transfer edge its bias (test_engine.cpp:57-67)."""
        out = []
        off = 0
        for eid, e in enumerate(self.edges):
            if e.kind == "conv":
                sz = int(np.prod(e.k))
                out.append((eid, off, sz))
                off += sz
            elif e.kind == "transfer":
                out.append((eid, off, 1))
                off += 1
        return out, off


def _vec3(s):
    parts = s.split(",")
    if len(parts) != 3:
        raise ValueError(f"expected three comma-separated integers, got '{s}'")
    return tuple(int(p) for p in parts)


def parse_netspec(text, output_override=None):
    """netspec.hpp:158-223 (sections [node]/[edge]/[layered])."""
    g = Graph()
    out_dims = tuple(output_override) if output_override else None
    sections = []
    for raw in text.splitlines():
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if line.startswith("["):
            close = line.index("]")
            head = line[1:close].split()
            sections.append({"kind": head[0], "name": head[1] if len(head) > 1 else "",
                             "kv": {}})
            line = line[close + 1:].strip()
            if not line:
                continue
        for tok in line.split():
            k, v = tok.split("=", 1)
            sections[-1]["kv"][k] = v
    for sec in sections:
        kv = sec["kv"]
        if sec["kind"] == "layered":
            od = _expand_layered(g, kv)
            if out_dims is None:
                out_dims = od
        elif sec["kind"] == "node":
            role = kv.get("role", "internal")
            g.add_node(sec["name"], role)
            if "dims" in kv and role == "output" and out_dims is None:
                out_dims = _vec3(kv["dims"])
        elif sec["kind"] == "edge":
            src, dst = g.node_id(kv["from"]), g.node_id(kv["to"])
            t = kv["type"]
            if t == "conv":
                e = Edge(sec["name"], src, dst, "conv", _vec3(kv.get("kernel", "1,1,1")),
                         _vec3(kv.get("sparsity", "1,1,1")))
            elif t == "transfer":
                e = Edge(sec["name"], src, dst, "transfer", fn=_FN[kv.get("fn", "relu")])
            elif t == "pool":
                e = Edge(sec["name"], src, dst, "pool", _vec3(kv.get("p", "2,2,2")))
            elif t == "filter":
                e = Edge(sec["name"], src, dst, "filter", _vec3(kv.get("k", "2,2,2")),
                         _vec3(kv.get("sparsity", "1,1,1")))
            else:
                raise ValueError(f"unknown edge type {t}")
            g.add_edge(e)
        else:
            raise ValueError(f"unknown section {sec['kind']}")
    infer_shapes(g, out_dims)
    return g


def _expand_layered(g, kv):
    """netspec.hpp:103-151."""
    seq = kv["seq"]
    width = int(kv.get("width", "1"))
    kd = _vec3(kv.get("kernel", "3,3,3"))
    pd = _vec3(kv.get("pool", "2,2,2"))
    fn = _FN[kv.get("fn", "relu")]
    od = _vec3(kv["output"])
    prev = [g.add_node("in", "input")]
    for li, c in enumerate(seq):
        role = "output" if li + 1 == len(seq) else "internal"
        lname = f"L{li + 1}"
        cur = []
        if c == "C":
            for j in range(width):
                cur.append(g.add_node(f"{lname}_{j}", role))
            for u in prev:
                for j, v in enumerate(cur):
                    g.add_edge(Edge(f"c{li + 1}_{g.nodes[u].name}_{j}", u, v, "conv", kd))
        else:
            for j, u in enumerate(prev):
                v = g.add_node(f"{lname}_{j}", role)
                cur.append(v)
                name = f"{c.lower()}{li + 1}_{j}"
                if c == "T":
                    g.add_edge(Edge(name, u, v, "transfer", fn=fn))
                elif c == "M":
                    g.add_edge(Edge(name, u, v, "filter", pd, (1, 1, 1)))
                elif c == "P":
                    g.add_edge(Edge(name, u, v, "pool", pd))
                else:
                    raise ValueError(f"unknown layer letter {c}")
        prev = cur
    return od


def _tail_dims(e, head):
    if e.kind in ("conv", "filter"):
        w = eff(e.k, e.s)
        return tuple(head[a] + w[a] - 1 for a in range(3))
    if e.kind == "pool":
        return tuple(head[a] * e.k[a] for a in range(3))
    return tuple(head)


def _head_dims(e, tail):
    if e.kind in ("conv", "filter"):
        w = eff(e.k, e.s)
        if any(w[a] > tail[a] for a in range(3)):
            raise ValueError(f"edge {e.name}: window exceeds image")
        return tuple(tail[a] - w[a] + 1 for a in range(3))
    if e.kind == "pool":
        if any(tail[a] % e.k[a] for a in range(3)):
            raise ValueError(f"edge {e.name}: not divisible by pool window")
        return tuple(tail[a] // e.k[a] for a in range(3))
    return tuple(tail)


def infer_shapes(g, out_dims):
    """netgraph.hpp:209-254: backward sweep from the outputs, forward cross-check."""
    topo = g.topo()
    dims = [None] * len(g.nodes)
    for i, n in enumerate(g.nodes):
        if n.role == "output":
            dims[i] = tuple(out_dims)
    for v in reversed(topo):
        if dims[v] is None:
            raise ValueError(f"node {g.nodes[v].name} unreachable from outputs")
        for eid in g.nodes[v].in_edges:
            e = g.edges[eid]
            t = _tail_dims(e, dims[v])
            if dims[e.src] is not None and dims[e.src] != t:
                raise ValueError(f"shape inference conflict at {g.nodes[e.src].name}")
            dims[e.src] = t
    for v in topo:
        for eid in g.nodes[v].out_edges:
            e = g.edges[eid]
            if _head_dims(e, dims[v]) != dims[e.dst]:
                raise ValueError(f"shape inference: edge {e.name} inconsistent")
    for i, n in enumerate(g.nodes):
        n.dims = dims[i]


def to_sliding_equivalent(g):
    """netgraph.hpp:321-354: pools become filters, downstream sparsity multiplies."""
    import copy
    out = copy.deepcopy(g)
    mult = [None] * len(out.nodes)
    for i, n in enumerate(out.nodes):
        if n.role == "input":
            mult[i] = (1, 1, 1)
    for v in out.topo():
        for eid in out.nodes[v].out_edges:
            e = out.edges[eid]
            hm = mult[v]
            if e.kind == "conv":
                e.s = tuple(e.s[a] * mult[v][a] for a in range(3))
            elif e.kind == "pool":
                win = e.k
                e.kind, e.s = "filter", tuple(mult[v])
                hm = tuple(mult[v][a] * win[a] for a in range(3))
            elif e.kind == "filter":
                e.s = tuple(e.s[a] * mult[v][a] for a in range(3))
            if mult[e.dst] is not None and mult[e.dst] != hm:
                raise ValueError("inconsistent pooling factors")
            mult[e.dst] = hm
    return out


# --------------------------------------------------------------------------
# one training step (oracles.hpp:155-252 extended with batch/momentum/CE)
# --------------------------------------------------------------------------

def forward(g, params, inputs):
    """Forward images per node for ONE patch. inputs: list per input node."""
    fwd = [None] * len(g.nodes)
    recs = {}
    layout, _ = g.param_layout()
    poff = {eid: (off, sz) for eid, off, sz in layout}
    for i, v in enumerate(g.inputs()):
        fwd[v] = _f64(inputs[i]).reshape(g.nodes[v].dims)
    for v in g.topo():
        if g.nodes[v].role == "input":
            continue
        acc = None
        for eid in sorted(g.nodes[v].in_edges):
            e = g.edges[eid]
            x = fwd[e.src]
            if e.kind == "conv":
                off, sz = poff[eid]
                c = conv_valid(x, params[off:off + sz].reshape(e.k), e.s)
            elif e.kind == "transfer":
                off, _ = poff[eid]
                c = transfer_fwd(x, e.fn, params[off])
            elif e.kind == "pool":
                c, r = maxpool_fwd(x, e.k)
                recs[eid] = r
            else:
                c, r = maxfilter_fwd(x, e.k, e.s)
                recs[eid] = r
            acc = c if acc is None else acc + c
        fwd[v] = acc
    return fwd, recs


def patch_gradients(g, params, inputs, labels, loss="l2"):
    """Loss and parameter gradient (flat, param_layout order) for ONE patch."""
    layout, nparam = g.param_layout()
    poff = {eid: (off, sz) for eid, off, sz in layout}
    fwd, recs = forward(g, params, inputs)
    bwd = [None] * len(g.nodes)
    total = 0.0
    pre_override = {}  # CE: transfer edge into an output gets a - d directly
    for oi, v in enumerate(g.outputs()):
        a = fwd[v]
        d = _f64(labels[oi]).reshape(a.shape)
        if loss == "l2":
            l, gr = loss_l2(a, d)
            bwd[v] = gr
        elif loss == "ce":
            ins = g.nodes[v].in_edges
            if len(ins) != 1 or g.edges[ins[0]].kind != "transfer" or \
                    g.edges[ins[0]].fn != LOGISTIC:
                raise ValueError("cross-entropy needs a logistic transfer into each output")
            l, gr = loss_ce(a, d)
            pre_override[ins[0]] = gr
            bwd[v] = np.zeros_like(a)
        else:
            raise ValueError(loss)
        total += l
    grads = np.zeros(nparam, dtype=np.float64)
    for u in reversed(g.topo()):
        if g.nodes[u].role == "output":
            continue
        acc = None
        for eid in sorted(g.nodes[u].out_edges):
            e = g.edges[eid]
            gv = bwd[e.dst]
            if e.kind == "conv":
                off, sz = poff[eid]
                k = params[off:off + sz].reshape(e.k)
                c = conv_full(gv, reflect(k), e.s)
                grads[off:off + sz] = kernel_grad(fwd[u], gv, e.k, e.s).reshape(-1)
            elif e.kind == "transfer":
                off, _ = poff[eid]
                if eid in pre_override:
                    c = pre_override[eid]
                    grads[off] = float(np.sum(c))
                else:
                    c = transfer_bwd(gv, fwd[u], e.fn, params[off])
                    grads[off] = transfer_bias_grad(fwd[u], gv, e.fn, params[off])
            elif e.kind == "pool":
                c = maxpool_bwd(gv, recs[eid], e.k)
            else:
                c = maxfilter_bwd(gv, recs[eid], g.nodes[u].dims)
            acc = c if acc is None else acc + c
        bwd[u] = acc
    return total, grads, fwd, bwd, recs


def train_step(g, params, velocity, inputs, labels, lr=0.01, momentum=0.9, loss="l2"):
    """One SGD+momentum step over a batch. inputs[b][i], labels[b][o].

    Batch convention (unspecified by the reference): the step
    gradient is the MEAN of the per-patch gradients and the reported loss is
    the mean per-patch loss; at B=1 this is exactly the reference round.
    Momentum: v <- mu*v + grad; w <- w - lr*v (v0 = 0 makes step 1 plain SGD,
    engine.hpp:795,800)."""
    B = len(inputs)
    grad = None
    total = 0.0
    for b in range(B):
        l, gr, *_ = patch_gradients(g, params, inputs[b], labels[b], loss)
        total += l
        grad = gr if grad is None else grad + gr
    grad /= B
    v = momentum * _f64(velocity) + grad
    new_params = _f64(params) - lr * v
    return total / B, grad, new_params, v
