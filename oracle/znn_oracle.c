/*
 * znn_oracle.c — plain-loop CPU restatement of ZNN's hot-path operators.
 *
 * TEST INFRASTRUCTURE ONLY (see znn_oracle.h). Double precision, scalar
 * loops, written to be obviously correct rather than fast. Each function
 * cites the reference file:line whose semantics it restates; the restated
 * behaviour is pinned by tests/test_oracle_pins.py against the known-answer
 * cases of the reference's own test suite (test_conv.cpp, test_maxops.cpp,
 * test_transfer.cpp) and against the reference compiled in oracle/_ref.
 */
#include "znn_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define IDX(d, i, j, l) ((((i) * (d)[1]) + (j)) * (d)[2] + (l))

static void out_dims_valid(const int64_t n[3], const int64_t kd[3], const int64_t s[3],
                           int64_t m[3]) {
    for (int a = 0; a < 3; ++a) m[a] = n[a] - s[a] * (kd[a] - 1);
}

/* conv_direct.hpp:39-68 (cross-correlation, no flip) */
void zo_conv_valid(const double* x, const int64_t n[3], const double* k, const int64_t kd[3],
                   const int64_t s[3], double* out) {
    int64_t m[3];
    out_dims_valid(n, kd, s, m);
    for (int64_t i = 0; i < m[0]; ++i)
        for (int64_t j = 0; j < m[1]; ++j)
            for (int64_t l = 0; l < m[2]; ++l) {
                double acc = 0.0;
                for (int64_t a = 0; a < kd[0]; ++a)
                    for (int64_t b = 0; b < kd[1]; ++b)
                        for (int64_t c = 0; c < kd[2]; ++c)
                            acc += x[IDX(n, i + s[0] * a, j + s[1] * b, l + s[2] * c)] *
                                   k[IDX(kd, a, b, c)];
                out[IDX(m, i, j, l)] = acc;
            }
}

void zo_conv_valid_at(const double* x, const int64_t n[3], const double* k,
                      const int64_t kd[3], const int64_t s[3], const int64_t* idx,
                      int64_t count, double* out) {
    int64_t m[3];
    out_dims_valid(n, kd, s, m);
    for (int64_t q = 0; q < count; ++q) {
        const int64_t f = idx[q];
        const int64_t i = f / (m[1] * m[2]), j = (f / m[2]) % m[1], l = f % m[2];
        double acc = 0.0;
        for (int64_t a = 0; a < kd[0]; ++a)
            for (int64_t b = 0; b < kd[1]; ++b)
                for (int64_t c = 0; c < kd[2]; ++c)
                    acc += x[IDX(n, i + s[0] * a, j + s[1] * b, l + s[2] * c)] *
                           k[IDX(kd, a, b, c)];
        out[q] = acc;
    }
}

/* conv_direct.hpp:74-101; gather form of the same sum (oracles.hpp:93-116) */
void zo_conv_full(const double* g, const int64_t m[3], const double* k, const int64_t kd[3],
                  const int64_t s[3], double* out) {
    int64_t od[3];
    for (int a = 0; a < 3; ++a) od[a] = m[a] + s[a] * (kd[a] - 1);
    for (int64_t i = 0; i < od[0]; ++i)
        for (int64_t j = 0; j < od[1]; ++j)
            for (int64_t l = 0; l < od[2]; ++l) {
                double acc = 0.0;
                for (int64_t a = 0; a < kd[0]; ++a)
                    for (int64_t b = 0; b < kd[1]; ++b)
                        for (int64_t c = 0; c < kd[2]; ++c) {
                            const int64_t gi = i + s[0] * (a - (kd[0] - 1));
                            const int64_t gj = j + s[1] * (b - (kd[1] - 1));
                            const int64_t gl = l + s[2] * (c - (kd[2] - 1));
                            if (gi < 0 || gi >= m[0] || gj < 0 || gj >= m[1] || gl < 0 ||
                                gl >= m[2])
                                continue;
                            acc += k[IDX(kd, a, b, c)] * g[IDX(m, gi, gj, gl)];
                        }
                out[IDX(od, i, j, l)] = acc;
            }
}

void zo_conv_full_at(const double* g, const int64_t m[3], const double* k, const int64_t kd[3],
                     const int64_t s[3], const int64_t* idx, int64_t count, double* out) {
    int64_t od[3];
    for (int a = 0; a < 3; ++a) od[a] = m[a] + s[a] * (kd[a] - 1);
    for (int64_t q = 0; q < count; ++q) {
        const int64_t f = idx[q];
        const int64_t i = f / (od[1] * od[2]), j = (f / od[2]) % od[1], l = f % od[2];
        double acc = 0.0;
        for (int64_t a = 0; a < kd[0]; ++a)
            for (int64_t b = 0; b < kd[1]; ++b)
                for (int64_t c = 0; c < kd[2]; ++c) {
                    const int64_t gi = i + s[0] * (a - (kd[0] - 1));
                    const int64_t gj = j + s[1] * (b - (kd[1] - 1));
                    const int64_t gl = l + s[2] * (c - (kd[2] - 1));
                    if (gi < 0 || gi >= m[0] || gj < 0 || gj >= m[1] || gl < 0 || gl >= m[2])
                        continue;
                    acc += k[IDX(kd, a, b, c)] * g[IDX(m, gi, gj, gl)];
                }
        out[q] = acc;
    }
}

/* conv_direct.hpp:108-132 */
void zo_kernel_grad(const double* x, const int64_t n[3], const double* g, const int64_t m[3],
                    const int64_t kd[3], const int64_t s[3], double* out) {
    for (int64_t a = 0; a < kd[0]; ++a)
        for (int64_t b = 0; b < kd[1]; ++b)
            for (int64_t c = 0; c < kd[2]; ++c) {
                double acc = 0.0;
                for (int64_t i = 0; i < m[0]; ++i)
                    for (int64_t j = 0; j < m[1]; ++j)
                        for (int64_t l = 0; l < m[2]; ++l)
                            acc += x[IDX(n, i + s[0] * a, j + s[1] * b, l + s[2] * c)] *
                                   g[IDX(m, i, j, l)];
                out[IDX(kd, a, b, c)] = acc;
            }
}

/* volume.hpp:141-150 */
void zo_reflect(const double* x, const int64_t n[3], double* out) {
    for (int64_t i = 0; i < n[0]; ++i)
        for (int64_t j = 0; j < n[1]; ++j)
            for (int64_t l = 0; l < n[2]; ++l)
                out[IDX(n, i, j, l)] = x[IDX(n, n[0] - 1 - i, n[1] - 1 - j, n[2] - 1 - l)];
}

/* conv_direct.hpp:137-151 */
void zo_dilate(const double* k, const int64_t kd[3], const int64_t s[3], double* out) {
    int64_t e[3];
    for (int a = 0; a < 3; ++a) e[a] = s[a] * (kd[a] - 1) + 1;
    memset(out, 0, sizeof(double) * (size_t)(e[0] * e[1] * e[2]));
    for (int64_t i = 0; i < kd[0]; ++i)
        for (int64_t j = 0; j < kd[1]; ++j)
            for (int64_t l = 0; l < kd[2]; ++l)
                out[IDX(e, i * s[0], j * s[1], l * s[2])] = k[IDX(kd, i, j, l)];
}

/* maxops.hpp:32-56. For each residue class r mod s the stream r, r+s, ...
 * is scanned with a deque of stream positions whose values decrease; an
 * element evicts tail entries that are STRICTLY smaller, so among equal
 * values the earlier (lower) index survives at the head. */
void zo_sliding_max_1d(const double* in, int64_t n, int64_t stride, int64_t k, int64_t s,
                       double* out, int64_t out_stride, int32_t* argmax) {
    const int64_t m = n - s * (k - 1);
    int64_t* dq = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t r = 0; r < s; ++r) {
        int64_t head = 0, tail = 0;
        const int64_t len = (n - r + s - 1) / s;
        for (int64_t t = 0; t < len; ++t) {
            const double v = in[(r + t * s) * stride];
            while (tail > head && in[(r + dq[tail - 1] * s) * stride] < v) --tail;
            dq[tail++] = t;
            if (dq[head] <= t - k) ++head;
            if (t + 1 >= k) {
                const int64_t o = r + (t - (k - 1)) * s;
                if (o < m) {
                    const int64_t src = r + dq[head] * s;
                    out[o * out_stride] = in[src * stride];
                    if (argmax) argmax[o * out_stride] = (int32_t)src;
                }
            }
        }
    }
    free(dq);
}

/* maxops.hpp:60-88: strict '>' scan in lexicographic order */
void zo_maxpool_fwd(const double* x, const int64_t n[3], const int64_t p[3], double* out,
                    int32_t* rec) {
    const int64_t m[3] = {n[0] / p[0], n[1] / p[1], n[2] / p[2]};
    for (int64_t bi = 0; bi < m[0]; ++bi)
        for (int64_t bj = 0; bj < m[1]; ++bj)
            for (int64_t bl = 0; bl < m[2]; ++bl) {
                double best = 0.0;
                int64_t best_idx = -1;
                for (int64_t i = bi * p[0]; i < (bi + 1) * p[0]; ++i)
                    for (int64_t j = bj * p[1]; j < (bj + 1) * p[1]; ++j)
                        for (int64_t l = bl * p[2]; l < (bl + 1) * p[2]; ++l) {
                            const double v = x[IDX(n, i, j, l)];
                            if (best_idx < 0 || v > best) {
                                best = v;
                                best_idx = IDX(n, i, j, l);
                            }
                        }
                out[IDX(m, bi, bj, bl)] = best;
                rec[IDX(m, bi, bj, bl)] = (int32_t)best_idx;
            }
}

/* maxops.hpp:93-104 */
void zo_maxpool_bwd(const double* g, const int32_t* rec, const int64_t m[3],
                    const int64_t p[3], double* out) {
    const int64_t total_in = m[0] * p[0] * m[1] * p[1] * m[2] * p[2];
    memset(out, 0, sizeof(double) * (size_t)total_in);
    for (int64_t i = 0; i < m[0] * m[1] * m[2]; ++i) out[rec[i]] = g[i];
}

/* maxops.hpp:111-164 */
void zo_maxfilter_fwd(const double* x, const int64_t n[3], const int64_t k[3],
                      const int64_t s[3], double* out, int32_t* rec) {
    int64_t m[3];
    out_dims_valid(n, k, s, m);
    const int64_t d1[3] = {n[0], n[1], m[2]};
    const int64_t d2[3] = {n[0], m[1], m[2]};
    double* v1 = (double*)malloc(sizeof(double) * (size_t)(d1[0] * d1[1] * d1[2]));
    int32_t* sz = (int32_t*)malloc(sizeof(int32_t) * (size_t)(d1[0] * d1[1] * d1[2]));
    double* v2 = (double*)malloc(sizeof(double) * (size_t)(d2[0] * d2[1] * d2[2]));
    int32_t* sy = (int32_t*)malloc(sizeof(int32_t) * (size_t)(d2[0] * d2[1] * d2[2]));
    int32_t* sx = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m[0] * m[1] * m[2]));
    /* pass z */
    for (int64_t i = 0; i < n[0]; ++i)
        for (int64_t j = 0; j < n[1]; ++j)
            zo_sliding_max_1d(&x[IDX(n, i, j, 0)], n[2], 1, k[2], s[2], &v1[IDX(d1, i, j, 0)],
                              1, &sz[IDX(d1, i, j, 0)]);
    /* pass y */
    for (int64_t i = 0; i < n[0]; ++i)
        for (int64_t l = 0; l < m[2]; ++l)
            zo_sliding_max_1d(&v1[IDX(d1, i, 0, l)], n[1], m[2], k[1], s[1],
                              &v2[IDX(d2, i, 0, l)], m[2], &sy[IDX(d2, i, 0, l)]);
    /* pass x */
    for (int64_t j = 0; j < m[1]; ++j)
        for (int64_t l = 0; l < m[2]; ++l)
            zo_sliding_max_1d(&v2[IDX(d2, 0, j, l)], n[0], m[1] * m[2], k[0], s[0],
                              &out[IDX(m, 0, j, l)], m[1] * m[2], &sx[IDX(m, 0, j, l)]);
    /* resolve per-axis winners into one flat source index */
    for (int64_t i = 0; i < m[0]; ++i)
        for (int64_t j = 0; j < m[1]; ++j)
            for (int64_t l = 0; l < m[2]; ++l) {
                const int64_t xs = sx[IDX(m, i, j, l)];
                const int64_t ys = sy[IDX(d2, xs, j, l)];
                const int64_t zs = sz[IDX(d1, xs, ys, l)];
                rec[IDX(m, i, j, l)] = (int32_t)IDX(n, xs, ys, zs);
            }
    free(v1);
    free(sz);
    free(v2);
    free(sy);
    free(sx);
}

/* maxops.hpp:169-182 */
void zo_maxfilter_bwd(const double* g, const int32_t* rec, const int64_t m[3],
                      const int64_t in_dims[3], double* out) {
    memset(out, 0, sizeof(double) * (size_t)(in_dims[0] * in_dims[1] * in_dims[2]));
    for (int64_t i = 0; i < m[0] * m[1] * m[2]; ++i) out[rec[i]] += g[i];
}

/* transfer.hpp:29-36 */
double zo_transfer_value(int kind, double x) {
    switch (kind) {
        case ZO_LOGISTIC: return 1.0 / (1.0 + exp(-x));
        case ZO_TANH: return tanh(x);
        default: return x > 0.0 ? x : 0.0;
    }
}

/* transfer.hpp:40-53; relu'(0) = 0 */
double zo_transfer_derivative(int kind, double x) {
    switch (kind) {
        case ZO_LOGISTIC: {
            const double v = 1.0 / (1.0 + exp(-x));
            return v * (1.0 - v);
        }
        case ZO_TANH: {
            const double v = tanh(x);
            return 1.0 - v * v;
        }
        default: return x > 0.0 ? 1.0 : 0.0;
    }
}

void zo_transfer_fwd(const double* x, int64_t count, int kind, double bias, double* out) {
    for (int64_t i = 0; i < count; ++i) out[i] = zo_transfer_value(kind, x[i] + bias);
}

void zo_transfer_bwd(const double* g, const double* x, int64_t count, int kind, double bias,
                     double* out) {
    for (int64_t i = 0; i < count; ++i) out[i] = g[i] * zo_transfer_derivative(kind, x[i] + bias);
}

double zo_transfer_bias_grad(const double* x, const double* g, int64_t count, int kind,
                             double bias) {
    double acc = 0.0;
    for (int64_t i = 0; i < count; ++i) acc += g[i] * zo_transfer_derivative(kind, x[i] + bias);
    return acc;
}

/* taskgraph.hpp:116-126 */
double zo_loss_l2(const double* a, const double* d, int64_t count, double* grad) {
    double loss = 0.0;
    for (int64_t i = 0; i < count; ++i) {
        const double e = a[i] - d[i];
        if (grad) grad[i] = e;
        loss += 0.5 * e * e;
    }
    return loss;
}

double zo_loss_ce(const double* a, const double* d, int64_t count, double* grad_pre) {
    double loss = 0.0;
    for (int64_t i = 0; i < count; ++i) {
        const double p = a[i];
        loss -= d[i] * log(p) + (1.0 - d[i]) * log(1.0 - p);
        if (grad_pre) grad_pre[i] = p - d[i];
    }
    return loss;
}

double zo_max_rel_error(const double* a, const double* b, int64_t count) {
    double worst = 0.0;
    for (int64_t i = 0; i < count; ++i) {
        const double e = fabs(a[i] - b[i]) / (fabs(b[i]) + 1.0);
        if (e > worst || e != e) worst = e;
    }
    return worst;
}
