/*
 * znn_oracle.h — CPU restatement of the ZNN (arXiv 1510.06706) hot-path
 * arithmetic, used ONLY as the parity checker for the CUDA path.
 *
 * TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product
 * path (paper_1510_06706_b200) never links or calls it.
 *
 * Every function works on ONE per-map volume in the reference layout:
 * x-major flat index (i*ny + j)*nz + l, z contiguous (volume.hpp:21-24).
 * Scalars are double; dims are int64[3] = {x, y, z}. Argmax records are
 * int32 flat indices into the per-map input volume (maxops.hpp:24-25).
 */
#ifndef ZNN_ORACLE_H
#define ZNN_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* transfer kinds, same numbering as transfer.hpp:11 */
enum { ZO_LOGISTIC = 0, ZO_TANH = 1, ZO_RELU = 2 };

/* conv_direct.hpp:39-68 — out[o] = sum_w x[o + s*w] * k[w] */
void zo_conv_valid(const double* x, const int64_t n[3], const double* k, const int64_t kd[3],
                   const int64_t s[3], double* out);
/* same, evaluated only at the listed flat output indices (sampled parity) */
void zo_conv_valid_at(const double* x, const int64_t n[3], const double* k,
                      const int64_t kd[3], const int64_t s[3], const int64_t* idx,
                      int64_t count, double* out);
/* conv_direct.hpp:74-101 — out[t] = sum_w k[w] * g[t + s*(w - (k-1))], g zero outside */
void zo_conv_full(const double* g, const int64_t m[3], const double* k, const int64_t kd[3],
                  const int64_t s[3], double* out);
/* conv_full evaluated only at the listed flat output indices */
void zo_conv_full_at(const double* g, const int64_t m[3], const double* k, const int64_t kd[3],
                     const int64_t s[3], const int64_t* idx, int64_t count, double* out);
/* conv_direct.hpp:108-132 — dk[w] = sum_o x[o + s*w] * g[o] */
void zo_kernel_grad(const double* x, const int64_t n[3], const double* g, const int64_t m[3],
                    const int64_t kd[3], const int64_t s[3], double* out);
/* volume.hpp:141-150 — out[i,j,l] = x[nx-1-i, ny-1-j, nz-1-l] */
void zo_reflect(const double* x, const int64_t n[3], double* out);
/* conv_direct.hpp:137-151 */
void zo_dilate(const double* k, const int64_t kd[3], const int64_t s[3], double* out);

/* maxops.hpp:32-56 — monotonic-deque sliding max, lowest index on ties */
void zo_sliding_max_1d(const double* in, int64_t n, int64_t stride, int64_t k, int64_t s,
                       double* out, int64_t out_stride, int32_t* argmax);
/* maxops.hpp:60-88 */
void zo_maxpool_fwd(const double* x, const int64_t n[3], const int64_t p[3], double* out,
                    int32_t* rec);
/* maxops.hpp:93-104 */
void zo_maxpool_bwd(const double* g, const int32_t* rec, const int64_t m[3],
                    const int64_t p[3], double* out);
/* maxops.hpp:111-164 — three separable passes z, y, x; composed flat source */
void zo_maxfilter_fwd(const double* x, const int64_t n[3], const int64_t k[3],
                      const int64_t s[3], double* out, int32_t* rec);
/* maxops.hpp:169-182 — accumulate g at the recorded sources */
void zo_maxfilter_bwd(const double* g, const int32_t* rec, const int64_t m[3],
                      const int64_t in_dims[3], double* out);

/* transfer.hpp:29-53 scalar forms */
double zo_transfer_value(int kind, double x);
double zo_transfer_derivative(int kind, double x);
/* transfer.hpp:58-73 — out = phi(x + b) */
void zo_transfer_fwd(const double* x, int64_t count, int kind, double bias, double* out);
/* transfer.hpp:77-101 — out = g * phi'(x + b) */
void zo_transfer_bwd(const double* g, const double* x, int64_t count, int kind, double bias,
                     double* out);
/* transfer.hpp:111-121 — sum g * phi'(x + b) */
double zo_transfer_bias_grad(const double* x, const double* g, int64_t count, int kind,
                             double bias);

/* taskgraph.hpp:116-126 half-L2: L = 1/2 sum (a-d)^2, dL/da = a - d */
double zo_loss_l2(const double* a, const double* d, int64_t count, double* grad);
/* binomial cross-entropy on a logistic output (extension for configs 2-5):
 * L = -sum d log a + (1-d) log(1-a); grad w.r.t. the PRE-activation is a - d */
double zo_loss_ce(const double* a, const double* d, int64_t count, double* grad_pre);

/* max_i |a_i - b_i| / (|b_i| + 1)  (volume.hpp:170-176) */
double zo_max_rel_error(const double* a, const double* b, int64_t count);

#ifdef __cplusplus
}
#endif
#endif
