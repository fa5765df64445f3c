// FFT-memoised convolution engine (see fft.hpp). All transforms are
// hand-written: a 1D transform of one line runs in shared memory as a
// Stockham autosort FFT (radix 4/2/3 stages compiled per pad size, twiddles
// from a per-CTA table), 32 lines per 256-thread CTA. A 3D transform is three
// passes over a spectrum laid out [image][Px][Py][Pz/2+1] (complex64):
//   z : real -> half spectrum (R2C), one line per (x, y) of the VALID input
//   y : columns of 32 consecutive z-bins, rows y; rows beyond the valid
//       input are known zeros and are never read
//   x : same, rows x
// Inverses run x, y then z (C2R) and only write the rows / planes / voxels
// that the consumer keeps (crop to the valid output, or the s*w taps of a
// kernel gradient), so pruning comes for free from the row selections.
#include <cmath>
#include <string>
#include <type_traits>

#include "fft.hpp"

namespace znn_fft {

using znn_gpu::ceil_div;
using znn_gpu::dims3;
using znn_gpu::launch_check;
using znn_gpu::require;

namespace {

constexpr int LINES = 32;     // lines per CTA
constexpr int THREADS = 256;  // 8 threads per line
constexpr int TPL = THREADS / LINES;
constexpr int MAXP = 128;
// pad sizes with compiled transforms (2^a 3^b, every stage radix 4, 2 or 3)
constexpr int kPads[] = {2, 4, 8, 12, 16, 24, 32, 48, 64, 72, 96, 128};

// smallest compiled pad >= n
int64_t good_size(int64_t n) {
    for (int p : kPads)
        if (p >= n) return p;
    return 1 << 30;
}

__device__ __forceinline__ float2 cmul(float2 a, float2 b) { return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
// a * conj(b)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) { return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y); }

template <int R, bool INV>
__device__ __forceinline__ void dft_small(float2* v);

// radix 8 = two radix-4 DFTs of the even / odd samples merged with W8^k
template <bool INV>
__device__ __forceinline__ void dft8(float2* v) {
    float2 e[4] = {v[0], v[2], v[4], v[6]};
    float2 o[4] = {v[1], v[3], v[5], v[7]};
    dft_small<4, INV>(e);
    dft_small<4, INV>(o);
    const float c = 0.7071067811865476f;
    o[1] = INV ? make_float2(c * (o[1].x - o[1].y), c * (o[1].x + o[1].y))
               : make_float2(c * (o[1].x + o[1].y), c * (o[1].y - o[1].x));
    o[2] = INV ? make_float2(-o[2].y, o[2].x) : make_float2(o[2].y, -o[2].x);
    o[3] = INV ? make_float2(-c * (o[3].x + o[3].y), c * (o[3].x - o[3].y))
               : make_float2(c * (o[3].y - o[3].x), -c * (o[3].x + o[3].y));
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        v[k] = make_float2(e[k].x + o[k].x, e[k].y + o[k].y);
        v[k + 4] = make_float2(e[k].x - o[k].x, e[k].y - o[k].y);
    }
}

template <int R, bool INV>
__device__ __forceinline__ void dft_small(float2* v) {
    if constexpr (R == 8) {
        dft8<INV>(v);
    } else if constexpr (R == 2) {
        const float2 a = v[0], b = v[1];
        v[0] = make_float2(a.x + b.x, a.y + b.y);
        v[1] = make_float2(a.x - b.x, a.y - b.y);
    } else if constexpr (R == 4) {
        const float2 t0 = make_float2(v[0].x + v[2].x, v[0].y + v[2].y);
        const float2 t1 = make_float2(v[0].x - v[2].x, v[0].y - v[2].y);
        const float2 t2 = make_float2(v[1].x + v[3].x, v[1].y + v[3].y);
        const float2 t3 = make_float2(v[1].x - v[3].x, v[1].y - v[3].y);
        v[0] = make_float2(t0.x + t2.x, t0.y + t2.y);
        v[2] = make_float2(t0.x - t2.x, t0.y - t2.y);
        if (!INV) {  // y1 = t1 - i t3, y3 = t1 + i t3
            v[1] = make_float2(t1.x + t3.y, t1.y - t3.x);
            v[3] = make_float2(t1.x - t3.y, t1.y + t3.x);
        } else {
            v[1] = make_float2(t1.x - t3.y, t1.y + t3.x);
            v[3] = make_float2(t1.x + t3.y, t1.y - t3.x);
        }
    } else {  // R == 3
        const float s = 0.8660254037844386f;
        const float2 a = v[0], b = v[1], c = v[2];
        const float2 t1 = make_float2(b.x + c.x, b.y + c.y);
        const float2 t2 = make_float2(a.x - 0.5f * t1.x, a.y - 0.5f * t1.y);
        const float2 d = make_float2(b.x - c.x, b.y - c.y);
        v[0] = make_float2(a.x + t1.x, a.y + t1.y);
        if (!INV) {
            v[1] = make_float2(t2.x + s * d.y, t2.y - s * d.x);
            v[2] = make_float2(t2.x - s * d.y, t2.y + s * d.x);
        } else {
            v[1] = make_float2(t2.x - s * d.y, t2.y + s * d.x);
            v[2] = make_float2(t2.x + s * d.y, t2.y - s * d.x);
        }
    }
}

// twiddle table tw[m] = exp(-2 pi i m / P), m < P, in shared memory
template <int P>
__device__ __forceinline__ void fill_twiddles(float2* tw) {
    for (int m = threadIdx.x; m < P; m += blockDim.x) {
        float sn, cs;
        sincospif(-2.f * float(m) / float(P), &sn, &cs);
        tw[m] = make_float2(cs, sn);
    }
}

// One Stockham stage (Govindaraju et al. formulation): sub-transform size
// Ns grows by the stage radix R (4 while possible, then 2, then 3). All
// sizes are compile-time so index math folds to shifts / constant divides.
// Every thread of the CTA calls this (uniform __syncthreads).
template <int P, int Ns, bool INV>
__device__ __forceinline__ float2* fft_stages(float2* src, float2* dst, int t, const float2* tw) {
    if constexpr (Ns >= P) {
        return src;
    } else {
        constexpr int rem = P / Ns;
        constexpr int R = (rem % 8 == 0) ? 8 : (rem % 4 == 0) ? 4 : ((rem % 2 == 0) ? 2 : 3);
        constexpr int nb = P / R;
        constexpr int tstep = P / (Ns * R);  // stage twiddle w^(k q) = tw[k q tstep]
#pragma unroll
        for (int j0 = 0; j0 < nb; j0 += TPL) {
            const int j = j0 + t;
            if (nb % TPL == 0 || j < nb) {
                float2 v[R];
                const int k = j % Ns;
                v[0] = src[j];
#pragma unroll
                for (int q = 1; q < R; ++q) {
                    float2 w = tw[k * q * tstep];
                    if (INV) w.y = -w.y;
                    v[q] = cmul(src[j + q * nb], w);
                }
                dft_small<R, INV>(v);
                const int d = (j / Ns) * Ns * R + k;
#pragma unroll
                for (int q = 0; q < R; ++q) dst[d + q * Ns] = v[q];
            }
        }
        __syncthreads();
        return fft_stages<P, Ns * R, INV>(dst, src, t, tw);
    }
}

// ---- z pass, forward (R2C): lines (img, x < nx, y < ny) of the real input ----
template <int P>
__global__ void __launch_bounds__(THREADS) fft_z_fwd_k(const float* __restrict__ in, int64_t in_img_stride, int nx,
                                                        int ny, int nz, int64_t nlines, float2* __restrict__ spec,
                                                        int64_t spec_img_stride, int Py) {
    constexpr int Zh = P / 2 + 1;
    extern __shared__ float2 sm[];
    const int l = threadIdx.x / TPL, t = threadIdx.x % TPL;
    const int64_t line = int64_t(blockIdx.x) * LINES + l;
    const bool ok = line < nlines;
    float2* a = sm + l * (2 * P + 1);
    float2* b = a + P;
    float2* tw = sm + LINES * (2 * P + 1);
    fill_twiddles<P>(tw);
    int64_t img = 0;
    int x = 0, y = 0;
    if (ok) {  // 32-bit decode (nlines < 2^32, checked on the host)
        const uint32_t pl = uint32_t(nx) * uint32_t(ny);
        const uint32_t im = uint32_t(line) / pl;
        img = im;
        const int r = int(uint32_t(line) - im * pl);
        x = r / ny;
        y = r - x * ny;
        const float* src = in + img * in_img_stride + (int64_t(x) * ny + y) * nz;
        for (int j = t; j < P; j += TPL) a[j] = make_float2(j < nz ? src[j] : 0.f, 0.f);
    }
    __syncthreads();
    float2* res = fft_stages<P, 1, false>(a, b, t, tw);
    if (ok) {
        float2* dst = spec + img * spec_img_stride + (int64_t(x) * Py + y) * Zh;
        for (int j = t; j < Zh; j += TPL) dst[j] = res[j];
    }
}

struct col_args {
    int rows_in;                       // rows >= rows_in are zero (never read)
    int out_first, out_step, out_cnt;  // rows written
    int zh;                            // contiguous columns per plane (z-bins)
    int a_first, a_step, a_cnt;        // planes of the other spatial axis folded into the columns
    int64_t a_stride;
    int64_t row_stride;
    int64_t img_stride;
    int64_t imgs;
};

// ---- column pass (y or x axis), in place on the spectrum. Columns are
// (plane a, z-bin) pairs flattened, 32 per CTA, so no tile is mostly empty.
template <int P, bool INV>
__global__ void __launch_bounds__(THREADS) fft_col_k(float2* __restrict__ spec, col_args g) {
    extern __shared__ float2 sm[];
    const int64_t img = blockIdx.y + int64_t(blockIdx.z) * gridDim.y;
    if (img >= g.imgs) return;  // uniform per CTA
    const int ncols = g.a_cnt * g.zh;
    const int lc = threadIdx.x % LINES, lr = threadIdx.x / LINES;  // 8 rows per sweep
    const int c = blockIdx.x * LINES + lc;
    const bool cok = c < ncols;
    int64_t coff = 0;
    if (cok) {
        const int ai = c / g.zh;
        coff = int64_t(g.a_first + ai * g.a_step) * g.a_stride + (c - ai * g.zh);
    }
    float2* base = spec + img * g.img_stride + coff;
    float2* tw = sm + LINES * (2 * P + 1);
    fill_twiddles<P>(tw);
    for (int j = lr; j < P; j += THREADS / LINES) {
        float2 v = make_float2(0.f, 0.f);
        if (j < g.rows_in && cok) v = base[int64_t(j) * g.row_stride];
        sm[lc * (2 * P + 1) + j] = v;
    }
    __syncthreads();
    const int l = threadIdx.x / TPL, t = threadIdx.x % TPL;
    float2* la = sm + l * (2 * P + 1);
    float2* res = fft_stages<P, 1, INV>(la, la + P, t, tw);
    const int half = int(res - la);  // 0 or P, same for every line
    if (cok)
        for (int q = lr; q < g.out_cnt; q += THREADS / LINES) {
            const int j = g.out_first + q * g.out_step;
            base[int64_t(j) * g.row_stride] = sm[lc * (2 * P + 1) + half + j];
        }
}

struct zinv_args {
    int Py;
    int64_t spec_img_stride;
    int x_step, x_cnt, y_step, y_cnt, z_step, z_cnt;  // selections start at 0
    int64_t nlines;                                   // images * x_cnt * y_cnt
    float scale;
    int64_t out_img_stride;
    int oy, oz;                                       // output box dims (y, z)
    int act;                                          // ZNN_ACT_* (3 = none)
    int bias_mod;                                     // bias index = img % bias_mod
};

// ---- z pass, inverse (C2R) with crop / tap selection and fused epilogue ----
template <int P>
__global__ void __launch_bounds__(THREADS) fft_z_inv_k(const float2* __restrict__ spec, zinv_args g,
                                                        const float* __restrict__ bias, float* __restrict__ out) {
    constexpr int Zh = P / 2 + 1;
    extern __shared__ float2 sm[];
    const int l = threadIdx.x / TPL, t = threadIdx.x % TPL;
    const int64_t line = int64_t(blockIdx.x) * LINES + l;
    const bool ok = line < g.nlines;
    float2* a = sm + l * (2 * P + 1);
    float2* b = a + P;
    float2* tw = sm + LINES * (2 * P + 1);
    fill_twiddles<P>(tw);
    int64_t img = 0;
    int xi = 0, yi = 0;
    if (ok) {  // 32-bit decode (nlines < 2^32, checked on the host)
        const uint32_t per = uint32_t(g.x_cnt) * uint32_t(g.y_cnt);
        const uint32_t im = uint32_t(line) / per;
        img = im;
        const int r = int(uint32_t(line) - im * per);
        xi = r / g.y_cnt;
        yi = r - xi * g.y_cnt;
        const float2* src = spec + img * g.spec_img_stride + (int64_t(xi * g.x_step) * g.Py + yi * g.y_step) * Zh;
        for (int j = t; j < P; j += TPL) {
            float2 v;
            if (j < Zh) {
                v = src[j];
            } else {
                const float2 c = src[P - j];  // Hermitian symmetry of a real signal
                v = make_float2(c.x, -c.y);
            }
            a[j] = v;
        }
    }
    __syncthreads();
    float2* res = fft_stages<P, 1, true>(a, b, t, tw);
    if (ok) {
        float* dst = out + img * g.out_img_stride + (int64_t(xi) * g.oy + yi) * g.oz;
        const float bv = bias ? bias[img % g.bias_mod] : 0.f;
        for (int q = t; q < g.z_cnt; q += TPL) {
            float v = res[q * g.z_step].x * g.scale + bv;
            if (g.act == 2) v = v > 0.f ? v : 0.f;
            else if (g.act == 0) v = 1.f / (1.f + expf(-v));
            else if (g.act == 1) v = tanhf(v);
            dst[q] = v;
        }
    }
}

// dilated kernels: dil[e][f_in][s*w] = w[e][f_in][w], zeros elsewhere (conv_direct.hpp:137-151)
__global__ void dilate_k(const float* __restrict__ w, int64_t nker, int kx, int ky, int kz, int sx, int sy, int sz,
                         float* __restrict__ dil) {
    const int ex = sx * (kx - 1) + 1, ey = sy * (ky - 1) + 1, ez = sz * (kz - 1) + 1;
    const int64_t ev = int64_t(ex) * ey * ez;
    const int64_t total = nker * ev;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t kk = i < (int64_t(1) << 32) ? int64_t(uint32_t(i) / uint32_t(ev)) : i / ev;
        const int r = int(i - kk * ev);
        const int x = r / (ey * ez), y = (r / ez) % ey, z = r % ez;
        float v = 0.f;
        if (x % sx == 0 && y % sy == 0 && z % sz == 0)
            v = w[kk * (int64_t(kx) * ky * kz) + ((x / sx) * ky + y / sy) * kz + z / sz];
        dil[i] = v;
    }
}

// ---- per-frequency complex multiply-accumulate over converging edges ----
constexpr int CM_T = 128;  // threads (= frequency bins) per CTA
// register tile: 8 x 8 complex accumulators per thread; the shared operand
// (X, G) is re-read f/8 times, from L2 (tiles of one frequency block are
// adjacent in launch order), the per-edge kernel spectrum exactly once
constexpr int TA = 8, TB = 8;

// fwd: Y[b][o] = sum_i X[b][i] * conj(K[o][i])      (tile TA b x TB o)
__global__ void __launch_bounds__(CM_T) cmac_fwd_k(const float2* __restrict__ X, const float2* __restrict__ K,
                                                    float2* __restrict__ Y, int B, int f, int fo, int64_t bins) {
    const int64_t w = int64_t(blockIdx.y) * CM_T + threadIdx.x;  // tiles on x: L2 reuse of shared operands
    if (w >= bins) return;
    const int o0 = blockIdx.x * TB, b0 = blockIdx.z * TA;
    float2 acc[TA][TB];
#pragma unroll
    for (int a = 0; a < TA; ++a)
#pragma unroll
        for (int c = 0; c < TB; ++c) acc[a][c] = make_float2(0.f, 0.f);
    for (int i = 0; i < f; ++i) {
        float2 xv[TA], kv[TB];
#pragma unroll
        for (int a = 0; a < TA; ++a) xv[a] = (b0 + a < B) ? X[(int64_t(b0 + a) * f + i) * bins + w] : make_float2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < TB; ++c) kv[c] = (o0 + c < fo) ? K[(int64_t(o0 + c) * f + i) * bins + w] : make_float2(0.f, 0.f);
#pragma unroll
        for (int a = 0; a < TA; ++a)
#pragma unroll
            for (int c = 0; c < TB; ++c) {
                const float2 p = cmulc(xv[a], kv[c]);
                acc[a][c].x += p.x;
                acc[a][c].y += p.y;
            }
    }
#pragma unroll
    for (int a = 0; a < TA; ++a)
#pragma unroll
        for (int c = 0; c < TB; ++c)
            if (b0 + a < B && o0 + c < fo) Y[(int64_t(b0 + a) * fo + o0 + c) * bins + w] = acc[a][c];
}

// bwd: dX[b][i] = sum_o G[b][o] * K[o][i]    (tile TA b x TB i)
__global__ void __launch_bounds__(CM_T) cmac_bwd_k(const float2* __restrict__ G, const float2* __restrict__ K,
                                                    float2* __restrict__ DX, int B, int f, int fo, int64_t bins) {
    const int64_t w = int64_t(blockIdx.y) * CM_T + threadIdx.x;  // tiles on x: L2 reuse of shared operands
    if (w >= bins) return;
    const int i0 = blockIdx.x * TB, b0 = blockIdx.z * TA;
    float2 acc[TA][TB];
#pragma unroll
    for (int a = 0; a < TA; ++a)
#pragma unroll
        for (int c = 0; c < TB; ++c) acc[a][c] = make_float2(0.f, 0.f);
    for (int o = 0; o < fo; ++o) {
        float2 gv[TA], kv[TB];
#pragma unroll
        for (int a = 0; a < TA; ++a) gv[a] = (b0 + a < B) ? G[(int64_t(b0 + a) * fo + o) * bins + w] : make_float2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < TB; ++c) kv[c] = (i0 + c < f) ? K[(int64_t(o) * f + i0 + c) * bins + w] : make_float2(0.f, 0.f);
#pragma unroll
        for (int a = 0; a < TA; ++a)
#pragma unroll
            for (int c = 0; c < TB; ++c) {
                const float2 p = cmul(gv[a], kv[c]);
                acc[a][c].x += p.x;
                acc[a][c].y += p.y;
            }
    }
#pragma unroll
    for (int a = 0; a < TA; ++a)
#pragma unroll
        for (int c = 0; c < TB; ++c)
            if (b0 + a < B && i0 + c < f) DX[(int64_t(b0 + a) * f + i0 + c) * bins + w] = acc[a][c];
}

// upd: dK[o][i] = sum_b X[b][i] * conj(G[b][o])   (tile TU o x TU i; only B terms per
// output, so a smaller tile keeps occupancy up for the output-write-bound pass)
constexpr int TU = 4;
__global__ void __launch_bounds__(CM_T) cmac_upd_k(const float2* __restrict__ X, const float2* __restrict__ G,
                                                    float2* __restrict__ DK, int B, int f, int fo, int64_t bins) {
    const int64_t w = int64_t(blockIdx.y) * CM_T + threadIdx.x;  // tiles on x: L2 reuse of shared operands
    if (w >= bins) return;
    const int i0 = blockIdx.x * TU, o0 = blockIdx.z * TU;
    float2 acc[TU][TU];
#pragma unroll
    for (int a = 0; a < TU; ++a)
#pragma unroll
        for (int c = 0; c < TU; ++c) acc[a][c] = make_float2(0.f, 0.f);
    for (int b = 0; b < B; ++b) {
        float2 gv[TU], xv[TU];
#pragma unroll
        for (int a = 0; a < TU; ++a) gv[a] = (o0 + a < fo) ? G[(int64_t(b) * fo + o0 + a) * bins + w] : make_float2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < TU; ++c) xv[c] = (i0 + c < f) ? X[(int64_t(b) * f + i0 + c) * bins + w] : make_float2(0.f, 0.f);
#pragma unroll
        for (int a = 0; a < TU; ++a)
#pragma unroll
            for (int c = 0; c < TU; ++c) {
                const float2 p = cmulc(xv[c], gv[a]);
                acc[a][c].x += p.x;
                acc[a][c].y += p.y;
            }
    }
#pragma unroll
    for (int a = 0; a < TU; ++a)
#pragma unroll
        for (int c = 0; c < TU; ++c)
            if (o0 + a < fo && i0 + c < f) DK[(int64_t(o0 + a) * f + i0 + c) * bins + w] = acc[a][c];
}

}  // namespace

struct plan {
    dims3 P{1, 1, 1};
    int64_t Zh = 1, bins = 1;
    int64_t B = 0, f = 0, fo = 0;
    float2* X = nullptr;  // memo: image spectra of the layer input [B*f][bins]
    float2* K = nullptr;  // memo: kernel spectra [fo*f][bins]
    float* dil = nullptr; // dilated kernels [fo*f][e^3]
    transform_counts cnt;
};

void plan_deleter::operator()(plan* p) const {
    if (!p) return;
    cudaFree(p->X);
    cudaFree(p->K);
    cudaFree(p->dil);
    delete p;
}

const transform_counts& counts(const plan& p) { return p.cnt; }
void pad_dims(const plan& p, int64_t out[3]) { out[0] = p.P.x, out[1] = p.P.y, out[2] = p.P.z; }

namespace {

constexpr int64_t kMaxSpectrumBytes = int64_t(24) << 30;  // kernel spectra budget per layer

int64_t pad_axis(int64_t n) { return n <= 1 ? 1 : good_size(n); }

dims3 pads_for(const conv_shape& c) {
    dims3 P{pad_axis(c.n.x), pad_axis(c.n.y), pad_axis(c.n.z)};
    if (P.z % 2) P.z = good_size(P.z + 1);  // R2C axis must be even
    return P;
}

size_t smem_for(int P) { return sizeof(float2) * (size_t(LINES) * size_t(2 * P + 1) + size_t(P)); }

// compile-time pad dispatch: f(std::integral_constant<int, P>) for P in kPads
template <typename F>
void dispatch_pad(int P, F&& f) {
    switch (P) {
        case 2: f(std::integral_constant<int, 2>{}); break;
        case 4: f(std::integral_constant<int, 4>{}); break;
        case 8: f(std::integral_constant<int, 8>{}); break;
        case 12: f(std::integral_constant<int, 12>{}); break;
        case 16: f(std::integral_constant<int, 16>{}); break;
        case 24: f(std::integral_constant<int, 24>{}); break;
        case 32: f(std::integral_constant<int, 32>{}); break;
        case 48: f(std::integral_constant<int, 48>{}); break;
        case 64: f(std::integral_constant<int, 64>{}); break;
        case 72: f(std::integral_constant<int, 72>{}); break;
        case 96: f(std::integral_constant<int, 96>{}); break;
        case 128: f(std::integral_constant<int, 128>{}); break;
        default: throw znn_gpu::shape_error("fft: no compiled transform for pad " + std::to_string(P));
    }
}

template <typename K>
void allow_smem(K* k, int P) {
    ZNN_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_for(P))));
}

void col_pass(cudaStream_t st, const plan& p, float2* spec, int64_t imgs, bool x_axis, bool inv, int rows_in,
              int out_first, int out_step, int out_cnt, int a_first, int a_step, int a_cnt) {
    const int P = int(x_axis ? p.P.x : p.P.y);
    if (P == 1) return;  // 1-point DFT: identity
    col_args g;
    g.rows_in = rows_in;
    g.out_first = out_first, g.out_step = out_step, g.out_cnt = out_cnt;
    g.zh = int(p.Zh);
    g.img_stride = p.bins;
    if (x_axis) {
        g.row_stride = p.P.y * p.Zh;
        g.a_stride = p.Zh;  // the folded axis is y
    } else {
        g.row_stride = p.Zh;
        g.a_stride = p.P.y * p.Zh;  // the folded axis is x
    }
    g.a_first = a_first, g.a_step = a_step, g.a_cnt = a_cnt;
    g.imgs = imgs;
    const int64_t gy = imgs < 65535 ? imgs : 65535;
    const dim3 grid{unsigned(ceil_div(int64_t(a_cnt) * p.Zh, LINES)), unsigned(gy), unsigned(ceil_div(imgs, gy))};
    dispatch_pad(P, [&](auto pc) {
        constexpr int PP = decltype(pc)::value;
        if (inv) {
            allow_smem(fft_col_k<PP, true>, PP);
            fft_col_k<PP, true><<<grid, THREADS, smem_for(PP), st>>>(spec, g);
        } else {
            allow_smem(fft_col_k<PP, false>, PP);
            fft_col_k<PP, false><<<grid, THREADS, smem_for(PP), st>>>(spec, g);
        }
    });
    launch_check("fft_col");
}

// forward 3D R2C of imgs real volumes (valid dims n, image stride in floats)
void forward3d(cudaStream_t st, const plan& p, const float* in, int64_t in_img_stride, dims3 n, int64_t imgs,
               float2* spec) {
    const int64_t nlines = imgs * n.x * n.y;
    require(nlines < (int64_t(1) << 32), "fft: too many transform lines");
    dispatch_pad(int(p.P.z), [&](auto pc) {
        constexpr int PP = decltype(pc)::value;
        allow_smem(fft_z_fwd_k<PP>, PP);
        fft_z_fwd_k<PP><<<unsigned(ceil_div(nlines, LINES)), THREADS, smem_for(PP), st>>>(
            in, in_img_stride, int(n.x), int(n.y), int(n.z), nlines, spec, p.bins, int(p.P.y));
    });
    launch_check("fft_z_fwd");
    // y: planes x < n.x, rows y < n.y valid -> all Py rows
    col_pass(st, p, spec, imgs, false, false, int(n.y), 0, 1, int(p.P.y), 0, 1, int(n.x));
    // x: every y row, planes x < n.x valid -> all Px planes
    col_pass(st, p, spec, imgs, true, false, int(n.x), 0, 1, int(p.P.x), 0, 1, int(p.P.y));
}

// inverse 3D C2R keeping voxels (x,y,z) = (step*i) for i < cnt per axis,
// written as a dense box [imgs][cnt.x][cnt.y][cnt.z] (image stride given)
void inverse3d(cudaStream_t st, const plan& p, float2* spec, int64_t imgs, dims3 step, dims3 cnt, float* out,
               int64_t out_img_stride, const float* bias, int bias_mod, int act) {
    // x: all rows in, keep planes step.x * i
    col_pass(st, p, spec, imgs, true, true, int(p.P.x), 0, int(step.x), int(cnt.x), 0, 1, int(p.P.y));
    // y: on the kept planes, keep rows step.y * i
    col_pass(st, p, spec, imgs, false, true, int(p.P.y), 0, int(step.y), int(cnt.y), 0, int(step.x), int(cnt.x));
    zinv_args g;
    g.Py = int(p.P.y);
    g.spec_img_stride = p.bins;
    g.x_step = int(step.x), g.x_cnt = int(cnt.x);
    g.y_step = int(step.y), g.y_cnt = int(cnt.y);
    g.z_step = int(step.z), g.z_cnt = int(cnt.z);
    g.nlines = imgs * cnt.x * cnt.y;
    require(g.nlines < (int64_t(1) << 32), "fft: too many transform lines");
    g.scale = float(1.0 / double(p.P.x * p.P.y * p.P.z));
    g.out_img_stride = out_img_stride;
    g.oy = int(cnt.y), g.oz = int(cnt.z);
    g.act = act;
    g.bias_mod = bias_mod > 0 ? bias_mod : 1;
    dispatch_pad(int(p.P.z), [&](auto pc) {
        constexpr int PP = decltype(pc)::value;
        allow_smem(fft_z_inv_k<PP>, PP);
        fft_z_inv_k<PP><<<unsigned(ceil_div(g.nlines, LINES)), THREADS, smem_for(PP), st>>>(spec, g, bias, out);
    });
    launch_check("fft_z_inv");
}

float2* carve(char*& cur, int64_t count) {
    float2* p = reinterpret_cast<float2*>(cur);
    cur += ((sizeof(float2) * size_t(count) + 255) / 256) * 256;
    return p;
}

}  // namespace

bool supported(const conv_shape& c) {
    const dims3 P = pads_for(c);
    if (P.x > MAXP || P.y > MAXP || P.z > MAXP) return false;
    const int64_t bins = P.x * P.y * (P.z / 2 + 1);
    if (c.f_in * c.f_out * bins * int64_t(sizeof(float2)) > kMaxSpectrumBytes) return false;
    return true;
}

plan_ptr make_plan(const conv_shape& c) {
    require(supported(c), "fft engine: layer unsupported (pad > 128 or spectra exceed the memory budget)");
    plan_ptr p(new plan);
    p->P = pads_for(c);
    p->Zh = p->P.z / 2 + 1;
    p->bins = p->P.x * p->P.y * p->Zh;
    p->B = c.B, p->f = c.f_in, p->fo = c.f_out;
    const dims3 e{c.s.x * (c.k.x - 1) + 1, c.s.y * (c.k.y - 1) + 1, c.s.z * (c.k.z - 1) + 1};
    ZNN_CUDA_CHECK(cudaMalloc(&p->X, sizeof(float2) * size_t(c.B * c.f_in * p->bins)));
    ZNN_CUDA_CHECK(cudaMalloc(&p->K, sizeof(float2) * size_t(c.f_out * c.f_in * p->bins)));
    ZNN_CUDA_CHECK(cudaMalloc(&p->dil, sizeof(float) * size_t(c.f_out * c.f_in * e.vol())));
    return p;
}

void conv_fwd(cudaStream_t st, plan& p, const conv_shape& c, const float* x, const float* w, const float* bias,
              int act, float* y, znn_gpu::scratch& ws) {
    require(p.B == c.B && p.f == c.f_in && p.fo == c.f_out, "fft engine: plan/layer mismatch");
    const dims3 e{c.s.x * (c.k.x - 1) + 1, c.s.y * (c.k.y - 1) + 1, c.s.z * (c.k.z - 1) + 1};
    const int64_t nker = c.f_out * c.f_in;
    // image spectra (memoised for the backward / update passes)
    forward3d(st, p, x, c.n.vol(), c.n, c.B * c.f_in, p.X);
    p.cnt.fwd_image += c.B * c.f_in;
    // kernel spectra of the dilated kernels (memoised for the backward pass)
    int64_t blocks = ceil_div(nker * e.vol(), 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    dilate_k<<<unsigned(blocks), 256, 0, st>>>(w, nker, int(c.k.x), int(c.k.y), int(c.k.z), int(c.s.x), int(c.s.y),
                                               int(c.s.z), p.dil);
    launch_check("fft_dilate");
    forward3d(st, p, p.dil, e.vol(), e, nker, p.K);
    p.cnt.fwd_kernel += nker;
    // Y = sum_i X * conj(K), one inverse per output node, crop + bias + transfer
    char* cur = static_cast<char*>(ws.get(sizeof(float2) * size_t(c.B * c.f_out * p.bins) + 512));
    float2* Y = carve(cur, c.B * c.f_out * p.bins);
    const dim3 grid{unsigned(ceil_div(c.f_out, TB)), unsigned(ceil_div(p.bins, CM_T)), unsigned(ceil_div(c.B, TA))};
    cmac_fwd_k<<<grid, CM_T, 0, st>>>(p.X, p.K, Y, int(c.B), int(c.f_in), int(c.f_out), p.bins);
    launch_check("fft_cmac_fwd");
    inverse3d(st, p, Y, c.B * c.f_out, dims3{1, 1, 1}, c.m, y, c.m.vol(), bias, int(c.f_out), act);
    p.cnt.fwd_inverse += c.B * c.f_out;
}

void conv_bwd(cudaStream_t st, plan& p, const conv_shape& c, const float*, const float* g, const float*, float* gw,
              float* gin, znn_gpu::scratch& ws) {
    const int64_t nB = c.B;
    const size_t need = sizeof(float2) * size_t(nB * c.f_out * p.bins + nB * c.f_in * p.bins +
                                                 c.f_out * c.f_in * p.bins) + 1024;
    char* cur = static_cast<char*>(ws.get(need));
    float2* G = carve(cur, nB * c.f_out * p.bins);
    float2* DX = carve(cur, nB * c.f_in * p.bins);
    float2* DK = carve(cur, c.f_out * c.f_in * p.bins);
    // backward image spectra, padded to the tail dims (engine.hpp:757-759)
    forward3d(st, p, g, c.m.vol(), c.m, nB * c.f_out, G);
    p.cnt.bwd_image += nB * c.f_out;
    if (gin) {
        const dim3 grid{unsigned(ceil_div(c.f_in, TB)), unsigned(ceil_div(p.bins, CM_T)), unsigned(ceil_div(nB, TA))};
        cmac_bwd_k<<<grid, CM_T, 0, st>>>(G, p.K, DX, int(nB), int(c.f_in), int(c.f_out), p.bins);
        launch_check("fft_cmac_bwd");
        inverse3d(st, p, DX, nB * c.f_in, dims3{1, 1, 1}, c.n, gin, c.n.vol(), nullptr, 1, 3);
        p.cnt.bwd_inverse += nB * c.f_in;
    }
    // kernel gradient: one gradient-specific inverse per edge, sampled at s*w
    const dim3 gu{unsigned(ceil_div(c.f_in, TU)), unsigned(ceil_div(p.bins, CM_T)), unsigned(ceil_div(c.f_out, TU))};
    cmac_upd_k<<<gu, CM_T, 0, st>>>(p.X, G, DK, int(nB), int(c.f_in), int(c.f_out), p.bins);
    launch_check("fft_cmac_upd");
    inverse3d(st, p, DK, c.f_out * c.f_in, c.s, c.k, gw, c.taps(), nullptr, 1, 3);
    p.cnt.upd_inverse += c.f_out * c.f_in;
}

}  // namespace znn_fft
