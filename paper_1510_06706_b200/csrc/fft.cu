// FFT-memoised convolution engine (see fft.hpp). All transforms are
// hand-written: a 1D transform of one line runs in registers + shared memory
// as a four-step FFT (P = R1 * R2, radix 2/3/4/5/8 codelets compiled per pad
// size, twiddles from a per-CTA table), 32 lines per 256-thread CTA. Kernel
// spectra and kernel-gradient inverses do not use these passes (sparse-tap
// plane DFTs, see kspec_k / dkinv_xy_k).
//
// Spectrum layout, per image: [Pz/2+1][Px][Py] complex64 (z-bin major), so an
// (x, y) plane of one z-bin is contiguous. A 3D forward transform is two
// passes over HBM:
//   z  : real lines (x, y) of the VALID input -> half spectra (R2C), stored
//        transposed into the z-bin planes (only the valid (x, y) entries)
//   xy : one CTA per z-bin plane: loads the valid region, row FFTs (y) on the
//        valid rows, column FFTs (x) on every column, writes the whole plane
// and the inverse mirrors it:
//   xy : loads a plane, column inverse FFTs, keeps the selected rows, row
//        inverse FFTs on those, keeps the selected columns and writes the
//        compact kept block (the crop of a valid output or the s*w taps of a
//        kernel gradient)
//   z  : C2R lines of the kept (x, y) with the consumer's crop / tap stride
//        and the fused bias + transfer epilogue.
#include <algorithm>
#include <cmath>
#include <string>
#include <type_traits>

#include "bgemm_tc.hpp"
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
constexpr int kPads[] = {2, 4, 8, 12, 16, 20, 24, 32, 40, 48, 64, 72, 80, 96, 128};

// smallest compiled pad >= n
int64_t good_size(int64_t n) {
    for (int p : kPads)
        if (p >= n) return p;
    return 1 << 30;
}

__device__ __forceinline__ float2 cmul(float2 a, float2 b) { return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
// a * conj(b)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) { return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y); }
// acc += a * b and acc += a * conj(b) as four dependent-pair FMAs (the
// product-then-add form costs six FP32 instructions per complex MAC)
__device__ __forceinline__ void cmac(float& re, float& im, float ax, float ay, float bx, float by) {
    re = fmaf(ax, bx, re);
    re = fmaf(-ay, by, re);
    im = fmaf(ax, by, im);
    im = fmaf(ay, bx, im);
}
__device__ __forceinline__ void cmacc(float& re, float& im, float ax, float ay, float bx, float by) {
    re = fmaf(ax, bx, re);
    re = fmaf(ay, by, re);
    im = fmaf(ay, bx, im);
    im = fmaf(-ax, by, im);
}

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
    } else if constexpr (R == 5) {
        // X1,4 = a1 -/+ i b1, X2,3 = a2 -/+ i b2 (signs of i flipped for the inverse)
        const float c1 = 0.30901699437494745f, c2 = -0.8090169943749473f;
        const float s1 = 0.9510565162951535f, s2 = 0.5877852522924732f;
        const float2 t1 = make_float2(v[1].x + v[4].x, v[1].y + v[4].y);
        const float2 t2 = make_float2(v[2].x + v[3].x, v[2].y + v[3].y);
        const float2 t3 = make_float2(v[1].x - v[4].x, v[1].y - v[4].y);
        const float2 t4 = make_float2(v[2].x - v[3].x, v[2].y - v[3].y);
        const float2 a1 = make_float2(v[0].x + c1 * t1.x + c2 * t2.x, v[0].y + c1 * t1.y + c2 * t2.y);
        const float2 a2 = make_float2(v[0].x + c2 * t1.x + c1 * t2.x, v[0].y + c2 * t1.y + c1 * t2.y);
        const float2 b1 = make_float2(s1 * t3.x + s2 * t4.x, s1 * t3.y + s2 * t4.y);
        const float2 b2 = make_float2(s2 * t3.x - s1 * t4.x, s2 * t3.y - s1 * t4.y);
        v[0] = make_float2(v[0].x + t1.x + t2.x, v[0].y + t1.y + t2.y);
        if (!INV) {  // -i b = (b.y, -b.x)
            v[1] = make_float2(a1.x + b1.y, a1.y - b1.x);
            v[4] = make_float2(a1.x - b1.y, a1.y + b1.x);
            v[2] = make_float2(a2.x + b2.y, a2.y - b2.x);
            v[3] = make_float2(a2.x - b2.y, a2.y + b2.x);
        } else {
            v[1] = make_float2(a1.x - b1.y, a1.y + b1.x);
            v[4] = make_float2(a1.x + b1.y, a1.y - b1.x);
            v[2] = make_float2(a2.x - b2.y, a2.y + b2.x);
            v[3] = make_float2(a2.x + b2.y, a2.y - b2.x);
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

// W_P^m (conjugated for the inverse) from the table
template <int P, bool INV>
__device__ __forceinline__ float2 twid(const float2* tw, int m) {
    float2 w = tw[m % P];
    if (INV) w.y = -w.y;
    return w;
}

// DFT of R points held in registers (R in {1,2,3,4,5,6,8,9,10,12,15,16,...}); composite
// sizes are split R = A*B in registers (n = a + A b, k = kb + B ka) with
// twiddles W_R^(a kb) = W_P^(a kb P/R) from the line's table.
template <int R, int P, bool INV>
__device__ __forceinline__ void dft_r(float2* v, const float2* tw) {
    if constexpr (R == 1) {
        return;
    } else if constexpr (R == 2 || R == 3 || R == 4 || R == 5 || R == 8) {
        dft_small<R, INV>(v);
    } else {
        constexpr int A = (R % 4 == 0) ? 4 : ((R % 3 == 0) ? 3 : ((R % 2 == 0) ? 2 : 5));
        constexpr int B = R / A;
        float2 t[R];
#pragma unroll
        for (int a = 0; a < A; ++a) {
            float2 u[B];
#pragma unroll
            for (int b = 0; b < B; ++b) u[b] = v[a + A * b];
            dft_r<B, P, INV>(u, tw);
#pragma unroll
            for (int kb = 0; kb < B; ++kb) t[a * B + kb] = (a * kb == 0) ? u[kb] : cmul(u[kb], twid<P, INV>(tw, a * kb * (P / R)));
        }
#pragma unroll
        for (int kb = 0; kb < B; ++kb) {
            float2 w[A];
#pragma unroll
            for (int a = 0; a < A; ++a) w[a] = t[a * B + kb];
            dft_r<A, P, INV>(w, tw);
#pragma unroll
            for (int ka = 0; ka < A; ++ka) v[kb + B * ka] = w[ka];
        }
    }
}

// One P-point line transform by the TPL = 8 threads of a line (all in one
// warp), four-step P = R1 * R2: thread n1 < R1 holds v[n2] = x[n1 + R1 n2]
// and does an R2-point DFT in registers; twiddle W_P^(n1 k2); one exchange
// through the line's shared buffer xb (P complex); then R1-point DFTs in
// registers for k2 = t, t + 8, ..., and emit(k2 + R2 k1, X) for every output.
__host__ __device__ constexpr int line_r1(int P) { return (P % 8 == 0) ? 8 : ((P % 4 == 0) ? 4 : 2); }
// Exchange-buffer layout: group k2 of R1 values at k2 * (R1 + 1) (the
// transposed reads of thread t, xb[t * (R1 + 1) + n1], hit distinct banks)
// and a line pitch = 8 mod 16 float2, so the two lines of a half-warp (one
// 64-bit shared-memory wavefront) use disjoint bank halves.
__host__ __device__ constexpr int xpitch(int P) {
    const int v = (P / line_r1(P)) * (line_r1(P) + 1);
    return v <= 8 ? 8 : ((v - 8 + 15) / 16) * 16 + 8;
}
template <int P>
struct line_shape {
    static constexpr int R1 = line_r1(P);
    static constexpr int R2 = P / R1;
    static constexpr int XP = xpitch(P);
};

template <int P, bool INV, typename Emit>
__device__ __forceinline__ void line_fft(float2* v, float2* xb, const float2* tw, int t, Emit&& emit) {
    constexpr int R1 = line_shape<P>::R1, R2 = line_shape<P>::R2;
    if (t < R1) {
        dft_r<R2, P, INV>(v, tw);
#pragma unroll
        for (int k2 = 0; k2 < R2; ++k2) xb[k2 * (R1 + 1) + t] = (k2 == 0) ? v[k2] : cmul(v[k2], twid<P, INV>(tw, t * k2));
    }
    __syncwarp();
#pragma unroll
    for (int k2 = t; k2 < R2; k2 += TPL) {
        float2 w[R1];
#pragma unroll
        for (int n1 = 0; n1 < R1; ++n1) w[n1] = xb[k2 * (R1 + 1) + n1];
        dft_r<R1, P, INV>(w, tw);
#pragma unroll
        for (int k1 = 0; k1 < R1; ++k1) emit(k2 + R2 * k1, w[k1]);
    }
    __syncwarp();
}

// ---- phase geometry of a dilated layer's polyphase plan: phase image
// img = (b S + r) f + i of the original tensor [B][f][nx][ny][nz], phase
// r = (rx sy + ry) sz + rz holds the voxels (s q + r) ----
struct phase_geom {
    int f, nx, ny, nz;     // original tensor (maps, dims)
    int sx, sy, sz, zsh;   // sparsity; zsh = log2(sz) when sz is a power of two, else -1
    int nrx, nry, nrz;     // phase dims
};

__device__ __forceinline__ void zsplit(int z, int sz, int zsh, int& q, int& r) {
    if (zsh >= 0) {
        q = z >> zsh;
        r = z & (sz - 1);
    } else {
        q = z / sz;
        r = z - q * sz;
    }
}

// phase image img = (b S + r) f + i decoded once per CTA
struct phase_img {
    int64_t base;  // offset of map (b, i) in the original tensor
    int rx, ry, rz;
};
__device__ __forceinline__ phase_img phase_decode(const phase_geom& G, int img) {
    const int S = G.sx * G.sy * G.sz;
    const int b = img / (S * G.f), rem = img - b * S * G.f;
    const int r = rem / G.f, i = rem - r * G.f;
    phase_img d;
    d.rz = r % G.sz;
    const int t = r / G.sz;
    d.ry = t % G.sy, d.rx = t / G.sy;
    d.base = (int64_t(b) * G.f + i) * G.nx * G.ny * int64_t(G.nz);
    return d;
}
// original-tensor base of phase line (qx, qy); -1 outside the volume (ragged phase)
__device__ __forceinline__ int64_t phase_line(const phase_geom& G, const phase_img& d, int qx, int qy) {
    const int x = G.sx * qx + d.rx, y = G.sy * qy + d.ry;
    if (x >= G.nx || y >= G.ny) return -1;
    return d.base + (int64_t(x) * G.ny + y) * G.nz;
}

// Line order of the z passes over phase images: the sz z-phases of one
// original z-line are adjacent lines (line = ((g * pl) + xy) * sz + rz with
// g = (b, rx, ry, map)), so the thread groups of a warp read / write the
// interleaved voxels of the same original line together: whole sectors
// instead of every sz-th float from a different CTA. Returns the phase image.
__device__ __forceinline__ uint32_t phase_pair_line(const phase_geom& G, uint32_t line, uint32_t pl, uint32_t* xy) {
    const uint32_t sz = uint32_t(G.sz);
    const uint32_t rz = line % sz, l2 = line / sz;
    const uint32_t g = l2 / pl;
    *xy = l2 - g * pl;
    const uint32_t f = uint32_t(G.f), sxy = uint32_t(G.sx * G.sy);
    const uint32_t i = g % f, t = g / f, rxy = t % sxy, b = t / sxy;
    return ((b * sxy + rxy) * sz + rz) * f + i;
}

// Row-bin-major spectra (tensor-core plans, bgemm_tc.hpp): element (img =
// r F + c, bin) at (r bins + bin) F + c. "gF" arguments below are F for such
// spectra and 0 for image-major ones. Line order of the z passes: the F maps
// of a row are adjacent lines, so a warp's transposed z-bin stores are whole
// runs of maps. Dense: line = (r * pl + xy) * F + c. Phased: the z-phases stay
// adjacent inside each map: line = (((g * pl + xy) * F + c) * sz + rz) with
// g = (b, rx, ry). Returns the image.
__device__ __forceinline__ uint32_t rbm_line(uint32_t line, uint32_t pl, uint32_t F, uint32_t* xy) {
    const uint32_t c = line % F, l2 = line / F, r = l2 / pl;
    *xy = l2 - r * pl;
    return r * F + c;
}
__device__ __forceinline__ uint32_t phase_rbm_line(const phase_geom& G, uint32_t line, uint32_t pl, uint32_t* xy) {
    const uint32_t sz = uint32_t(G.sz), F = uint32_t(G.f);
    const uint32_t rz = line % sz, l2 = line / sz;
    const uint32_t c = l2 % F, l3 = l2 / F;
    const uint32_t g = l3 / pl;
    *xy = l3 - g * pl;
    const uint32_t sxy = uint32_t(G.sx * G.sy), rxy = g % sxy, b = g / sxy;
    return ((b * sxy + rxy) * sz + rz) * F + c;
}
// float2 index of (img, bin) in a spectrum: image-major (gF = 0) or row-bin-major
__device__ __forceinline__ int64_t spec_at(int gF, int64_t img, int64_t bins, int64_t bin) {
    return gF ? ((img / gF) * bins + bin) * gF + (img % gF) : img * bins + bin;
}

// ---- z pass, forward (R2C): lines (img, x < nx, y < ny) of the real input,
// half spectra stored transposed: spec[img][zb][x][y] ----
template <int P>
__global__ void __launch_bounds__(THREADS) fft_z_fwd_k(const float* __restrict__ in, int64_t in_img_stride, int nx,
                                                        int ny, int nz, int64_t nlines, float2* __restrict__ spec,
                                                        int Px, int Py, const float* __restrict__ gate,
                                                        phase_geom ph, int phased, int gF) {
    constexpr int Zh = P / 2 + 1;
    constexpr int R1 = line_shape<P>::R1, R2 = line_shape<P>::R2;
    extern __shared__ float2 sm[];
    __shared__ int64_t obase[LINES];
    float2* tw = sm;                   // P
    float2* xbuf = tw + P;             // LINES x P
    float2* stash = xbuf + LINES * line_shape<P>::XP;  // LINES x (Zh + 1)
    fill_twiddles<P>(tw);
    const int l = threadIdx.x / TPL, t = threadIdx.x % TPL;
    const int64_t line = int64_t(blockIdx.x) * LINES + l;
    const bool ok = line < nlines;
    float2 v[R2];
#pragma unroll
    for (int n2 = 0; n2 < R2; ++n2) v[n2] = make_float2(0.f, 0.f);
    if (ok) {  // 32-bit decode (nlines < 2^32, checked on the host)
        const uint32_t pl = uint32_t(nx) * uint32_t(ny);
        uint32_t im, rr;
        if (phased) {
            im = gF ? phase_rbm_line(ph, uint32_t(line), pl, &rr) : phase_pair_line(ph, uint32_t(line), pl, &rr);
        } else if (gF) {
            im = rbm_line(uint32_t(line), pl, uint32_t(gF), &rr);
        } else {
            im = uint32_t(line) / pl;
            rr = uint32_t(line) - im * pl;
        }
        const int r = int(rr);
        const int x = r / ny, y = r - (r / ny) * ny;
        // element j of the line: off + z0 + zs * j (phased: the phase's voxels of
        // the original tensor, valid below zlim; dense: contiguous)
        int64_t off = int64_t(im) * in_img_stride + (int64_t(x) * ny + y) * nz;
        int z0 = 0, zs = 1, zlim = nz;
        if (phased) {
            const phase_img pd = phase_decode(ph, int(im));
            off = phase_line(ph, pd, x, y);
            z0 = pd.rz, zs = ph.sz, zlim = off >= 0 ? ph.nz : 0;
        }
        if (t < R1 && off >= 0) {
            const float* src = in + off;
#pragma unroll
            for (int n2 = 0; n2 < R2; ++n2) {
                const int j = t + R1 * n2, z = z0 + zs * j;
                if (j < nz && z < zlim) v[n2].x = __ldg(src + z);
            }
            if (gate) {  // fused ReLU backward: g * (y > 0) (transfer.hpp:99-106, ReLU'(0) = 0)
                const float* gp = gate + off;
#pragma unroll
                for (int n2 = 0; n2 < R2; ++n2) {
                    const int j = t + R1 * n2, z = z0 + zs * j;
                    if (j < nz && z < zlim && !(__ldg(gp + z) > 0.f)) v[n2].x = 0.f;
                }
            }
        }
        if (t == 0) obase[l] = spec_at(gF, im, int64_t(Zh) * Px * Py, int64_t(x) * Py + y);
    }
    __syncthreads();  // twiddles
    float2* st = stash + l * (Zh + 1);
    line_fft<P, false>(v, xbuf + l * line_shape<P>::XP, tw, t, [&](int k, float2 val) {
        if (k < Zh) st[k] = val;
    });
    __syncthreads();
    // transposed store: a warp writes one z-bin of 32 consecutive lines
    const int64_t zstride = int64_t(Px) * Py * (gF ? gF : 1);
    for (int idx = threadIdx.x; idx < LINES * Zh; idx += THREADS) {
        const int l2 = idx % LINES, zb = idx / LINES;
        if (int64_t(blockIdx.x) * LINES + l2 < nlines) spec[obase[l2] + zb * zstride] = stash[l2 * (Zh + 1) + zb];
    }
}

// ---- xy pass, forward: one CTA per z-bin plane [PX][PY] (PX == PY, or PX == 1)
// rows (y transforms) of the valid rows x < nx read straight from HBM into
// the plane, then columns (x transforms) written straight back ----
template <int PX, int PY>
__global__ void __launch_bounds__(THREADS) fft_xy_fwd_k(float2* __restrict__ spec, int64_t planes, int nx, int ny) {
    constexpr int PYP = PY + 1;
    constexpr int RY1 = line_shape<PY>::R1, RY2 = line_shape<PY>::R2;
    constexpr int RX1 = line_shape<PX>::R1, RX2 = line_shape<PX>::R2;
    extern __shared__ float2 sm[];
    float2* twy = sm;                 // PY
    float2* twx = twy + PY;           // PX
    float2* xbuf = twx + PX;          // LINES x max exchange pitch
    constexpr int PM = line_shape<PX>::XP > line_shape<PY>::XP ? line_shape<PX>::XP : line_shape<PY>::XP;
    float2* pl = xbuf + LINES * PM;   // [PX][PYP]
    const int64_t q = blockIdx.x + int64_t(blockIdx.y) * gridDim.x;
    if (q >= planes) return;  // uniform per CTA
    float2* g = spec + q * (int64_t(PX) * PY);
    fill_twiddles<PY>(twy);
    if constexpr (PX > 1) fill_twiddles<PX>(twx);
    __syncthreads();
    const int l = threadIdx.x / TPL, t = threadIdx.x % TPL;
    float2* xb = xbuf + l * PM;
    for (int r0 = 0; r0 < nx; r0 += LINES) {
        const int x = r0 + l;
        const bool ok = x < nx;
        float2 v[RY2];
#pragma unroll
        for (int n2 = 0; n2 < RY2; ++n2) {
            const int y = t + RY1 * n2;
            v[n2] = (ok && t < RY1 && y < ny) ? g[x * PY + y] : make_float2(0.f, 0.f);
        }
        if constexpr (PX == 1) {
            line_fft<PY, false>(v, xb, twy, t, [&](int k, float2 val) {
                if (ok) g[k] = val;
            });
        } else {
            line_fft<PY, false>(v, xb, twy, t, [&](int k, float2 val) {
                if (ok) pl[x * PYP + k] = val;
            });
        }
    }
    if constexpr (PX > 1) {
        __syncthreads();
        for (int c0 = 0; c0 < PY; c0 += LINES) {
            const int y = c0 + l;
            const bool ok = y < PY;
            float2 v[RX2];
#pragma unroll
            for (int n2 = 0; n2 < RX2; ++n2) {
                const int x = t + RX1 * n2;
                v[n2] = (ok && t < RX1 && x < nx) ? pl[x * PYP + y] : make_float2(0.f, 0.f);
            }
            line_fft<PX, false>(v, xb, twx, t, [&](int k, float2 val) {
                if (ok) pl[k * PYP + y] = val;  // the column was consumed into registers
            });
        }
        __syncthreads();
        // coalesced write-back of the whole plane, 2 bins per 16-byte store
        for (int idx = threadIdx.x; idx < PX * PY / 2; idx += THREADS) {
            const int e = 2 * idx, x = e / PY, y = e - (e / PY) * PY;
            const float2 a = pl[x * PYP + y], b = pl[x * PYP + y + 1];
            reinterpret_cast<float4*>(g)[idx] = make_float4(a.x, a.y, b.x, b.y);
        }
    }
}

// ---- xy pass, inverse: plane -> compact kept block [xc][yc] (rows x_step*i,
// columns y_step*j) written to out plane q ----
template <int PX, int PY>
__global__ void __launch_bounds__(THREADS) fft_xy_inv_k(const float2* __restrict__ spec, float2* __restrict__ out,
                                                         int64_t planes, int x_step, int xc, int y_step, int yc) {
    constexpr int PYP = PY + 1;
    constexpr int RY1 = line_shape<PY>::R1, RY2 = line_shape<PY>::R2;
    constexpr int RX1 = line_shape<PX>::R1, RX2 = line_shape<PX>::R2;
    extern __shared__ float2 sm[];
    float2* twy = sm;
    float2* twx = twy + PY;
    float2* xbuf = twx + PX;
    constexpr int PM = line_shape<PX>::XP > line_shape<PY>::XP ? line_shape<PX>::XP : line_shape<PY>::XP;
    float2* pl = xbuf + LINES * PM;
    const int64_t q = blockIdx.x + int64_t(blockIdx.y) * gridDim.x;
    if (q >= planes) return;
    const float2* g = spec + q * (int64_t(PX) * PY);
    float2* o = out + q * (int64_t(xc) * yc);
    fill_twiddles<PY>(twy);
    if constexpr (PX > 1) fill_twiddles<PX>(twx);
    __syncthreads();
    const int l = threadIdx.x / TPL, t = threadIdx.x % TPL;
    float2* xb = xbuf + l * PM;
    if constexpr (PX > 1) {
        // coalesced load of the whole plane (16-byte loads), then column
        // inverses from shared memory; keep rows x_step * i (i < xc)
        for (int idx = threadIdx.x; idx < PX * PY / 2; idx += THREADS) {
            const int e = 2 * idx, x = e / PY, y = e - (e / PY) * PY;
            const float4 a = __ldcs(reinterpret_cast<const float4*>(g) + idx);
            pl[x * PYP + y] = make_float2(a.x, a.y);
            pl[x * PYP + y + 1] = make_float2(a.z, a.w);
        }
        __syncthreads();
        for (int c0 = 0; c0 < PY; c0 += LINES) {
            const int y = c0 + l;
            const bool ok = y < PY;
            float2 v[RX2];
#pragma unroll
            for (int n2 = 0; n2 < RX2; ++n2) {
                const int x = t + RX1 * n2;
                v[n2] = (ok && t < RX1) ? pl[x * PYP + y] : make_float2(0.f, 0.f);
            }
            line_fft<PX, true>(v, xb, twx, t, [&](int k, float2 val) {
                const int i = k / x_step;
                if (ok && i * x_step == k && i < xc) pl[i * PYP + y] = val;
            });
        }
        __syncthreads();
    }
    // row inverses of the kept rows; keep columns y_step * j (j < yc)
    for (int r0 = 0; r0 < xc; r0 += LINES) {
        const int i = r0 + l;
        const bool ok = i < xc;
        float2 v[RY2];
#pragma unroll
        for (int n2 = 0; n2 < RY2; ++n2) {
            const int y = t + RY1 * n2;
            float2 val = make_float2(0.f, 0.f);
            if (ok && t < RY1) val = (PX > 1) ? pl[i * PYP + y] : __ldcs(g + y);
            v[n2] = val;
        }
        line_fft<PY, true>(v, xb, twy, t, [&](int k, float2 val) {
            const int j = k / y_step;
            if (ok && j * y_step == k && j < yc) o[i * yc + j] = val;
        });
    }
}

// ---- persistent, double-buffered xy passes (square planes, PX == PY > 1) ----
// A CTA walks planes q, q + G, ...; the next plane streams into the second
// shared buffer with cp.async while the current one is transformed, so HBM
// traffic overlaps the shared-memory FFT work. Rows have an even pitch so
// 16-byte copies stay aligned.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16p(void* smem, const void* gmem) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// 8-byte async copy, zero-filled when !ok
__device__ __forceinline__ void cp_async8z(void* smem, const void* gmem, bool ok) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(gmem), "r"(ok ? 8 : 0) : "memory");
}
// 4-byte async copy, zero-filled when !ok
__device__ __forceinline__ void cp_async4z(void* smem, const void* gmem, bool ok) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(gmem), "r"(ok ? 4 : 0) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int P>
__global__ void __launch_bounds__(THREADS) fft_xy_inv_pipe_k(const float2* __restrict__ spec, float2* __restrict__ out,
                                                              int64_t planes, int x_step, int xc, int y_step, int yc) {
    constexpr int PP = P + 2;
    constexpr int R1 = line_shape<P>::R1, R2 = line_shape<P>::R2;
    extern __shared__ float2 sm[];
    float2* tw = sm;                       // P
    float2* xbuf = tw + P;                 // LINES x P
    float2* plb0 = xbuf + LINES * line_shape<P>::XP;       // [P][PP]
    float2* plb1 = plb0 + P * PP;
    fill_twiddles<P>(tw);
    const int l = threadIdx.x / TPL, t = threadIdx.x % TPL;
    float2* xb = xbuf + l * line_shape<P>::XP;
    auto issue = [&](int64_t qq, float2* dst) {
        if (qq < planes) {
            const float2* g = spec + qq * (int64_t(P) * P);
            for (int idx = threadIdx.x; idx < P * P / 2; idx += THREADS) {
                const int e = 2 * idx, x = e / P, y = e - (e / P) * P;
                cp_async16p(dst + x * PP + y, g + e);
            }
        }
        cp_commit();
    };
    int64_t q = blockIdx.x;
    issue(q, plb0);
    int buf = 0;
    for (; q < planes; q += gridDim.x) {
        float2* pl = buf ? plb1 : plb0;
        issue(q + gridDim.x, buf ? plb0 : plb1);
        cp_wait<1>();
        __syncthreads();
        // column inverses; keep rows x_step * i (i < xc), compacted into rows i
        for (int c0 = 0; c0 < P; c0 += LINES) {
            const int y = c0 + l;
            const bool ok = y < P;  // planes narrower than LINES
            float2 v[R2];
#pragma unroll
            for (int n2 = 0; n2 < R2; ++n2) v[n2] = (ok && t < R1) ? pl[(t + R1 * n2) * PP + y] : make_float2(0.f, 0.f);
            line_fft<P, true>(v, xb, tw, t, [&](int k, float2 val) {
                const int i = k / x_step;
                if (ok && i * x_step == k && i < xc) pl[i * PP + y] = val;
            });
        }
        __syncthreads();
        float2* o = out + q * (int64_t(xc) * yc);
        for (int r0 = 0; r0 < xc; r0 += LINES) {
            const int i = r0 + l;
            const bool ok = i < xc;
            float2 v[R2];
#pragma unroll
            for (int n2 = 0; n2 < R2; ++n2) v[n2] = (ok && t < R1) ? pl[i * PP + t + R1 * n2] : make_float2(0.f, 0.f);
            line_fft<P, true>(v, xb, tw, t, [&](int k, float2 val) {
                const int j = k / y_step;
                if (ok && j * y_step == k && j < yc) o[i * yc + j] = val;
            });
        }
        __syncthreads();  // this buffer is refilled by the next iteration's prefetch
        buf ^= 1;
    }
}

template <int P>
__global__ void __launch_bounds__(THREADS) fft_xy_fwd_pipe_k(float2* __restrict__ spec, int64_t planes, int nx, int ny) {
    constexpr int PP = P + 2;
    constexpr int R1 = line_shape<P>::R1, R2 = line_shape<P>::R2;
    extern __shared__ float2 sm[];
    float2* tw = sm;
    float2* xbuf = tw + P;
    float2* plb0 = xbuf + LINES * line_shape<P>::XP;
    float2* plb1 = plb0 + P * PP;
    fill_twiddles<P>(tw);
    const int l = threadIdx.x / TPL, t = threadIdx.x % TPL;
    float2* xb = xbuf + l * line_shape<P>::XP;
    auto issue = [&](int64_t qq, float2* dst) {  // the valid nx x ny region written by the z pass
        if (qq < planes) {
            const float2* g = spec + qq * (int64_t(P) * P);
            for (int idx = threadIdx.x; idx < nx * ny; idx += THREADS) {
                const int x = idx / ny, y = idx - (idx / ny) * ny;
                cp_async8(dst + x * PP + y, g + x * P + y);
            }
        }
        cp_commit();
    };
    int64_t q = blockIdx.x;
    issue(q, plb0);
    int buf = 0;
    for (; q < planes; q += gridDim.x) {
        float2* pl = buf ? plb1 : plb0;
        issue(q + gridDim.x, buf ? plb0 : plb1);
        cp_wait<1>();
        __syncthreads();
        for (int r0 = 0; r0 < nx; r0 += LINES) {  // rows (y transforms) of the valid rows
            const int x = r0 + l;
            const bool ok = x < nx;
            float2 v[R2];
#pragma unroll
            for (int n2 = 0; n2 < R2; ++n2) {
                const int y = t + R1 * n2;
                v[n2] = (ok && t < R1 && y < ny) ? pl[x * PP + y] : make_float2(0.f, 0.f);
            }
            line_fft<P, false>(v, xb, tw, t, [&](int k, float2 val) {
                if (ok) pl[x * PP + k] = val;
            });
        }
        __syncthreads();
        for (int c0 = 0; c0 < P; c0 += LINES) {  // columns (x transforms); rows >= nx are zero
            const int y = c0 + l;
            const bool ok = y < P;  // planes narrower than LINES
            float2 v[R2];
#pragma unroll
            for (int n2 = 0; n2 < R2; ++n2) {
                const int x = t + R1 * n2;
                v[n2] = (ok && t < R1 && x < nx) ? pl[x * PP + y] : make_float2(0.f, 0.f);
            }
            line_fft<P, false>(v, xb, tw, t, [&](int k, float2 val) {
                if (ok) pl[k * PP + y] = val;
            });
        }
        __syncthreads();
        float4* g4 = reinterpret_cast<float4*>(spec + q * (int64_t(P) * P));
        for (int idx = threadIdx.x; idx < P * P / 2; idx += THREADS) {
            const int e = 2 * idx, x = e / P, y = e - (e / P) * P;
            const float2 a = pl[x * PP + y], b = pl[x * PP + y + 1];
            __stcs(g4 + idx, make_float4(a.x, a.y, b.x, b.y));
        }
        __syncthreads();  // this buffer is refilled by the next iteration's prefetch
        buf ^= 1;
    }
}

// ---- single-input-map layers (f_in = 1): the CMACs have no reduction over
// input maps, so they fuse into the plane passes and the product spectra
// never touch HBM ----
// forward: Y[b][o] = X[b] * conj(K[o]) formed while loading each plane, then
// the inverse xy pass (keep rows / columns) -> compact planes
template <int P>
__global__ void __launch_bounds__(THREADS) fft_xy_inv_mul1_k(const float2* __restrict__ X, const float2* __restrict__ K,
                                                              float2* __restrict__ out, int64_t planes, int fo, int Zh,
                                                              int x_step, int xc, int y_step, int yc) {
    constexpr int PP = P + 2;
    constexpr int R1 = line_shape<P>::R1, R2 = line_shape<P>::R2;
    extern __shared__ float2 sm[];
    float2* tw = sm;
    float2* xbuf = tw + P;
    float2* pl = xbuf + LINES * line_shape<P>::XP;  // [P][PP]
    fill_twiddles<P>(tw);
    const int l = threadIdx.x / TPL, t = threadIdx.x % TPL;
    float2* xb = xbuf + l * line_shape<P>::XP;
    for (int64_t q = blockIdx.x; q < planes; q += gridDim.x) {
        const int64_t img = q / Zh;
        const int zb = int(q - img * Zh);
        const int64_t b = img / fo, o = img - (img / fo) * fo;
        const float4* xs = reinterpret_cast<const float4*>(X + (b * Zh + zb) * int64_t(P) * P);
        const float4* ks = reinterpret_cast<const float4*>(K + (o * Zh + zb) * int64_t(P) * P);
        __syncthreads();  // previous plane fully consumed
        for (int idx = threadIdx.x; idx < P * P / 2; idx += THREADS) {
            const int e = 2 * idx, x = e / P, y = e - (e / P) * P;
            const float4 a = __ldg(xs + idx), kk = __ldg(ks + idx);
            pl[x * PP + y] = cmulc(make_float2(a.x, a.y), make_float2(kk.x, kk.y));
            pl[x * PP + y + 1] = cmulc(make_float2(a.z, a.w), make_float2(kk.z, kk.w));
        }
        __syncthreads();
        for (int c0 = 0; c0 < P; c0 += LINES) {  // column inverses, keep rows x_step * i
            const int y = c0 + l;
            const bool ok = y < P;
            float2 v[R2];
#pragma unroll
            for (int n2 = 0; n2 < R2; ++n2) v[n2] = (ok && t < R1) ? pl[(t + R1 * n2) * PP + y] : make_float2(0.f, 0.f);
            line_fft<P, true>(v, xb, tw, t, [&](int k, float2 val) {
                const int i = k / x_step;
                if (ok && i * x_step == k && i < xc) pl[i * PP + y] = val;
            });
        }
        __syncthreads();
        float2* o_ = out + q * (int64_t(xc) * yc);
        for (int r0 = 0; r0 < xc; r0 += LINES) {  // row inverses of the kept rows
            const int i = r0 + l;
            const bool ok = i < xc;
            float2 v[R2];
#pragma unroll
            for (int n2 = 0; n2 < R2; ++n2) v[n2] = (ok && t < R1) ? pl[i * PP + t + R1 * n2] : make_float2(0.f, 0.f);
            line_fft<P, true>(v, xb, tw, t, [&](int k, float2 val) {
                const int j = k / y_step;
                if (ok && j * y_step == k && j < yc) o_[i * yc + j] = val;
            });
        }
    }
}

// backward (no input gradient): for each (o, z-bin) the CTA transforms the
// z-pass planes G[b][o] of every patch (rows, then columns) and accumulates
// dK[o] = sum_b X[b] * conj(G[b][o]) in registers; only dK is written
template <int P>
__global__ void __launch_bounds__(THREADS) fft_xy_fwd_upd1_k(const float2* __restrict__ gz, const float2* __restrict__ X,
                                                              float2* __restrict__ DK, int64_t planes, int B, int fo,
                                                              int Zh, int nx, int ny) {
    constexpr int PP = P + 2;
    constexpr int R1 = line_shape<P>::R1, R2 = line_shape<P>::R2;
    constexpr int E = (P * P + THREADS - 1) / THREADS;  // plane elements per thread
    extern __shared__ float2 sm[];
    float2* tw = sm;
    float2* xbuf = tw + P;
    float2* pl = xbuf + LINES * line_shape<P>::XP;
    fill_twiddles<P>(tw);
    const int l = threadIdx.x / TPL, t = threadIdx.x % TPL;
    float2* xb = xbuf + l * line_shape<P>::XP;
    for (int64_t q = blockIdx.x; q < planes; q += gridDim.x) {  // q = o * Zh + zb
        const int64_t o = q / Zh;
        const int zb = int(q - o * Zh);
        float2 acc[E];
#pragma unroll
        for (int i = 0; i < E; ++i) acc[i] = make_float2(0.f, 0.f);
        for (int b = 0; b < B; ++b) {
            const float2* g = gz + ((int64_t(b) * fo + o) * Zh + zb) * int64_t(P) * P;
            __syncthreads();  // previous plane fully consumed
            for (int r0 = 0; r0 < nx; r0 += LINES) {  // rows (y transforms) of the valid rows, from HBM
                const int x = r0 + l;
                const bool ok = x < nx;
                float2 v[R2];
#pragma unroll
                for (int n2 = 0; n2 < R2; ++n2) {
                    const int y = t + R1 * n2;
                    v[n2] = (ok && t < R1 && y < ny) ? __ldcs(g + x * P + y) : make_float2(0.f, 0.f);
                }
                line_fft<P, false>(v, xb, tw, t, [&](int k, float2 val) {
                    if (ok) pl[x * PP + k] = val;
                });
            }
            __syncthreads();
            for (int c0 = 0; c0 < P; c0 += LINES) {  // columns (x transforms); rows >= nx are zero
                const int y = c0 + l;
                const bool ok = y < P;
                float2 v[R2];
#pragma unroll
                for (int n2 = 0; n2 < R2; ++n2) {
                    const int x = t + R1 * n2;
                    v[n2] = (ok && t < R1 && x < nx) ? pl[x * PP + y] : make_float2(0.f, 0.f);
                }
                line_fft<P, false>(v, xb, tw, t, [&](int k, float2 val) {
                    if (ok) pl[k * PP + y] = val;
                });
            }
            __syncthreads();
            const float2* xs = X + (int64_t(b) * Zh + zb) * int64_t(P) * P;
#pragma unroll
            for (int i = 0; i < E; ++i) {
                const int e = threadIdx.x + i * THREADS;
                if (e < P * P) {
                    const int x = e / P, y = e - (e / P) * P;
                    const float2 xv = __ldg(xs + e), kv = pl[x * PP + y];
                    cmacc(acc[i].x, acc[i].y, xv.x, xv.y, kv.x, kv.y);
                }
            }
        }
        float2* dk = DK + q * int64_t(P) * P;
#pragma unroll
        for (int i = 0; i < E; ++i) {
            const int e = threadIdx.x + i * THREADS;
            if (e < P * P) dk[e] = acc[i];
        }
    }
}

// ---- fused 3D transforms of small pads (P <= 32): one CTA holds an
// image's whole half spectrum [Zh][P][P] in shared memory and runs the z,
// y and x line passes there, so each image is read once and its spectrum
// written once (the split z / xy passes round-trip the spectrum through HBM
// and leave most of a CTA idle on 12-24 point planes). Sources / outputs
// are dense boxes or, for polyphase plans, the phases of the original
// tensor addressed in place (no split / merge pass). ----
constexpr int SMALLP = 32;

struct cube_io {
    const float* src;        // forward: real images (dense) or the original tensor (phased)
    const float* gate;       // forward: fused ReLU backward gate (same addressing), or null
    float* dst;              // inverse: output (dense box) or the original tensor (phased)
    int64_t img_stride;      // dense addressing: floats between images
    int nx, ny, nz;          // forward: valid input dims of an image
    int xs, xc, ys, yc, zs, zc;  // inverse: kept voxels (step * i, i < count) per axis
    int oy, oz;              // inverse dense box dims
    int bias_mod, act;
    float scale;
    int phased;
    phase_geom ph;
    int gF;                  // row-bin-major spectra: maps per row (0: image-major)
    int vec4;                // dense z lines of whole float4s (16-byte aligned): vector loads / stores
};

template <int P>
constexpr size_t cube_smem() {
    return sizeof(float2) * (size_t(P) + size_t(LINES) * size_t(line_shape<P>::XP) +
                             size_t(P / 2 + 1) * size_t(P) * size_t(P + 1));
}
// the forward stages the whole real image in shared memory first (every load
// of the CTA in flight at once) when it fits beside the cube
template <int P>
constexpr bool cube_pref() { return false; }  // staging the image cost occupancy (measured slower); kept for reference
template <int P>
constexpr size_t cube_fwd_smem() {
    return cube_smem<P>() + (cube_pref<P>() ? sizeof(float) * size_t(P) * P * P : 0);
}

template <int P>
__global__ void __launch_bounds__(THREADS) fft3_fwd_small_k(cube_io a, float2* __restrict__ spec) {
    constexpr int Zh = P / 2 + 1, PYP = P + 1;
    constexpr int R1 = line_shape<P>::R1, R2 = line_shape<P>::R2;
    extern __shared__ float2 sm[];
    float2* tw = sm;
    float2* xbuf = tw + P;
    float2* cube = xbuf + LINES * line_shape<P>::XP;  // [Zh][P][PYP]
    float* inb = reinterpret_cast<float*>(cube + Zh * P * PYP);  // [nx][ny][nz] (cube_pref)
    fill_twiddles<P>(tw);
    const int img = blockIdx.x;
    const int l = threadIdx.x / TPL, t = threadIdx.x % TPL;
    float2* xb = xbuf + l * line_shape<P>::XP;
    phase_img pd{};
    if (a.phased) pd = phase_decode(a.ph, img);
    // source of voxel (x, y, z) of this image: -1 = zero padding
    auto src_of = [&](int x, int y, int z) -> int64_t {
        if (a.phased) {
            const int64_t b = phase_line(a.ph, pd, x, y);
            const int zz = pd.rz + a.ph.sz * z;
            return (b >= 0 && zz < a.ph.nz) ? b + zz : -1;
        }
        return int64_t(img) * a.img_stride + (int64_t(x) * a.ny + y) * a.nz + z;
    };
    const int nl1 = a.nx * a.ny;
    if constexpr (cube_pref<P>()) {
        // the whole real image into shared memory: a warp per z-line (lanes
        // along z, nz <= 32), four lines' loads in flight per warp
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int l0 = warp; l0 < nl1; l0 += 4 * (THREADS / 32)) {
            float v4[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int ln = l0 + u * (THREADS / 32);
                v4[u] = 0.f;
                if (ln < nl1 && lane < a.nz) {
                    const int x = ln / a.ny, y = ln - x * a.ny;
                    int64_t o;
                    if (a.phased) {
                        const int64_t b = phase_line(a.ph, pd, x, y);
                        const int zz = pd.rz + a.ph.sz * lane;
                        o = (b >= 0 && zz < a.ph.nz) ? b + zz : -1;
                    } else {
                        o = int64_t(img) * a.img_stride + int64_t(ln) * a.nz + lane;
                    }
                    if (o >= 0) {
                        float val = __ldg(a.src + o);
                        if (a.gate && !(__ldg(a.gate + o) > 0.f)) val = 0.f;
                        v4[u] = val;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int ln = l0 + u * (THREADS / 32);
                if (ln < nl1 && lane < a.nz) inb[ln * a.nz + lane] = v4[u];
            }
        }
    }
    __syncthreads();
    // z lines (R2C) of the valid (x, y) lines; the next group's loads are
    // issued before this group's transform (register double buffer)
    auto load_line = [&](int ln, float (&r)[R2]) {
#pragma unroll
        for (int n2 = 0; n2 < R2; ++n2) r[n2] = 0.f;
        if (ln < nl1 && t < R1) {
            const int x = ln / a.ny, y = ln - (ln / a.ny) * a.ny;
#pragma unroll
            for (int n2 = 0; n2 < R2; ++n2) {
                const int z = t + R1 * n2;
                if (z < a.nz) {
                    if constexpr (cube_pref<P>()) {
                        r[n2] = inb[ln * a.nz + z];
                    } else {
                        const int64_t o = src_of(x, y, z);
                        if (o >= 0) {
                            float val = __ldg(a.src + o);
                            if (a.gate && !(__ldg(a.gate + o) > 0.f)) val = 0.f;
                            r[n2] = val;
                        }
                    }
                }
            }
        }
    };
    float nxt[R2];
    load_line(l, nxt);
    for (int b0 = 0; b0 < nl1; b0 += LINES) {
        const int ln = b0 + l;
        const bool ok = ln < nl1;
        const int x = ok ? ln / a.ny : 0, y = ok ? ln - (ln / a.ny) * a.ny : 0;
        float2 v[R2];
#pragma unroll
        for (int n2 = 0; n2 < R2; ++n2) v[n2] = make_float2(nxt[n2], 0.f);
        load_line(ln + LINES, nxt);
        line_fft<P, false>(v, xb, tw, t, [&](int k, float2 val) {
            if (ok && k < Zh) cube[(k * P + x) * PYP + y] = val;
        });
    }
    __syncthreads();
    // y lines of the valid rows x < nx (columns y >= ny are the zero padding)
    const int nl2 = Zh * a.nx;
    for (int b0 = 0; b0 < nl2; b0 += LINES) {
        const int ln = b0 + l;
        const bool ok = ln < nl2;
        const int zb = ok ? ln / a.nx : 0, x = ok ? ln - (ln / a.nx) * a.nx : 0;
        float2* row = cube + (zb * P + x) * PYP;
        float2 v[R2];
#pragma unroll
        for (int n2 = 0; n2 < R2; ++n2) {
            const int y = t + R1 * n2;
            v[n2] = (ok && t < R1 && y < a.ny) ? row[y] : make_float2(0.f, 0.f);
        }
        line_fft<P, false>(v, xb, tw, t, [&](int k, float2 val) {
            if (ok) row[k] = val;
        });
    }
    __syncthreads();
    // x lines of every column (rows x >= nx are the zero padding)
    const int nl3 = Zh * P;
    for (int b0 = 0; b0 < nl3; b0 += LINES) {
        const int ln = b0 + l;
        const bool ok = ln < nl3;
        const int zb = ok ? ln / P : 0, y = ok ? ln - (ln / P) * P : 0;
        float2* col = cube + zb * P * PYP + y;
        float2 v[R2];
#pragma unroll
        for (int n2 = 0; n2 < R2; ++n2) {
            const int x = t + R1 * n2;
            v[n2] = (ok && t < R1 && x < a.nx) ? col[x * PYP] : make_float2(0.f, 0.f);
        }
        line_fft<P, false>(v, xb, tw, t, [&](int k, float2 val) {
            if (ok) col[k * PYP] = val;
        });
    }
    __syncthreads();
    // the whole half spectrum out, [Zh][P][P], two bins per 16-byte store
    float4* g4 = reinterpret_cast<float4*>(spec + int64_t(img) * (Zh * P * P));
    for (int idx = threadIdx.x; idx < Zh * P * P / 2; idx += THREADS) {
        const int e = 2 * idx, zb = e / (P * P), r = e - zb * (P * P), x = r / P, y = r - x * P;
        const float2 u = cube[(zb * P + x) * PYP + y], w = cube[(zb * P + x) * PYP + y + 1];
        __stcs(g4 + idx, make_float4(u.x, u.y, w.x, w.y));
    }
}

template <int P, bool UNIT>  // UNIT: every kept voxel step is 1 (no per-output division)
__global__ void __launch_bounds__(THREADS) fft3_inv_small_k(const float2* __restrict__ spec, cube_io a,
                                                            const float* __restrict__ bias) {
    constexpr int Zh = P / 2 + 1, PYP = P + 1;
    constexpr int R1 = line_shape<P>::R1, R2 = line_shape<P>::R2;
    extern __shared__ float2 sm[];
    float2* tw = sm;
    float2* xbuf = tw + P;
    float2* cube = xbuf + LINES * line_shape<P>::XP;
    fill_twiddles<P>(tw);
    const int img = blockIdx.x;
    const int l = threadIdx.x / TPL, t = threadIdx.x % TPL;
    float2* xb = xbuf + l * line_shape<P>::XP;
    const float4* g4 = reinterpret_cast<const float4*>(spec + int64_t(img) * (Zh * P * P));
    constexpr int NV = Zh * P * P / 2;
    for (int i0 = threadIdx.x; i0 < NV; i0 += 4 * THREADS) {  // 4 x 16-byte loads in flight per thread
        float4 u4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (i0 + u * THREADS < NV) u4[u] = __ldcs(g4 + i0 + u * THREADS);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int idx = i0 + u * THREADS;
            if (idx < NV) {
                const int e = 2 * idx, zb = e / (P * P), r = e - zb * (P * P), x = r / P, y = r - x * P;
                cube[(zb * P + x) * PYP + y] = make_float2(u4[u].x, u4[u].y);
                cube[(zb * P + x) * PYP + y + 1] = make_float2(u4[u].z, u4[u].w);
            }
        }
    }
    phase_img pd{};
    if (a.phased) pd = phase_decode(a.ph, img);
    __syncthreads();
    // x lines (columns), keep rows xs * i, i < xc, compacted into rows i
    const int nl1 = Zh * P;
    for (int b0 = 0; b0 < nl1; b0 += LINES) {
        const int ln = b0 + l;
        const bool ok = ln < nl1;
        const int zb = ok ? ln / P : 0, y = ok ? ln - (ln / P) * P : 0;
        float2* col = cube + zb * P * PYP + y;
        float2 v[R2];
#pragma unroll
        for (int n2 = 0; n2 < R2; ++n2) v[n2] = (ok && t < R1) ? col[(t + R1 * n2) * PYP] : make_float2(0.f, 0.f);
        line_fft<P, true>(v, xb, tw, t, [&](int k, float2 val) {
            const int i = UNIT ? k : k / a.xs;
            if (ok && (UNIT || i * a.xs == k) && i < a.xc) col[i * PYP] = val;
        });
    }
    __syncthreads();
    // y lines of the kept rows, keep columns ys * j, j < yc
    const int nl2 = Zh * a.xc;
    for (int b0 = 0; b0 < nl2; b0 += LINES) {
        const int ln = b0 + l;
        const bool ok = ln < nl2;
        const int zb = ok ? ln / a.xc : 0, i = ok ? ln - (ln / a.xc) * a.xc : 0;
        float2* row = cube + (zb * P + i) * PYP;
        float2 v[R2];
#pragma unroll
        for (int n2 = 0; n2 < R2; ++n2) v[n2] = (ok && t < R1) ? row[t + R1 * n2] : make_float2(0.f, 0.f);
        line_fft<P, true>(v, xb, tw, t, [&](int k, float2 val) {
            const int j = UNIT ? k : k / a.ys;
            if (ok && (UNIT || j * a.ys == k) && j < a.yc) row[j] = val;
        });
    }
    __syncthreads();
    // z lines (C2R) of the kept (i, j), keep zs * q, q < zc; scale, bias, transfer
    const int nl3 = a.xc * a.yc;
    const float bv = bias ? bias[img % a.bias_mod] : 0.f;
    for (int b0 = 0; b0 < nl3; b0 += LINES) {
        const int ln = b0 + l;
        const bool ok = ln < nl3;
        const int i = ok ? ln / a.yc : 0, j = ok ? ln - (ln / a.yc) * a.yc : 0;
        float2 v[R2];
#pragma unroll
        for (int n2 = 0; n2 < R2; ++n2) {
            const int zz = t + R1 * n2;
            float2 val = make_float2(0.f, 0.f);
            if (ok && t < R1) {
                if (zz < Zh) {
                    val = cube[(zz * P + i) * PYP + j];
                } else {  // Hermitian symmetry of a real signal
                    const float2 c = cube[((P - zz) * P + i) * PYP + j];
                    val = make_float2(c.x, -c.y);
                }
            }
            v[n2] = val;
        }
        int64_t base = -1;
        const int rz = pd.rz;
        if (ok) {
            if (a.phased)
                base = phase_line(a.ph, pd, i, j);
            else
                base = int64_t(img) * a.img_stride + (int64_t(i) * a.oy + j) * a.oz;
        }
        line_fft<P, true>(v, xb, tw, t, [&](int k, float2 val) {
            const int q = UNIT ? k : k / a.zs;
            if (base >= 0 && (UNIT || q * a.zs == k) && q < a.zc) {
                float r = val.x * a.scale + bv;
                if (a.act == 2) r = r > 0.f ? r : 0.f;
                else if (a.act == 0) r = 1.f / (1.f + expf(-r));
                else if (a.act == 1) r = tanhf(r);
                if (a.phased) {
                    const int z = rz + a.ph.sz * q;
                    if (z < a.ph.nz) a.dst[base + z] = r;
                } else {
                    a.dst[base + q] = r;
                }
            }
        });
    }
}

// ---- small cubes, one line per thread (P <= 24): a thread holds a whole
// P-point line in registers and transforms it with the register codelets
// (dft_r, natural-order output), so a pass over Zh*P lines is one or two
// iterations of the CTA with no exchange buffer and no warp sync; the cube
// needs only the twiddle table beside it (more CTAs per SM) ----
constexpr int REGP = 24;
constexpr int RTHREADS = 256;
// threads of a cube CTA: 512 when it holds four cubes (one CTA per SM at
// P = 20: the extra warps hide the load latency), else 256
template <int NI>
__host__ __device__ constexpr int cube_threads() { return NI >= 4 ? 512 : RTHREADS; }

// NI images per CTA: NI = 1 image-major spectra; NI > 1 (tensor-core plans) the
// NI consecutive maps of one row of a row-bin-major spectrum (bgemm_tc.hpp),
// whose bins are NI * 8-byte pieces: whole 16 / 32-byte pieces per bin
template <int P, int NI = 1>
constexpr size_t cube_reg_smem() {
    return sizeof(float2) * (size_t(P) + size_t(NI) * size_t(P / 2 + 1) * size_t(P) * size_t(P + 1));
}
// images per CTA of the row-bin-major cube kernels: four cubes when they fit
// in ~80 KB (whole 32-byte sectors per bin), else two
// (ZNN_FFT_GRP_NI = 1 / 2 / 4 overrides: 1 = one image per CTA, 8-byte pieces merged in L2)
int grp_ni_env(const char* name, int dflt) {
    const char* e = std::getenv(name);
    const int v = e ? std::atoi(e) : dflt;
    return (v == 1 || v == 2 || v == 4) ? v : dflt;
}
// measured on c5 with row-bin-major spectra (in-step, four transforms per
// layer): four images per CTA at every pad (P = 20: 30.4 ms vs 31.0 / 37.5 for
// one / two; P = 16: 12.1 vs 14.5 / 12.3; P = 12: 4.7 vs 4.9 for two)
// with phase-major tensors and lane-pair stores (in-step, c5): the inverse at
// P = 16 runs faster with two cubes per CTA (three CTAs per SM: dgrad 1.65 vs
// 2.00 ms, image 1.31 vs 1.83); P = 20 inverses need the whole 32-byte pieces
// (3.8 vs 7.1 ms), forwards are within 5% either way
template <int P>
int cube_grp_ni(bool inverse = false) { return grp_ni_env("ZNN_FFT_GRP_NI", inverse && P == 16 ? 2 : 4); }

// row-bin-major piece of NI images at one bin: NI float2 <-> NI / 2 float4
template <int NI>
__device__ __forceinline__ void grp_put(float2* __restrict__ dst, const float2 (&v)[NI]) {
    if constexpr (NI == 1) {
        __stcs(dst, v[0]);
    } else {
        float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
        for (int j = 0; j < NI / 2; ++j)
            __stcs(d4 + j, make_float4(v[2 * j].x, v[2 * j].y, v[2 * j + 1].x, v[2 * j + 1].y));
    }
}
template <int NI>
__device__ __forceinline__ void grp_get(const float2* __restrict__ src, float2 (&v)[NI]) {
    if constexpr (NI == 1) {
        v[0] = __ldcs(src);
    } else {
        const float4* s4 = reinterpret_cast<const float4*>(src);
#pragma unroll
        for (int j = 0; j < NI / 2; ++j) {
            const float4 u = __ldcs(s4 + j);
            v[2 * j] = make_float2(u.x, u.y);
            v[2 * j + 1] = make_float2(u.z, u.w);
        }
    }
}

template <int P, int NI, bool GL = (NI > 1)>
__global__ void __launch_bounds__(cube_threads<NI>()) fft3_fwd_reg_k(cube_io a, float2* __restrict__ spec) {
    constexpr int CT = cube_threads<NI>();
    constexpr int Zh = P / 2 + 1, PYP = P + 1, CV = Zh * P * PYP, NB = Zh * P * P;
    extern __shared__ float2 sm[];
    float2* tw = sm;
    float2* cubes = tw + P;  // NI x [Zh][P][PYP]
    fill_twiddles<P>(tw);
    const int img0 = blockIdx.x * NI;
    phase_img pds[NI];
#pragma unroll
    for (int j = 0; j < NI; ++j) pds[j] = a.phased ? phase_decode(a.ph, img0 + j) : phase_img{};
    __syncthreads();
    // z lines (R2C) of the valid (x, y) lines, read straight from HBM / L2
    const int nl1 = a.nx * a.ny;
    bool z_done = false;
    if constexpr (NI >= 4 && P >= 20) {
        // one CTA per SM (four 37 KB cubes): nothing else hides the loads of a
        // round, so the next round's dense line is fetched before this round's
        // transform (phase-major tensors: Q4 float4s per line, + the gate's)
        if (a.vec4) {
            constexpr int Q4 = (P + 3) / 4;
            float4 cur[Q4], curg[Q4];
            auto fetch = [&](int ln, float4 (&u)[Q4], float4 (&gt)[Q4]) {
                const int j = ln / nl1, l1 = ln - j * nl1;
                const int64_t base = int64_t(img0 + j) * a.img_stride + int64_t(l1) * a.nz;
                const float4* __restrict__ p4 = reinterpret_cast<const float4*>(a.src + base);
                const float4* __restrict__ g4 = a.gate ? reinterpret_cast<const float4*>(a.gate + base) : nullptr;
#pragma unroll
                for (int z4 = 0; z4 < Q4; ++z4) {
                    const bool in = 4 * z4 < a.nz;
                    u[z4] = in ? __ldg(p4 + z4) : make_float4(0.f, 0.f, 0.f, 0.f);
                    gt[z4] = (in && g4) ? __ldg(g4 + z4) : make_float4(1.f, 1.f, 1.f, 1.f);
                }
            };
            const int total = NI * nl1;
            if (int(threadIdx.x) < total) fetch(threadIdx.x, cur, curg);
            for (int ln = threadIdx.x; ln < total; ln += CT) {
                float4 nxt[Q4], nxtg[Q4];
                if (ln + CT < total) fetch(ln + CT, nxt, nxtg);
                const int j = ln / nl1, l1 = ln - j * nl1;
                const int x = l1 / a.ny, y = l1 - x * a.ny;
                float2 v[P];
#pragma unroll
                for (int z4 = 0; z4 < Q4; ++z4) {
                    const float4 u = cur[z4], gt = curg[z4];
                    if (4 * z4 < P) v[4 * z4] = make_float2(gt.x > 0.f ? u.x : 0.f, 0.f);
                    if (4 * z4 + 1 < P) v[4 * z4 + 1 < P ? 4 * z4 + 1 : 0] = make_float2(gt.y > 0.f ? u.y : 0.f, 0.f);
                    if (4 * z4 + 2 < P) v[4 * z4 + 2 < P ? 4 * z4 + 2 : 0] = make_float2(gt.z > 0.f ? u.z : 0.f, 0.f);
                    if (4 * z4 + 3 < P) v[4 * z4 + 3 < P ? 4 * z4 + 3 : 0] = make_float2(gt.w > 0.f ? u.w : 0.f, 0.f);
                }
                dft_r<P, P, false>(v, tw);
                float2* cube = cubes + j * CV;
#pragma unroll
                for (int k = 0; k < Zh; ++k) cube[(k * P + x) * PYP + y] = v[k];
#pragma unroll
                for (int z4 = 0; z4 < Q4; ++z4) cur[z4] = nxt[z4], curg[z4] = nxtg[z4];
            }
            z_done = true;
        }
    }
    if (!z_done)
    for (int ln = threadIdx.x; ln < NI * nl1; ln += CT) {
        const int j = NI == 1 ? 0 : ln / nl1, l1 = ln - j * nl1;
        const int x = l1 / a.ny, y = l1 - x * a.ny;
        float2 v[P];
        int64_t base;
        int z0 = 0, zs = 1, zlim = a.nz;
        if (a.phased) {
            phase_img pd = pds[0];
#pragma unroll
            for (int jj = 1; jj < NI; ++jj)
                if (jj == j) pd = pds[jj];
            base = phase_line(a.ph, pd, x, y);
            z0 = pd.rz, zs = a.ph.sz, zlim = base >= 0 ? a.ph.nz : 0;
        } else {
            base = int64_t(img0 + j) * a.img_stride + int64_t(l1) * a.nz;
        }
        if (a.vec4) {  // dense images (phase-major tensors): a line is nz / 4 aligned float4s
            const float4* __restrict__ p4 = reinterpret_cast<const float4*>(a.src + base);
            const float4* __restrict__ g4 = a.gate ? reinterpret_cast<const float4*>(a.gate + base) : nullptr;
#pragma unroll
            for (int z4 = 0; z4 < (P + 3) / 4; ++z4) {
                float4 u = make_float4(0.f, 0.f, 0.f, 0.f);
                if (4 * z4 < a.nz) {
                    u = __ldg(p4 + z4);
                    if (g4) {
                        const float4 gt = __ldg(g4 + z4);
                        u.x = gt.x > 0.f ? u.x : 0.f, u.y = gt.y > 0.f ? u.y : 0.f;
                        u.z = gt.z > 0.f ? u.z : 0.f, u.w = gt.w > 0.f ? u.w : 0.f;
                    }
                }
                if (4 * z4 < P) v[4 * z4] = make_float2(u.x, 0.f);
                if (4 * z4 + 1 < P) v[4 * z4 + 1 < P ? 4 * z4 + 1 : 0] = make_float2(u.y, 0.f);
                if (4 * z4 + 2 < P) v[4 * z4 + 2 < P ? 4 * z4 + 2 : 0] = make_float2(u.z, 0.f);
                if (4 * z4 + 3 < P) v[4 * z4 + 3 < P ? 4 * z4 + 3 : 0] = make_float2(u.w, 0.f);
            }
        } else {
#pragma unroll
            for (int z = 0; z < P; ++z) {
                float val = 0.f;
                const int zz = z0 + zs * z;
                if (z < a.nz && zz < zlim) {
                    val = __ldg(a.src + base + zz);
                    if (a.gate && !(__ldg(a.gate + base + zz) > 0.f)) val = 0.f;
                }
                v[z] = make_float2(val, 0.f);
            }
        }
        dft_r<P, P, false>(v, tw);
        float2* cube = cubes + j * CV;
#pragma unroll
        for (int k = 0; k < Zh; ++k) cube[(k * P + x) * PYP + y] = v[k];
    }
    __syncthreads();
    // y lines of the valid rows x < nx (columns y >= ny are the zero padding)
    for (int ln = threadIdx.x; ln < NI * Zh * a.nx; ln += CT) {
        const int j = NI == 1 ? 0 : ln / (Zh * a.nx), l2 = ln - j * (Zh * a.nx);
        const int zb = l2 / a.nx, x = l2 - zb * a.nx;
        float2* row = cubes + j * CV + (zb * P + x) * PYP;
        float2 v[P];
#pragma unroll
        for (int y = 0; y < P; ++y) v[y] = y < a.ny ? row[y] : make_float2(0.f, 0.f);
        dft_r<P, P, false>(v, tw);
#pragma unroll
        for (int k = 0; k < P; ++k) row[k] = v[k];
    }
    __syncthreads();
    // x lines of every column (rows x >= nx are the zero padding)
    for (int ln = threadIdx.x; ln < NI * Zh * P; ln += CT) {
        const int j = NI == 1 ? 0 : ln / (Zh * P), l3 = ln - j * (Zh * P);
        const int zb = l3 / P, y = l3 - zb * P;
        float2* col = cubes + j * CV + zb * P * PYP + y;
        float2 v[P];
#pragma unroll
        for (int x = 0; x < P; ++x) v[x] = x < a.nx ? col[x * PYP] : make_float2(0.f, 0.f);
        dft_r<P, P, false>(v, tw);
#pragma unroll
        for (int k = 0; k < P; ++k) col[k * PYP] = v[k];
    }
    __syncthreads();
    if constexpr (!GL) {
        float4* g4 = reinterpret_cast<float4*>(spec + int64_t(img0) * NB);
        for (int idx = threadIdx.x; idx < NB / 2; idx += CT) {
            const int e = 2 * idx, zb = e / (P * P), r = e - zb * (P * P), x = r / P, y = r - x * P;
            const float2 u = cubes[(zb * P + x) * PYP + y], w = cubes[(zb * P + x) * PYP + y + 1];
            __stcs(g4 + idx, make_float4(u.x, u.y, w.x, w.y));
        }
    } else {  // row-bin-major layout: one NI * 8-byte piece per bin
        const int F = a.gF;
        float2* dst = spec + (int64_t(img0 / F) * NB) * F + (img0 % F);
        if constexpr (NI == 4) {
            // a lane pair stores a bin's 32-byte piece as the two 16-byte halves of one sector
            for (int b2 = threadIdx.x; b2 < 2 * NB; b2 += CT) {
                const int b = b2 >> 1, h = b2 & 1;
                const int zb = b / (P * P), r = b - zb * (P * P), x = r / P, y = r - x * P;
                const int off = (zb * P + x) * PYP + y;
                const float2 u = cubes[(2 * h) * CV + off], w = cubes[(2 * h + 1) * CV + off];
                __stcs(reinterpret_cast<float4*>(dst + int64_t(b) * F + 2 * h), make_float4(u.x, u.y, w.x, w.y));
            }
        } else
        for (int b = threadIdx.x; b < NB; b += CT) {
            const int zb = b / (P * P), r = b - zb * (P * P), x = r / P, y = r - x * P;
            float2 v[NI];
#pragma unroll
            for (int j = 0; j < NI; ++j) v[j] = cubes[j * CV + (zb * P + x) * PYP + y];
            grp_put<NI>(dst + int64_t(b) * F, v);
        }
    }
}

template <int P, int NI, bool UNIT, bool GL = (NI > 1)>
__global__ void __launch_bounds__(cube_threads<NI>()) fft3_inv_reg_k(const float2* __restrict__ spec, cube_io a,
                                                           const float* __restrict__ bias) {
    constexpr int CT = cube_threads<NI>();
    constexpr int Zh = P / 2 + 1, PYP = P + 1, CV = Zh * P * PYP, NB = Zh * P * P;
    extern __shared__ float2 sm[];
    float2* tw = sm;
    float2* cubes = tw + P;
    fill_twiddles<P>(tw);
    const int img0 = blockIdx.x * NI;
    if constexpr (!GL) {
        const float4* g4 = reinterpret_cast<const float4*>(spec + int64_t(img0) * NB);
        constexpr int NV = NB / 2;
        for (int i0 = threadIdx.x; i0 < NV; i0 += 4 * CT) {
            float4 u4[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i0 + u * CT < NV) u4[u] = __ldcs(g4 + i0 + u * CT);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int idx = i0 + u * CT;
                if (idx < NV) {
                    const int e = 2 * idx, zb = e / (P * P), r = e - zb * (P * P), x = r / P, y = r - x * P;
                    cubes[(zb * P + x) * PYP + y] = make_float2(u4[u].x, u4[u].y);
                    cubes[(zb * P + x) * PYP + y + 1] = make_float2(u4[u].z, u4[u].w);
                }
            }
        }
    } else {
        const int F = a.gF;
        const float2* src = spec + (int64_t(img0 / F) * NB) * F + (img0 % F);
        for (int b0 = threadIdx.x; b0 < NB; b0 += 2 * CT) {  // two bins' loads in flight per thread
            float2 v0[NI], v1[NI];
            const int b1 = b0 + CT;
            grp_get<NI>(src + int64_t(b0) * F, v0);
            if (b1 < NB) grp_get<NI>(src + int64_t(b1) * F, v1);
            {
                const int zb = b0 / (P * P), r = b0 - zb * (P * P), x = r / P, y = r - x * P;
#pragma unroll
                for (int j = 0; j < NI; ++j) cubes[j * CV + (zb * P + x) * PYP + y] = v0[j];
            }
            if (b1 < NB) {
                const int zb = b1 / (P * P), r = b1 - zb * (P * P), x = r / P, y = r - x * P;
#pragma unroll
                for (int j = 0; j < NI; ++j) cubes[j * CV + (zb * P + x) * PYP + y] = v1[j];
            }
        }
    }
    phase_img pds[NI];
#pragma unroll
    for (int j = 0; j < NI; ++j) pds[j] = a.phased ? phase_decode(a.ph, img0 + j) : phase_img{};
    __syncthreads();
    // x lines (columns), keep rows xs * i, i < xc
    for (int ln = threadIdx.x; ln < NI * Zh * P; ln += CT) {
        const int j = NI == 1 ? 0 : ln / (Zh * P), l1 = ln - j * (Zh * P);
        const int zb = l1 / P, y = l1 - zb * P;
        float2* col = cubes + j * CV + zb * P * PYP + y;
        float2 v[P];
#pragma unroll
        for (int x = 0; x < P; ++x) v[x] = col[x * PYP];
        dft_r<P, P, true>(v, tw);
        if (UNIT) {
#pragma unroll
            for (int i = 0; i < P; ++i)
                if (i < a.xc) col[i * PYP] = v[i];
        } else {
            for (int i = 0; i < a.xc; ++i) col[i * PYP] = v[i * a.xs];  // dynamic index: local memory
        }
    }
    __syncthreads();
    // y lines of the kept rows, keep columns ys * j, j < yc
    for (int ln = threadIdx.x; ln < NI * Zh * a.xc; ln += CT) {
        const int j = NI == 1 ? 0 : ln / (Zh * a.xc), l2 = ln - j * (Zh * a.xc);
        const int zb = l2 / a.xc, i = l2 - zb * a.xc;
        float2* row = cubes + j * CV + (zb * P + i) * PYP;
        float2 v[P];
#pragma unroll
        for (int y = 0; y < P; ++y) v[y] = row[y];
        dft_r<P, P, true>(v, tw);
        if (UNIT) {
#pragma unroll
            for (int jj = 0; jj < P; ++jj)
                if (jj < a.yc) row[jj] = v[jj];
        } else {
            for (int jj = 0; jj < a.yc; ++jj) row[jj] = v[jj * a.ys];
        }
    }
    __syncthreads();
    // z lines (C2R) of the kept (i, j), keep zs * q, q < zc; scale, bias, transfer
    const int nl3 = a.xc * a.yc;
    for (int ln = threadIdx.x; ln < NI * nl3; ln += CT) {
        const int j = NI == 1 ? 0 : ln / nl3, l3 = ln - j * nl3;
        const int i = l3 / a.yc, jj = l3 - i * a.yc;
        const int img = img0 + j;
        const float2* cube = cubes + j * CV;
        float2 v[P];
#pragma unroll
        for (int z = 0; z < P; ++z) {
            if (z < Zh) {
                v[z] = cube[(z * P + i) * PYP + jj];
            } else {  // Hermitian symmetry of a real signal
                const float2 c = cube[((P - z) * P + i) * PYP + jj];
                v[z] = make_float2(c.x, -c.y);
            }
        }
        dft_r<P, P, true>(v, tw);
        const float bv = bias ? bias[img % a.bias_mod] : 0.f;
        int64_t base;
        int z0 = 0, zst = 1, zlim = 1 << 30;
        if (a.phased) {
            phase_img pd = pds[0];
#pragma unroll
            for (int q = 1; q < NI; ++q)
                if (q == j) pd = pds[q];
            base = phase_line(a.ph, pd, i, jj);
            z0 = pd.rz, zst = a.ph.sz, zlim = a.ph.nz;
        } else {
            base = int64_t(img) * a.img_stride + (int64_t(i) * a.oy + jj) * a.oz;
        }
        if (base < 0) continue;
        if constexpr (UNIT) {
            if (a.vec4) {  // dense output lines of zc / 4 aligned float4s (phase-major tensors)
                auto fin = [&](float x) {
                    float r = x * a.scale + bv;
                    if (a.act == 2) r = r > 0.f ? r : 0.f;
                    else if (a.act == 0) r = 1.f / (1.f + expf(-r));
                    else if (a.act == 1) r = tanhf(r);
                    return r;
                };
                float4* __restrict__ d4 = reinterpret_cast<float4*>(a.dst + base);
#pragma unroll
                for (int q4 = 0; q4 < P / 4; ++q4)
                    if (4 * q4 < a.zc)
                        d4[q4] = make_float4(fin(v[4 * q4].x), fin(v[4 * q4 + 1].x), fin(v[4 * q4 + 2].x),
                                             fin(v[4 * q4 + 3].x));
                continue;
            }
        }
#pragma unroll
        for (int q = 0; q < P; ++q) {
            const int k = UNIT ? q : q * a.zs;
            if (q < a.zc && k < P && z0 + zst * q < zlim) {
                float r = v[UNIT ? q : 0].x;
                if (!UNIT) {  // rare (dense-kernel dK inverse): pick v[k] without dynamic register indexing
#pragma unroll
                    for (int kk = 0; kk < P; ++kk)
                        if (kk == k) r = v[kk].x;
                }
                r = r * a.scale + bv;
                if (a.act == 2) r = r > 0.f ? r : 0.f;
                else if (a.act == 0) r = 1.f / (1.f + expf(-r));
                else if (a.act == 1) r = tanhf(r);
                a.dst[base + z0 + zst * q] = r;
            }
        }
    }
}

// ---- row-bin-major xy passes (tensor-core plans, square planes): one CTA
// takes the z-bin plane of 4 consecutive maps of one row (item = (row, zb,
// part)); per bin the four maps are one 32-byte piece of the spectrum.
// Register variants: one line per thread, the P-point transform in registers,
// no exchange buffer; XP_T threads take the 4 planes' rows, then their
// columns, one pass each.
// The planes sit in shared memory as two PAIRS ([P][P + 1] bins of two
// adjacent float2: maps 2 h, 2 h + 1), so a lane pair moves a bin's 32-byte
// piece as two 16-byte halves of one sector (cp.async in, float4 out): with
// four separate planes every 8-byte copy was its own shared-memory wavefront
// and its own sector request (the pass ran at 84% of the L1 pipe). Lines are
// taken by lanes (map of the pair fastest, then the line), which keeps the
// line passes free of bank conflicts at the 16-byte bin pitch; the second
// pair is offset by 64 B so the two 16-byte slots of one bin fall in
// different bank groups.
// exact floor(n / d) for 0 <= n < 2^15, 0 < d < 2^13 (inv = 1 / d): the loops
// below index by runtime plane dims, and a 32-bit division is ~25 instructions
__device__ __forceinline__ int fdiv_small(int n, float inv) { return int((float(n) + 0.5f) * inv); }

constexpr int XP_NI = 4;
template <int P>
__host__ __device__ constexpr int xp_threads() { return (4 * P + 31) / 32 * 32 < 256 ? (4 * P + 31) / 32 * 32 : 256; }
template <int P>
__host__ __device__ constexpr int xp_pair() { return P * (P + 1) * 2 + 8; }  // float2 per plane pair
template <int P>
__host__ __device__ constexpr int xp_tw() { return (P + 1) & ~1; }            // twiddles, 16-byte multiple
template <int P>
constexpr size_t smem_xy_pair() { return sizeof(float2) * (size_t(xp_tw<P>()) + 2 * size_t(xp_pair<P>())); }

template <int P>
__global__ void __launch_bounds__(xp_threads<P>()) fft_xy_fwd_pair_k(float2* __restrict__ spec, int nx, int ny, int Zh,
                                                             int F) {
    constexpr int XT = xp_threads<P>();
    constexpr int PYP = P + 1, PP = xp_pair<P>();
    const int H = F / XP_NI;
    extern __shared__ __align__(16) float2 sm[];
    float2* tw = sm;
    float2* pls = sm + xp_tw<P>();  // 2 x [P][PYP][2]
    const int64_t q = blockIdx.x;
    const int part = int(q % H);
    const int64_t rest = q / H;
    const int zb = int(rest % Zh);
    float2* gq = spec + ((rest / Zh) * Zh * P * P + int64_t(zb) * P * P) * F + part * XP_NI;
    fill_twiddles<P>(tw);
    // the valid region the z pass wrote: 16-byte async copies, every load of the CTA in flight at once
    const float inv_ny = 1.f / float(ny);
    for (int e2 = threadIdx.x; e2 < 2 * nx * ny; e2 += XT) {
        const int e = e2 >> 1, h = e2 & 1;
        const int x = fdiv_small(e, inv_ny), y = e - x * ny;
        cp_async16p(pls + h * PP + (x * PYP + y) * 2, gq + (x * P + y) * F + 2 * h);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    for (int ln = threadIdx.x; ln < 4 * nx; ln += XT) {  // rows (y transforms) of the valid rows
        const int jj = ln & 1, r = ln >> 1, h = r >= nx ? 1 : 0, x = r - h * nx;
        float2* row = pls + h * PP + x * PYP * 2 + jj;
        float2 v[P];
#pragma unroll
        for (int y = 0; y < P; ++y) v[y] = y < ny ? row[2 * y] : make_float2(0.f, 0.f);
        dft_r<P, P, false>(v, tw);
#pragma unroll
        for (int k = 0; k < P; ++k) row[2 * k] = v[k];
    }
    __syncthreads();
    for (int ln = threadIdx.x; ln < 4 * P; ln += XT) {  // columns (x transforms); rows >= nx are zero
        const int jj = ln & 1, r = ln >> 1, h = r / P, y = r - h * P;
        float2* col = pls + h * PP + y * 2 + jj;
        float2 v[P];
#pragma unroll
        for (int x = 0; x < P; ++x) v[x] = x < nx ? col[x * PYP * 2] : make_float2(0.f, 0.f);
        dft_r<P, P, false>(v, tw);
#pragma unroll
        for (int k = 0; k < P; ++k) col[k * PYP * 2] = v[k];
    }
    __syncthreads();
    for (int e2 = threadIdx.x; e2 < 2 * P * P; e2 += XT) {  // a lane pair stores a bin's 32-byte piece
        const int e = e2 >> 1, h = e2 & 1;
        const int x = e / P, y = e - x * P;
        const float4 u = *reinterpret_cast<const float4*>(pls + h * PP + (x * PYP + y) * 2);
        __stcs(reinterpret_cast<float4*>(gq + e * F + 2 * h), u);
    }
}

template <int P, bool UNIT>  // UNIT: unit kept-voxel steps (no per-output division)
__global__ void __launch_bounds__(xp_threads<P>()) fft_xy_inv_pair_k(const float2* __restrict__ spec, float2* __restrict__ out,
                                                             int x_step, int xc, int y_step, int yc, int Zh, int F) {
    constexpr int XT = xp_threads<P>();
    constexpr int PYP = P + 1, PP = xp_pair<P>();
    const int H = F / XP_NI;
    extern __shared__ __align__(16) float2 sm[];
    float2* tw = sm;
    float2* pls = sm + xp_tw<P>();
    const int64_t q = blockIdx.x;
    const int part = int(q % H);
    const int64_t rest = q / H;
    const int zb = int(rest % Zh);
    const int64_t grp = rest / Zh;
    const float2* gq = spec + (grp * Zh * P * P + int64_t(zb) * P * P) * F + part * XP_NI;
    fill_twiddles<P>(tw);
    for (int e2 = threadIdx.x; e2 < 2 * P * P; e2 += XT) {  // 16-byte async copies, all in flight
        const int e = e2 >> 1, h = e2 & 1;
        const int x = e / P, y = e - x * P;
        cp_async16p(pls + h * PP + (x * PYP + y) * 2, gq + e * F + 2 * h);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    for (int ln = threadIdx.x; ln < 4 * P; ln += XT) {  // column inverses, keep rows x_step * i
        const int jj = ln & 1, r = ln >> 1, h = r / P, y = r - h * P;
        float2* col = pls + h * PP + y * 2 + jj;
        float2 v[P];
#pragma unroll
        for (int x = 0; x < P; ++x) v[x] = col[x * PYP * 2];
        dft_r<P, P, true>(v, tw);
        if constexpr (UNIT) {
#pragma unroll
            for (int i = 0; i < P; ++i)
                if (i < xc) col[i * PYP * 2] = v[i];
        } else {
#pragma unroll
            for (int k = 0; k < P; ++k) {
                const int i = k / x_step;
                if (i * x_step == k && i < xc) col[i * PYP * 2] = v[k];
            }
        }
    }
    __syncthreads();
    for (int ln = threadIdx.x; ln < 4 * xc; ln += XT) {  // row inverses of the kept rows
        const int jj = ln & 1, r = ln >> 1, h = r >= xc ? 1 : 0, i = r - h * xc;
        float2* row = pls + h * PP + i * PYP * 2 + jj;
        float2 v[P];
#pragma unroll
        for (int y = 0; y < P; ++y) v[y] = row[2 * y];
        dft_r<P, P, true>(v, tw);
        if constexpr (UNIT) {  // the kept columns back into the row (already in registers)
#pragma unroll
            for (int c = 0; c < P; ++c)
                if (c < yc) row[2 * c] = v[c];
        } else {
#pragma unroll
            for (int k = 0; k < P; ++k) {
                const int c = k / y_step;
                if (c * y_step == k && c < yc) row[2 * c] = v[k];
            }
        }
    }
    __syncthreads();
    // coalesced stores of the 4 compact blocks (plane img * Zh + zb, [xc][yc]): even / odd lanes
    // take the two maps of a pair (adjacent float2 in shared memory, 128-byte runs per map)
    const int blk = xc * yc;
    const float inv_yc = 1.f / float(yc);
    for (int e = threadIdx.x; e < 4 * blk; e += XT) {
        const int h = e >= 2 * blk ? 1 : 0, rem = e - h * 2 * blk, r = rem >> 1, jj = rem & 1;
        const int i = fdiv_small(r, inv_yc), c = r - i * yc;
        out[((grp * F + part * XP_NI + 2 * h + jj) * Zh + zb) * int64_t(blk) + r] =
            pls[h * PP + (i * PYP + c) * 2 + jj];
    }
}


struct zinv_args {
    int xc, yc;                        // kept block per z-bin plane (compact input)
    int z_step, z_cnt;                 // kept z voxels (selection starts at 0)
    int64_t nlines;                    // images * xc * yc
    float scale;
    int64_t out_img_stride;
    int oy, oz;                        // output box dims (y, z)
    int act;                           // ZNN_ACT_* (3 = none)
    int bias_mod;                      // bias index = img % bias_mod
    int phased;                        // outputs are the phases of an original tensor (ph)
    phase_geom ph;
};

// ---- z pass, inverse (C2R) of the compact kept lines, crop / tap selection
// and fused epilogue ----
template <int P>
__global__ void __launch_bounds__(THREADS) fft_z_inv_k(const float2* __restrict__ cspec, zinv_args g,
                                                        const float* __restrict__ bias, float* __restrict__ out) {
    constexpr int Zh = P / 2 + 1;
    constexpr int R1 = line_shape<P>::R1, R2 = line_shape<P>::R2;
    extern __shared__ float2 sm[];
    __shared__ int64_t ibase[LINES], obase[LINES];
    __shared__ float bvals[LINES];
    __shared__ int ozoff[LINES];
    float2* tw = sm;
    float2* xbuf = tw + P;
    float2* stash = xbuf + LINES * line_shape<P>::XP;  // LINES x (Zh + 1)
    fill_twiddles<P>(tw);
    const int l = threadIdx.x / TPL, t = threadIdx.x % TPL;
    const int64_t line = int64_t(blockIdx.x) * LINES + l;
    const bool ok = line < g.nlines;
    if (ok && t == 0) {  // 32-bit decode (nlines < 2^32, checked on the host)
        const uint32_t per = uint32_t(g.xc) * uint32_t(g.yc);
        uint32_t im, rr;
        if (g.phased) {
            im = phase_pair_line(g.ph, uint32_t(line), per, &rr);
        } else {
            im = uint32_t(line) / per;
            rr = uint32_t(line) - im * per;
        }
        const int r = int(rr);
        const int xi = r / g.yc, yi = r - (r / g.yc) * g.yc;
        ibase[l] = int64_t(im) * Zh * per + r;
        if (g.phased) {  // write the phase's voxels of the original tensor in place
            const phase_img pd = phase_decode(g.ph, int(im));
            obase[l] = phase_line(g.ph, pd, xi, yi);
            ozoff[l] = pd.rz;
        } else {
            obase[l] = int64_t(im) * g.out_img_stride + (int64_t(xi) * g.oy + yi) * g.oz;
            ozoff[l] = 0;
        }
        bvals[l] = bias ? bias[im % uint32_t(g.bias_mod)] : 0.f;
    }
    __syncthreads();
    // coalesced gather: a warp reads one z-bin of 32 consecutive lines; all of
    // a thread's loads are issued before any is stored (the pass was bound by
    // load latency: one load in flight per thread at a time)
    const int64_t zstride = int64_t(g.xc) * g.yc;
    {
        constexpr int NE = (LINES * Zh + THREADS - 1) / THREADS;
        const int64_t lines_left = g.nlines - int64_t(blockIdx.x) * LINES;
        float2 tmp[NE];
#pragma unroll
        for (int e = 0; e < NE; ++e) {
            const int idx = threadIdx.x + e * THREADS;
            const int l2 = idx % LINES, zb = idx / LINES;
            tmp[e] = (idx < LINES * Zh && l2 < lines_left) ? __ldcs(cspec + ibase[l2] + zb * zstride)
                                                          : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int e = 0; e < NE; ++e) {
            const int idx = threadIdx.x + e * THREADS;
            if (idx < LINES * Zh) stash[(idx % LINES) * (Zh + 1) + idx / LINES] = tmp[e];
        }
    }
    __syncthreads();
    const float2* st = stash + l * (Zh + 1);
    float2 v[R2];
#pragma unroll
    for (int n2 = 0; n2 < R2; ++n2) {
        const int j = t + R1 * n2;
        float2 val = make_float2(0.f, 0.f);
        if (ok && t < R1) {
            if (j < Zh) {
                val = st[j];
            } else {  // Hermitian symmetry of a real signal
                const float2 c = st[P - j];
                val = make_float2(c.x, -c.y);
            }
        }
        v[n2] = val;
    }
    const bool wok = ok && obase[l] >= 0;  // phased: ragged phase lines outside the tensor
    float* dst = out + (wok ? obase[l] + ozoff[l] : 0);
    const int zst = g.phased ? g.ph.sz : 1;
    const int zlim = g.phased ? g.ph.nz - (wok ? ozoff[l] : 0) : 1 << 30;
    const float bv = ok ? bvals[l] : 0.f;
    line_fft<P, true>(v, xbuf + l * line_shape<P>::XP, tw, t, [&](int k, float2 val) {
        const int q = k / g.z_step;
        if (wok && q * g.z_step == k && q < g.z_cnt && zst * q < zlim) {
            float r = val.x * g.scale + bv;
            if (g.act == 2) r = r > 0.f ? r : 0.f;
            else if (g.act == 0) r = 1.f / (1.f + expf(-r));
            else if (g.act == 1) r = tanhf(r);
            dst[zst * q] = r;
        }
    });
}

// ---- z passes with one line PAIR per thread (pads 40..64): two real lines
// are the real and imaginary parts of one complex P-point FFT held in
// registers (Hermitian split / merge), so there is no exchange buffer, no
// warp sync and half the arithmetic of a complex transform per real line.
// A warp owns 64 consecutive lines (lane l: lines l and l + 32); the global
// side goes through a per-warp staging tile so loads and stores are
// warp-cooperative along z (the per-thread lines are far apart in memory). ----
constexpr int ZR_THREADS = 128;
constexpr int ZR_LINES = 2 * ZR_THREADS;
__host__ __device__ constexpr int zr_pitch(int P) { return (P % 2) ? P : P + 1; }  // odd: conflict-free rows
template <int P>
constexpr size_t zr_smem(bool gated = false) { return sizeof(float) * size_t(ZR_LINES) * size_t(zr_pitch(P)) * (gated ? 2 : 1); }

template <int P>
__global__ void __launch_bounds__(ZR_THREADS) fft_z_fwd_reg_k(const float* __restrict__ in, int64_t in_img_stride,
                                                              int nx, int ny, int nz, int64_t nlines,
                                                              float2* __restrict__ spec, int Px, int Py,
                                                              const float* __restrict__ gate, phase_geom ph,
                                                              int phased, int gF) {
    constexpr int Zh = P / 2 + 1, SP = zr_pitch(P);
    __shared__ float2 tw[P];
    __shared__ int64_t obase[ZR_LINES];
    extern __shared__ float stage[];  // [ZR_LINES][SP]
    fill_twiddles<P>(tw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t wl0 = int64_t(blockIdx.x) * ZR_LINES + warp * 64;  // this warp's first line
    float* wst = stage + warp * 64 * SP;
    const uint32_t pl = uint32_t(nx) * uint32_t(ny);
    // pair2 (sparsity 2 along z, row-bin-major line order): lines 2 t, 2 t + 1
    // are the two z-phases of one original line, so thread t takes that pair:
    // its complex input is the original line read as float2s, staged by plain
    // contiguous 8-byte copies (a third of the staging instructions of the
    // per-phase 4-byte copies, which were most of this kernel's issue slots)
    const bool pair2 = phased && gF && ph.sz == 2 && !(ph.nz & 1) && !(nz > ph.nz / 2) &&
                       ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(gate)) & 7) == 0;
    // each lane decodes its two lines (lane, lane + 32; pair2: 2 lane, 2 lane + 1):
    // source offset (-1: none), first z, z stride and z limit
    int64_t soff[2];
    int sz0[2], szs[2], szl[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int l = pair2 ? 2 * lane + h : lane + 32 * h;
        const int64_t line = wl0 + l;
        soff[h] = -1, sz0[h] = 0, szs[h] = 1, szl[h] = 0;
        int64_t ob = -1;
        if (line < nlines) {  // 32-bit decode, as fft_z_fwd_k
            uint32_t im, rr;
            if (phased) {
                im = gF ? phase_rbm_line(ph, uint32_t(line), pl, &rr) : phase_pair_line(ph, uint32_t(line), pl, &rr);
            } else if (gF) {
                im = rbm_line(uint32_t(line), pl, uint32_t(gF), &rr);
            } else {
                im = uint32_t(line) / pl;
                rr = uint32_t(line) - im * pl;
            }
            const int r = int(rr), x = r / ny, y = r - (r / ny) * ny;
            soff[h] = int64_t(im) * in_img_stride + (int64_t(x) * ny + y) * nz;
            szl[h] = nz;
            if (phased) {
                const phase_img pd = phase_decode(ph, int(im));
                soff[h] = phase_line(ph, pd, x, y);
                sz0[h] = pd.rz, szs[h] = ph.sz, szl[h] = soff[h] >= 0 ? ph.nz : 0;
            }
            ob = spec_at(gF, im, int64_t(Zh) * Px * Py, int64_t(x) * Py + y);
        }
        obase[warp * 64 + l] = ob;
    }
    // warp-cooperative async copies into the staging tile (lanes along z, zero
    // fill past the line), every line of the warp in flight at once; line l's
    // parameters come from lane l % 32. With a gate the gate values go to a
    // second tile.
    constexpr int NJ = (P + 31) / 32;
    float* gst = gate ? stage + ZR_LINES * SP : nullptr;
    if (pair2) {
        float2* wst2 = reinterpret_cast<float2*>(wst);                                  // [32 original lines][SP]
        float2* gst2 = gate ? reinterpret_cast<float2*>(gst + warp * 64 * SP) : nullptr;
        for (int l = 0; l < 32; ++l) {
            const int64_t off = __shfl_sync(0xffffffffu, soff[0], l);
#pragma unroll
            for (int jj = 0; jj < NJ; ++jj) {
                const int j = jj * 32 + lane;
                if (j < P) {
                    const bool ok = off >= 0 && j < nz;
                    const int64_t e = ok ? off + 2 * j : 0;
                    cp_async8z(wst2 + l * SP + j, in + e, ok);
                    if (gate) cp_async8z(gst2 + l * SP + j, gate + e, ok);
                }
            }
        }
    } else
    for (int l = 0; l < 64; ++l) {
        const int src = l & 31;
        const bool hi = l >= 32;  // (uniform)
        const int64_t off = __shfl_sync(0xffffffffu, hi ? soff[1] : soff[0], src);
        const int z0 = __shfl_sync(0xffffffffu, hi ? sz0[1] : sz0[0], src);
        const int zs = __shfl_sync(0xffffffffu, hi ? szs[1] : szs[0], src);
        const int zl = __shfl_sync(0xffffffffu, hi ? szl[1] : szl[0], src);
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj) {
            const int j = jj * 32 + lane, z = z0 + zs * j;
            if (j < P) {
                const bool ok = off >= 0 && j < nz && z < zl;
                const int64_t e = ok ? off + z : 0;
                cp_async4z(wst + l * SP + j, in + e, ok);
                if (gate) cp_async4z(gst + (warp * 64 + l) * SP + j, gate + e, ok);
            }
        }
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();  // twiddles, obase
    float2 v[P];
    if (pair2) {
        const float2* a2 = reinterpret_cast<const float2*>(wst) + lane * SP;
        if (gate) {
            const float2* g2 = reinterpret_cast<const float2*>(gst + warp * 64 * SP) + lane * SP;
#pragma unroll
            for (int j = 0; j < P; ++j) {
                const float2 av = a2[j], gv = g2[j];
                v[j] = make_float2(gv.x > 0.f ? av.x : 0.f, gv.y > 0.f ? av.y : 0.f);
            }
        } else {
#pragma unroll
            for (int j = 0; j < P; ++j) v[j] = a2[j];
        }
    } else {
        const float* a = wst + lane * SP;
        const float* b = wst + (lane + 32) * SP;
        if (gate) {  // fused ReLU backward: g * (y > 0) (transfer.hpp:99-106, ReLU'(0) = 0)
            const float* ga = gst + (warp * 64 + lane) * SP;
            const float* gb = ga + 32 * SP;
#pragma unroll
            for (int j = 0; j < P; ++j) v[j] = make_float2(ga[j] > 0.f ? a[j] : 0.f, gb[j] > 0.f ? b[j] : 0.f);
        } else {
#pragma unroll
            for (int j = 0; j < P; ++j) v[j] = make_float2(a[j], b[j]);
        }
    }
    dft_r<P, P, false>(v, tw);
    // split: X1[k] = (Z[k] + conj Z[P-k]) / 2, X2[k] = (Z[k] - conj Z[P-k]) / (2 i)
    const int64_t o1 = obase[warp * 64 + (pair2 ? 2 * lane : lane)],
                  o2 = obase[warp * 64 + (pair2 ? 2 * lane + 1 : lane + 32)];
    const int64_t zstride = int64_t(Px) * Py * (gF ? gF : 1);
#pragma unroll
    for (int k = 0; k < Zh; ++k) {
        const float2 zk = v[k], zm = v[(P - k) % P];
        const float2 x1 = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y));
        const float2 x2 = make_float2(0.5f * (zk.y + zm.y), 0.5f * (zm.x - zk.x));
        if (o1 >= 0) spec[o1 + k * zstride] = x1;
        if (o2 >= 0) spec[o2 + k * zstride] = x2;
    }
}

// inverse (C2R) of the compact kept planes, line pairs per thread as above;
// the P outputs go through the staging tile, so any crop / tap stride is a
// shared-memory index and the stores are warp-cooperative along z
template <int P>
__global__ void __launch_bounds__(ZR_THREADS) fft_z_inv_reg_k(const float2* __restrict__ cspec, zinv_args g,
                                                              const float* __restrict__ bias, float* __restrict__ out) {
    constexpr int Zh = P / 2 + 1, SP = zr_pitch(P);
    __shared__ float2 tw[P];
    __shared__ float bvals[ZR_LINES];
    extern __shared__ float stage[];
    fill_twiddles<P>(tw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t wl0 = int64_t(blockIdx.x) * ZR_LINES + warp * 64;
    const uint32_t per = uint32_t(g.xc) * uint32_t(g.yc);
    const int64_t zstride = int64_t(g.xc) * g.yc;
    // pair2 (sparsity 2 along z): lines 2 t, 2 t + 1 are the two z-phases of one
    // original line; thread t takes that pair, its two real outputs per z are
    // adjacent voxels of the original line, staged as float2s and stored by
    // contiguous 8-byte stores (see fft_z_fwd_reg_k)
    const bool pair2 = g.phased && g.ph.sz == 2 && !(g.ph.nz & 1) && g.z_step == 1 && 2 * g.z_cnt <= g.ph.nz &&
                       (reinterpret_cast<uintptr_t>(out) & 7) == 0;
    int64_t ib[2], obh[2];
    int ozh[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // decode this thread's two lines
        const int l = pair2 ? 2 * lane + h : lane + 32 * h;
        const int64_t line = wl0 + l;
        ib[h] = -1;
        int64_t ob = -1;
        int oz = 0;
        float bv = 0.f;
        if (line < g.nlines) {
            uint32_t im, rr;
            if (g.phased) {
                im = phase_pair_line(g.ph, uint32_t(line), per, &rr);
            } else {
                im = uint32_t(line) / per;
                rr = uint32_t(line) - im * per;
            }
            const int r = int(rr), xi = r / g.yc, yi = r - (r / g.yc) * g.yc;
            ib[h] = int64_t(im) * Zh * per + r;
            if (g.phased) {
                const phase_img pd = phase_decode(g.ph, int(im));
                ob = phase_line(g.ph, pd, xi, yi);
                oz = pd.rz;
            } else {
                ob = int64_t(im) * g.out_img_stride + (int64_t(xi) * g.oy + yi) * g.oz;
            }
            bv = bias ? bias[im % uint32_t(g.bias_mod)] : 0.f;
        }
        obh[h] = ob, ozh[h] = oz;
        bvals[warp * 64 + l] = bv;
    }
    float2 v[P];
#pragma unroll
    for (int k = 0; k < Zh; ++k) {  // Z = X1 + i X2 (and its Hermitian extension)
        const float2 a = ib[0] >= 0 ? __ldcs(cspec + ib[0] + k * zstride) : make_float2(0.f, 0.f);
        const float2 b = ib[1] >= 0 ? __ldcs(cspec + ib[1] + k * zstride) : make_float2(0.f, 0.f);
        v[k] = make_float2(a.x - b.y, a.y + b.x);
        if (k > 0 && k < P - k) v[P - k] = make_float2(a.x + b.y, b.x - a.y);
    }
    dft_r<P, P, true>(v, tw);
    __syncthreads();  // twiddles read; per-line tables ready
    float* wst = stage + warp * 64 * SP;
    {
        const float b1 = bvals[warp * 64 + (pair2 ? 2 * lane : lane)],
                    b2 = bvals[warp * 64 + (pair2 ? 2 * lane + 1 : lane + 32)];
        float* a = wst + lane * SP;
        float* b = wst + (lane + 32) * SP;
        float2* ab = reinterpret_cast<float2*>(wst) + lane * SP;  // pair2: [32 original lines][SP] float2
#pragma unroll
        for (int z = 0; z < P; ++z) {
            float r1 = v[z].x * g.scale + b1, r2 = v[z].y * g.scale + b2;
            if (g.act == 2) r1 = r1 > 0.f ? r1 : 0.f, r2 = r2 > 0.f ? r2 : 0.f;
            else if (g.act == 0) r1 = 1.f / (1.f + expf(-r1)), r2 = 1.f / (1.f + expf(-r2));
            else if (g.act == 1) r1 = tanhf(r1), r2 = tanhf(r2);
            if (pair2) {
                ab[z] = make_float2(r1, r2);
            } else {
                a[z] = r1;
                b[z] = r2;
            }
        }
    }
    __syncwarp();
    if (pair2) {
        constexpr int NQ2 = (P + 31) / 32;
        const float2* wst2 = reinterpret_cast<const float2*>(wst);
        for (int l = 0; l < 32; ++l) {
            const int64_t ob = __shfl_sync(0xffffffffu, obh[0], l);
            if (ob < 0) continue;  // (uniform)
            float2* dst = reinterpret_cast<float2*>(out + ob);
#pragma unroll
            for (int u = 0; u < NQ2; ++u) {
                const int q = lane + 32 * u;
                if (q < g.z_cnt) dst[q] = wst2[l * SP + q];
            }
        }
        return;
    }
    // warp-cooperative stores of each line (lanes along the kept z); line l's
    // output base comes from lane l % 32 by shuffles, the per-lane z offsets
    // and staging indices are loop invariant
    const int zst = g.phased ? g.ph.sz : 1;
    constexpr int NQ = (P + 31) / 32;
    int zo[NQ], so[NQ];
    bool qa[NQ];
#pragma unroll
    for (int u = 0; u < NQ; ++u) {
        const int q = lane + 32 * u;
        qa[u] = q < g.z_cnt;
        zo[u] = zst * q;
        so[u] = q * g.z_step;
    }
    const int znz = g.phased ? g.ph.nz : 1 << 30;
#pragma unroll 4
    for (int l = 0; l < 64; ++l) {
        const int src = l & 31;
        const bool hi = l >= 32;  // (uniform)
        const int64_t ob = __shfl_sync(0xffffffffu, hi ? obh[1] : obh[0], src);
        const int oz = __shfl_sync(0xffffffffu, hi ? ozh[1] : ozh[0], src);
        if (ob < 0) continue;  // (uniform) past the end, or a ragged phase line outside the tensor
        float* dst = out + ob + oz;
        const float* sl = wst + l * SP;
        const int zlim = znz - oz;
#pragma unroll
        for (int u = 0; u < NQ; ++u)
            if (qa[u] && zo[u] < zlim) dst[zo[u]] = sl[so[u]];
    }
}

// dilated kernels: dil[e][f_in][s*w] = w[e][f_in][w], zeros elsewhere (conv_direct.hpp:137-151)
// dilated kernels [nker][ex][ey][ez]: the volume is zeroed by a memset, then
// one thread per tap (coalesced reads of w) scatters it to its lattice site
__global__ void dilate_k(const float* __restrict__ w, int64_t ntaps, int kx, int ky, int kz, int sx, int sy, int sz,
                         float* __restrict__ dil) {
    const int ex = sx * (kx - 1) + 1, ey = sy * (ky - 1) + 1, ez = sz * (kz - 1) + 1;
    const int T = kx * ky * kz;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < ntaps; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t kk = i / T;
        const int t = int(i - kk * T);
        const int wx = t / (ky * kz), r = t - wx * (ky * kz), wy = r / kz, wz = r - wy * kz;
        dil[((kk * ex + sx * wx) * ey + sy * wy) * int64_t(ez) + sz * wz] = __ldg(w + i);
    }
}

// ---- sparse-tap plane DFTs for kernel spectra and kernel gradients ----
// A (dilated) kernel has kx*ky*kz nonzeros on an s-strided grid, so its
// spectrum needs no padded volume and no FFT: per z-bin plane
//   K[wx][wy] = sum_a e(-wx a sx) sum_b e(-wy b sy) T[a][b],
//   T[a][b]   = sum_c e(-wz c sz) w[a][b][c]                  (e(m) = exp(2 pi i m / P))
// is kx complex MACs per output bin, so the kernel-spectrum pass is one
// streaming write of K. Its adjoint, the kernel-gradient inverse, keeps only
// the kx*ky tap positions of each dK plane:
//   C[a][b] = sum_wy e(+wy b sy) sum_wx e(+wx a sx) dK[wx][wy]
// (the z inverse of the compact C planes then runs as before), so the dK
// pass is one streaming read. Square planes (P_x = P_y = P), taps <= KMAX.
constexpr int KMAX = 8;
constexpr int KS_THREADS = 256;
// planes per CTA step: one thread per column pair, at most 16 planes
__host__ __device__ constexpr int ks_planes(int P) { return KS_THREADS / (P / 2) < 16 ? KS_THREADS / (P / 2) : 16; }

// kernel spectra: a CTA takes G = 256 / (P/2) planes at a time. T and U of
// those planes go to shared memory, then each thread owns one column pair
// of one plane, keeps its U[a][wy..wy+1] in registers and walks the rows:
// K[wx] = sum_a U[a] t^a with t = e(-wx sx) by Horner (one broadcast twiddle
// load and 8 kx FMAs per 16-byte store).
// row-bin-major kernel spectra (tensor-core plans, ker = o F + i): planes
// ordered ((o * Zh + wz) * F + i), threads (column pair, plane) with the plane
// fastest, so consecutive maps i of one (o, wz) write their shared runs together
__device__ __forceinline__ void plane_decode(int gF, int64_t q, int Zh, int64_t& ker, int& wz) {
    if (gF) {
        const int64_t r = q / gF;
        const int64_t o = r / Zh;
        wz = int(r - o * Zh);
        ker = o * gF + (q % gF);
    } else {
        ker = q / Zh;
        wz = int(q - ker * Zh);
    }
}
// float2 index of bin (wz, wx = 0, wy) of kernel ker = o F + i (row-bin-major)
__device__ __forceinline__ int64_t kspec_rbm(int gF, int64_t ker, int Zh, int P, int wz, int wy) {
    const int64_t o = ker / gF, i = ker - o * gF;
    return ((o * Zh + wz) * int64_t(P) * P + wy) * gF + i;
}

template <int P>
__global__ void __launch_bounds__(KS_THREADS) kspec_k(const float* __restrict__ w, int64_t planes, int Zh, int Pz,
                                                      int kx, int ky, int kz, int sx, int sy, int sz,
                                                      float2* __restrict__ K, int gF) {
    constexpr int CP = P / 2;
    constexpr int G = ks_planes(P);
    __shared__ float2 tw[P];                  // exp(-2 pi i m / P)
    __shared__ float2 twz[MAXP];              // exp(-2 pi i m / Pz)
    __shared__ float2 T[G * KMAX * KMAX];     // [g][a][b]
    __shared__ float4 U[G * KMAX * CP];       // [g][a][pair]
    for (int m = threadIdx.x; m < P; m += KS_THREADS) {
        float sn, cs;
        sincospif(-2.f * float(m) / float(P), &sn, &cs);
        tw[m] = make_float2(cs, sn);
    }
    for (int m = threadIdx.x; m < Pz; m += KS_THREADS) {
        float sn, cs;
        sincospif(-2.f * float(m) / float(Pz), &sn, &cs);
        twz[m] = make_float2(cs, sn);
    }
    const int taps = kx * ky * kz, kxy = kx * ky;
    // planes per step: row-bin-major steps take a multiple of 8 consecutive maps
    // (aligned runs of whole sectors; F is a multiple of 8)
    const int Gs = gF ? (G / 8) * 8 : G;
    int g, cp;
    if (gF) {
        g = threadIdx.x % Gs, cp = threadIdx.x / Gs;
    } else {
        g = threadIdx.x / CP, cp = threadIdx.x - (threadIdx.x / CP) * CP;
    }
    const int mx = sx % P;
    for (int64_t q0 = int64_t(blockIdx.x) * Gs; q0 < planes; q0 += int64_t(gridDim.x) * Gs) {
        __syncthreads();  // twiddles ready / previous planes' U consumed
        // T[g][a][b] = sum_c w[a][b][c] e(-wz c sz)
        for (int t = threadIdx.x; t < Gs * kxy; t += KS_THREADS) {
            const int gg = t / kxy, ab = t - gg * kxy;
            const int64_t q = q0 + gg;
            float2 acc = make_float2(0.f, 0.f);
            if (q < planes) {
                int64_t ker;
                int wz;
                plane_decode(gF, q, Zh, ker, wz);
                const float* wk = w + ker * taps + ab * kz;
                const int mz = (wz * sz) % Pz;
                int m = 0;
                for (int c = 0; c < kz; ++c) {
                    const float v = __ldg(wk + c);
                    const float2 e = twz[m];
                    acc.x = fmaf(v, e.x, acc.x);
                    acc.y = fmaf(v, e.y, acc.y);
                    m += mz;
                    if (m >= Pz) m -= Pz;
                }
            }
            T[gg * (KMAX * KMAX) + ab] = acc;
        }
        __syncthreads();
        // U[g][a][wy] = sum_b T[g][a][b] e(-wy b sy), two columns per entry
        for (int t = threadIdx.x; t < Gs * kx * CP; t += KS_THREADS) {
            const int gg = t / (kx * CP), r = t - gg * (kx * CP), a = r / CP, pr = r - (r / CP) * CP;
            const int my0 = (2 * pr * sy) % P, my1 = ((2 * pr + 1) * sy) % P;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            int m0 = 0, m1 = 0;
            for (int b = 0; b < ky; ++b) {
                const float2 v = T[gg * (KMAX * KMAX) + a * ky + b], e0 = tw[m0], e1 = tw[m1];
                cmac(acc.x, acc.y, v.x, v.y, e0.x, e0.y);
                cmac(acc.z, acc.w, v.x, v.y, e1.x, e1.y);
                m0 += my0;
                if (m0 >= P) m0 -= P;
                m1 += my1;
                if (m1 >= P) m1 -= P;
            }
            U[(gg * KMAX + a) * CP + pr] = acc;
        }
        __syncthreads();
        const int64_t q = q0 + g;
        if (g < Gs && cp < CP && q < planes) {
            float4 u[KMAX];
#pragma unroll
            for (int a = 0; a < KMAX; ++a) u[a] = a < kx ? U[(g * KMAX + a) * CP + cp] : make_float4(0.f, 0.f, 0.f, 0.f);
            float4* out = reinterpret_cast<float4*>(K + q * (int64_t(P) * P)) + cp;
            float2* outq = nullptr;  // row-bin-major: bin (wx, 2 cp) of this kernel
            if (gF) {
                int64_t ker;
                int wz;
                plane_decode(gF, q, Zh, ker, wz);
                outq = K + kspec_rbm(gF, ker, Zh, P, wz, 2 * cp);
            }
            int m = 0;
            for (int wx = 0; wx < P; ++wx) {
                const float2 t = tw[m];
                // Horner, entered at the kx-th coefficient (uniform branch)
                auto hs = [&](float4 acc, const float4& c) {  // acc * t + c
                    return make_float4(fmaf(acc.x, t.x, fmaf(-acc.y, t.y, c.x)), fmaf(acc.x, t.y, fmaf(acc.y, t.x, c.y)),
                                       fmaf(acc.z, t.x, fmaf(-acc.w, t.y, c.z)), fmaf(acc.z, t.y, fmaf(acc.w, t.x, c.w)));
                };
                float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
                switch (kx) {
                    case 8: acc = u[7]; [[fallthrough]];
                    case 7: acc = hs(acc, u[6]); [[fallthrough]];
                    case 6: acc = hs(acc, u[5]); [[fallthrough]];
                    case 5: acc = hs(acc, u[4]); [[fallthrough]];
                    case 4: acc = hs(acc, u[3]); [[fallthrough]];
                    case 3: acc = hs(acc, u[2]); [[fallthrough]];
                    case 2: acc = hs(acc, u[1]); [[fallthrough]];
                    default: acc = hs(acc, u[0]);
                }
                if (gF) {
                    __stcs(outq + int64_t(wx) * P * gF, make_float2(acc.x, acc.y));
                    __stcs(outq + int64_t(wx) * P * gF + gF, make_float2(acc.z, acc.w));
                } else {
                    __stcs(out + wx * CP, acc);
                }
                m += mx;
                if (m >= P) m -= P;
            }
        }
    }
}

// kernel-gradient inverse, xy part: a CTA takes G = 256 / (P/2) planes at a
// time, one thread per (plane, column pair) walking the rows (coalesced 16-B
// loads; the kx column sums in registers, twiddles of row wx read in pairs
// from a [wx][a] table), then the kx*ky outputs per plane as warp dot
// products over the columns. out: compact [plane][a][b].
template <int P>
__global__ void __launch_bounds__(KS_THREADS, 3) dkinv_xy_k(const float2* __restrict__ DK, int64_t planes, int kx,
                                                         int ky, int sx, int sy, float2* __restrict__ out, int Zh,
                                                         int gF) {
    constexpr int CP = P / 2;                  // column pairs per plane
    constexpr int G = ks_planes(P);            // planes per CTA step
    __shared__ float2 tw[P];                   // exp(-2 pi i m / P); the inverse uses conj
    __shared__ float4 tw2[P * (KMAX / 2)];     // [wx][a pair]: e(-wx a sx), e(-wx (a+1) sx)
    __shared__ float2 W[G * KMAX * P];         // [g][a][wy]
    constexpr bool TWB = P <= 96;              // (P = 128: no room under the 48 KB static limit)
    __shared__ float2 twb[TWB ? KMAX * P : 1]; // [b][wy]: e(-wy b sy) (lanes read consecutive wy)
    for (int m = threadIdx.x; m < P; m += KS_THREADS) {
        float sn, cs;
        sincospif(-2.f * float(m) / float(P), &sn, &cs);
        tw[m] = make_float2(cs, sn);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < P * (KMAX / 2); t += KS_THREADS) {
        const int wx = t / (KMAX / 2), ap = t - wx * (KMAX / 2);
        const float2 e0 = tw[(wx * 2 * ap * sx) % P], e1 = tw[(wx * (2 * ap + 1) * sx) % P];
        tw2[t] = make_float4(e0.x, e0.y, e1.x, e1.y);
    }
    if constexpr (TWB)
        for (int t = threadIdx.x; t < ky * P; t += KS_THREADS) {
            const int b = t / P, wy = t - (t / P) * P;
            twb[t] = tw[(wy * ((b * sy) % P)) % P];
        }
    const int Gs = gF ? (G / 8) * 8 : G;  // planes per step (row-bin-major: see kspec_k)
    int g, cp;
    if (gF) {
        g = threadIdx.x % Gs, cp = threadIdx.x / Gs;
    } else {
        g = threadIdx.x / CP, cp = threadIdx.x - (threadIdx.x / CP) * CP;
    }
    for (int64_t q0 = int64_t(blockIdx.x) * Gs; q0 < planes; q0 += int64_t(gridDim.x) * Gs) {
        __syncthreads();  // tables ready / previous W consumed
        const int64_t q = q0 + g;
        if (g < Gs && cp < CP && q < planes) {
            const float4* src = reinterpret_cast<const float4*>(DK + q * (int64_t(P) * P)) + cp;
            const float2* srcq = nullptr;
            if (gF) {
                int64_t ker;
                int zb;
                plane_decode(gF, q, Zh, ker, zb);
                srcq = DK + kspec_rbm(gF, ker, Zh, P, zb, 2 * cp);
            }
            float4 acc[KMAX];
#pragma unroll
            for (int a = 0; a < KMAX; ++a) acc[a] = make_float4(0.f, 0.f, 0.f, 0.f);
            // rows in groups of RG, all loads of a group in flight before its FMAs
            constexpr int RG = P % 8 == 0 ? 8 : (P % 4 == 0 ? 4 : 2);
#pragma unroll 1
            for (int wx0 = 0; wx0 < P; wx0 += RG) {
                float4 vr[RG];
#pragma unroll
                for (int j = 0; j < RG; ++j) {
                    if (gF) {
                        const float2 a0 = __ldcs(srcq + int64_t(wx0 + j) * P * gF),
                                     a1 = __ldcs(srcq + int64_t(wx0 + j) * P * gF + gF);
                        vr[j] = make_float4(a0.x, a0.y, a1.x, a1.y);
                    } else {
                        vr[j] = __ldcs(src + (wx0 + j) * CP);
                    }
                }
#pragma unroll
                for (int j = 0; j < RG; ++j) {
                const int wx = wx0 + j;
                const float4 v = vr[j];
#pragma unroll
                for (int ap = 0; ap < KMAX / 2; ++ap) {
                    if (2 * ap < kx) {
                        const float4 e = tw2[wx * (KMAX / 2) + ap];
                        cmacc(acc[2 * ap].x, acc[2 * ap].y, v.x, v.y, e.x, e.y);
                        cmacc(acc[2 * ap].z, acc[2 * ap].w, v.z, v.w, e.x, e.y);
                        if (2 * ap + 1 < kx) {
                            cmacc(acc[2 * ap + 1].x, acc[2 * ap + 1].y, v.x, v.y, e.z, e.w);
                            cmacc(acc[2 * ap + 1].z, acc[2 * ap + 1].w, v.z, v.w, e.z, e.w);
                        }
                    }
                }
                }
            }
#pragma unroll
            for (int a = 0; a < KMAX; ++a)
                if (a < kx) {
                    W[(g * KMAX + a) * P + 2 * cp] = make_float2(acc[a].x, acc[a].y);
                    W[(g * KMAX + a) * P + 2 * cp + 1] = make_float2(acc[a].z, acc[a].w);
                }
        }
        __syncthreads();
        // outputs (g, a, b): one thread per output, a serial dot product over wy
        // (a warp per output spent ~50 instructions per warp on 20-48 terms and a
        // shuffle tree: this phase, not the streaming read above, bound the small pads)
        const int nout = Gs * kx * ky;
        for (int o = threadIdx.x; o < nout; o += KS_THREADS) {
            const int gg = o / (kx * ky), r = o - gg * (kx * ky), a = r / ky, b = r - (r / ky) * ky;
            int64_t qq = q0 + gg;
            if (qq >= planes) continue;
            if (gF) {  // compact output stays in image-major plane order (ker * Zh + zb)
                int64_t ker;
                int zb;
                plane_decode(gF, qq, Zh, ker, zb);
                qq = ker * Zh + zb;
            }
            const float2* Wr = W + (gg * KMAX + a) * P;
            float2 acc = make_float2(0.f, 0.f);
#pragma unroll 4
            for (int wy = 0; wy < P; ++wy) {
                const float2 v = Wr[wy];
                const float2 e = TWB ? twb[TWB ? b * P + wy : 0] : tw[(wy * ((b * sy) % P)) % P];
                cmacc(acc.x, acc.y, v.x, v.y, e.x, e.y);
            }
            out[qq * (kx * ky) + a * ky + b] = acc;
        }
    }
}

// ---- per-frequency complex multiply-accumulate over converging edges ----
//
// Per frequency bin the sum over converging edges is a small complex matrix
// product (fwd: Y[b][o] = sum_i X[b][i] conj(K[o][i]); bwd: DX[b][i] =
// sum_o G[b][o] K[o][i]; upd: dK[o][i] = sum_b X[b][i] conj(G[b][o])). At
// B = 16 every kernel-spectrum element feeds 16 complex MACs, so these run
// near the FP32 FMA roofline, not the HBM one, and the register tiling has to
// keep shared-memory wavefronts well below the FMA issue rate:
//   * a CTA owns 16 bins; warp w owns bin pair w (float4 = 2 complex);
//   * lanes form an 8 x 4 grid over the two output dims, each thread a 4 x TB
//     (or 4 x 4) tile, so one reduction step is 8 shared loads (each touching
//     only 4 or 8 distinct 16-byte words: one wavefront, rows padded to an odd
//     16-byte pitch) against 128 FMAs per thread;
//   * operand rows of 16 bins (128 B) stream in by cp.async, double buffered;
//   * results leave through shared memory as whole 128-byte bin rows.
constexpr int CBINS = 16;     // bins per CTA
constexpr int CPR = 8;     // float4 pairs per bin row
constexpr int CPP = 9;     // padded row pitch (float4 units, odd: conflict-free)
constexpr int C_THREADS = 256;
constexpr int CNB = 32;    // fwd/bwd: outputs n per CTA (8 lanes x 4)
constexpr int CRC = 4;     // fwd/bwd: reduction steps per stage
constexpr int CSTAGES = 4; // fwd/bwd: cp.async ring depth
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    const int n = int(pred) << 4;  // 16 bytes, or zero-fill when out of range
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(gmem), "r"(n) : "memory");
}

template <int TB>
constexpr size_t cmac_smem() {
    return sizeof(float4) * size_t(CSTAGES * CRC * (CNB + 4 * TB) * CPP);
}

// fwd / bwd: O[b][n] = sum_r S[b][r] * op(K[n*kn + r*kr]), op = conj when CONJ.
// CTA: CNB n x 4*TB patches x CBINS bins. Grid x = (n block, patch block) with
// the patch blocks of one n block adjacent; grid y = bin blocks.
template <bool CONJ, int TB>
__global__ void __launch_bounds__(C_THREADS, 2) cmac_ss_k(const float2* __restrict__ S, const float2* __restrict__ K,
                                                          float2* __restrict__ O, int B, int nr, int nn, int64_t kn,
                                                          int64_t kr, int64_t bins) {
    constexpr int BB = 4 * TB;
    constexpr int KST = CRC * CNB * CPP, SST = CRC * BB * CPP;  // float4 per stage
    extern __shared__ float4 csm[];  // [CSTAGES][K stage] then [CSTAGES][S stage]
    float4* ks = csm;
    float4* ss = csm + CSTAGES * KST;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nl = lane & 7, bl = lane >> 3;
    const int nbb = (B + BB - 1) / BB;
    // 1-D grid: the (n block, patch block) tiles of one bin block adjacent
    // (S rows re-read from L2), bin blocks outermost (no 65535 grid.y limit)
    const int nxb = ((nn + CNB - 1) / CNB) * nbb;
    const int bx = int(blockIdx.x % unsigned(nxb));
    const int n0 = (bx / nbb) * CNB, b0 = (bx % nbb) * BB;
    const int64_t w0 = int64_t(blockIdx.x / unsigned(nxb)) * CBINS;
    // staging: thread -> (row, pair q); K rows (rr, n) for rr = j, S rows
    // (rr, b) for rr = rs + j * (32 / BB); per chunk the sources advance by
    // CRC reduction steps
    const int q = threadIdx.x & 7, trow = threadIdx.x >> 3;  // trow < 32
    const int64_t w = w0 + 2 * q;
    const bool wok = w < bins;
    const bool kok = wok && n0 + trow < nn;
    const float2* kp = K + (int64_t(n0 + trow) * kn) * bins + w;
    const int64_t kstep = kr * bins;
    constexpr int SJ = (CRC * BB + 31) / 32;          // S pieces per thread
    constexpr int RSTEP = 32 / BB;                     // rr advance per S piece
    const int sb_ = trow % BB, rs = trow / BB;
    const bool sok = wok && b0 + sb_ < B;
    const float2* sp = S + (int64_t(b0 + sb_) * nr + rs) * bins + w;
    float4* kdst = ks + trow * CPP + q;
    float4* sdst = ss + (rs * BB + sb_) * CPP + q;
    // running source pointers: one 64-bit add per piece
    const float2* kcur = kp;
    const float2* scur = sp;
    const int64_t sstep = int64_t(RSTEP) * bins;
    auto stage = [&](int c, int buf) {
        const int r0 = c * CRC;
#pragma unroll
        for (int j = 0; j < CRC; ++j) {
            const bool ok = kok && r0 + j < nr;
            cp_async16(kdst + buf * KST + j * (CNB * CPP), ok ? kcur : K, ok);
            kcur += kstep;
        }
#pragma unroll
        for (int j = 0; j < SJ; ++j) {
            if (rs + j * RSTEP < CRC) {  // TB = 1: half the threads stage S
                const bool ok = sok && r0 + rs + j * RSTEP < nr;
                cp_async16(sdst + buf * SST + j * (RSTEP * BB * CPP), ok ? scur + j * sstep : S, ok);
            }
        }
        scur += int64_t(CRC) * bins;
        cp_async_commit();
    };
    float4 acc[TB][4];
#pragma unroll
    for (int u = 0; u < TB; ++u)
#pragma unroll
        for (int t = 0; t < 4; ++t) acc[u][t] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int nchunks = (nr + CRC - 1) / CRC;
    // ring prologue: stages 0 .. CSTAGES-2 (one commit group each, empty past the end)
#pragma unroll
    for (int c = 0; c < CSTAGES - 1; ++c) {
        if (c < nchunks)
            stage(c, c);
        else
            cp_async_commit();
    }
    for (int c = 0; c < nchunks; ++c) {
        const int buf = c % CSTAGES;
        cp_async_wait<CSTAGES - 2>();  // stage c landed
        __syncthreads();               // ... for every thread; buffer (c-1) % CSTAGES is free
        if (c + CSTAGES - 1 < nchunks)
            stage(c + CSTAGES - 1, (c + CSTAGES - 1) % CSTAGES);
        else
            cp_async_commit();
        const float4* kb = ks + buf * KST + warp;
        const float4* sb = ss + buf * SST + warp;
#pragma unroll 1
        for (int rr = 0; rr < CRC; ++rr) {
            float4 kv[4], sv[TB];
#pragma unroll
            for (int t = 0; t < 4; ++t) kv[t] = kb[(rr * CNB + nl + 8 * t) * CPP];
#pragma unroll
            for (int u = 0; u < TB; ++u) sv[u] = sb[(rr * BB + bl + 4 * u) * CPP];
#pragma unroll
            for (int u = 0; u < TB; ++u)
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    float4& a = acc[u][t];
                    if (CONJ) {
                        cmacc(a.x, a.y, sv[u].x, sv[u].y, kv[t].x, kv[t].y);
                        cmacc(a.z, a.w, sv[u].z, sv[u].w, kv[t].z, kv[t].w);
                    } else {
                        cmac(a.x, a.y, sv[u].x, sv[u].y, kv[t].x, kv[t].y);
                        cmac(a.z, a.w, sv[u].z, sv[u].w, kv[t].z, kv[t].w);
                    }
                }
        }
    }
    cp_async_wait<0>();
    __syncthreads();  // every warp done with the ring before it holds the epilogue
    // epilogue: [BB][CNB] rows of 8 pairs through shared memory, whole rows out
    float4* es = csm;
#pragma unroll
    for (int u = 0; u < TB; ++u)
#pragma unroll
        for (int t = 0; t < 4; ++t) es[((bl + 4 * u) * CNB + nl + 8 * t) * CPP + warp] = acc[u][t];
    __syncthreads();
    for (int u = threadIdx.x; u < BB * CNB * CPR; u += C_THREADS) {
        const int qq = u & 7, row = u >> 3;
        const int nn_ = row % CNB, bb = row / CNB;
        const int b = b0 + bb, n = n0 + nn_;
        const int64_t ww = w0 + 2 * qq;
        if (b < B && n < nn && ww < bins)
            *reinterpret_cast<float4*>(O + (int64_t(b) * nn + n) * bins + ww) = es[(bb * CNB + nn_) * CPP + qq];
    }
}

// upd: dK[o][i] = sum_b X[b][i] * conj(G[b][o]). CTA: 32 o x 16 i x CBINS bins,
// lanes 8 (o) x 4 (i), thread tile 4 o x 4 i x 2 bins; X / G rows stream in
// UB-patch stages through a USTAGES-deep ring: the reduction is short (B =
// 16 is four stages), so all of a CTA's loads are in flight before its
// first FMA and only the first stage's latency is exposed (the other CTA on
// the SM covers it). A 2-deep ring left the SMs waiting (67 ms vs 47 ms for
// the equal-FLOP fwd CMAC on c5). Grid x = (o block, i block) with the i
// blocks of one o block adjacent (G rows re-read from L2); grid y = bin blocks.
constexpr int UO = 32, UI = 16, UB = 4, USTAGES = 4;
constexpr size_t kUpdSmem = sizeof(float4) * size_t(USTAGES * UB * (UO + UI) * CPP > UO * UI * CPP
                                                        ? USTAGES * UB * (UO + UI) * CPP
                                                        : UO * UI * CPP);
__global__ void __launch_bounds__(C_THREADS, 2) cmac_upd_ss_k(const float2* __restrict__ X,
                                                              const float2* __restrict__ G, float2* __restrict__ DK,
                                                              int B, int f, int fo, int64_t bins) {
    constexpr int ROWS = UO + UI;              // G rows then X rows per patch
    constexpr int STG = UB * ROWS * CPP;       // float4 per stage
    extern __shared__ float4 csm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ol = lane & 7, il = lane >> 3;
    const int nib = (f + UI - 1) / UI;
    // 1-D grid: (o block, i block) tiles of one bin block adjacent, bin blocks outermost
    const int nxb = nib * ((fo + UO - 1) / UO);
    const int bx = int(blockIdx.x % unsigned(nxb));
    const int i0 = (bx % nib) * UI, o0 = (bx / nib) * UO;
    const int64_t w0 = int64_t(blockIdx.x / unsigned(nxb)) * CBINS;
    // staging: thread -> (row, pair q); G rows (bb = j, o = trow), X rows
    // (bb = xb + 2 j, i = trow % 16); per chunk the sources advance UB patches
    const int q = threadIdx.x & 7, trow = threadIdx.x >> 3;  // trow < 32
    const int64_t w = w0 + 2 * q;
    const bool wok = w < bins;
    const bool gok = wok && o0 + trow < fo;
    const int xi = trow & 15, xb = trow >> 4;
    const bool xok = wok && i0 + xi < f;
    const float2* gp = G + int64_t(o0 + trow) * bins + w;
    const float2* xp = X + (int64_t(xb) * f + i0 + xi) * bins + w;
    const int64_t gstep = int64_t(fo) * bins, xstep = int64_t(f) * bins;
    float4* gdst = csm + trow * CPP + q;
    float4* xdst = csm + (xb * ROWS + UO + xi) * CPP + q;
    const float2* gcur = gp;
    const float2* xcur = xp;
    auto stage = [&](int c, int buf) {
        const int bc = c * UB;
#pragma unroll
        for (int j = 0; j < UB; ++j) {
            const bool ok = gok && bc + j < B;
            cp_async16(gdst + buf * STG + j * (ROWS * CPP), ok ? gcur : G, ok);
            gcur += gstep;
        }
#pragma unroll
        for (int j = 0; j < UB / 2; ++j) {
            const bool ok = xok && bc + xb + 2 * j < B;
            cp_async16(xdst + buf * STG + 2 * j * (ROWS * CPP), ok ? xcur : X, ok);
            xcur += 2 * xstep;
        }
        cp_async_commit();
    };
    float4 acc[4][4];  // [o t][i u]
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[t][u] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int nchunks = (B + UB - 1) / UB;
    // ring prologue: stages 0 .. USTAGES-2 (one commit group each, empty past the end)
#pragma unroll
    for (int c = 0; c < USTAGES - 1; ++c) {
        if (c < nchunks)
            stage(c, c);
        else
            cp_async_commit();
    }
    for (int c = 0; c < nchunks; ++c) {
        const int buf = c % USTAGES;
        cp_async_wait<USTAGES - 2>();  // stage c landed
        __syncthreads();               // ... for every thread; buffer (c-1) % USTAGES is free
        if (c + USTAGES - 1 < nchunks)
            stage(c + USTAGES - 1, (c + USTAGES - 1) % USTAGES);
        else
            cp_async_commit();
        const float4* base = csm + buf * STG + warp;
        const int nb = min(UB, B - c * UB);
#pragma unroll 1
        for (int bb = 0; bb < nb; ++bb) {
            float4 gv[4], xv[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) gv[t] = base[(bb * ROWS + ol + 8 * t) * CPP];
#pragma unroll
            for (int u = 0; u < 4; ++u) xv[u] = base[(bb * ROWS + UO + il + 4 * u) * CPP];
#pragma unroll
            for (int t = 0; t < 4; ++t)
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    cmacc(acc[t][u].x, acc[t][u].y, xv[u].x, xv[u].y, gv[t].x, gv[t].y);
                    cmacc(acc[t][u].z, acc[t][u].w, xv[u].z, xv[u].w, gv[t].z, gv[t].w);
                }
        }
    }
    cp_async_wait<0>();
    __syncthreads();  // every warp done with the ring before it holds the epilogue
    // epilogue: [UO][UI] rows of 8 pairs through shared memory
    float4* es = csm;
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int u = 0; u < 4; ++u) es[((il + 4 * u) * UO + ol + 8 * t) * CPP + warp] = acc[t][u];
    __syncthreads();
    for (int u = threadIdx.x; u < UO * UI * CPR; u += C_THREADS) {
        const int qq = u & 7, row = u >> 3;
        const int ii = row % UI, oo = row / UI;
        const int o = o0 + oo, i = i0 + ii;
        const int64_t ww = w0 + 2 * qq;
        if (o < fo && i < f && ww < bins)
            __stcs(reinterpret_cast<float4*>(DK + (int64_t(o) * f + i) * bins + ww), es[(ii * UO + oo) * CPP + qq]);
    }
}

}  // namespace

struct plan {
    dims3 P{1, 1, 1};
    int64_t Zh = 1, bins = 1;
    int64_t B = 0, f = 0, fo = 0;
    // polyphase plan of a dilated layer (sparsity s != 1): the layer runs as
    // the undilated layer `ce` over the s_x s_y s_z phase sub-volumes of every
    // patch (B*S "patches"); P, bins, X, K all belong to ce
    bool poly = false;
    conv_shape ce;
    int64_t S = 1;
    std::shared_ptr<znn_gpu::scratch> phase_ws;  // engine arena: phase-split tensors (explicit split path)
    int64_t ph_bytes = 0;    // phase-split tensors (explicit split path)
    bool tc = false;         // frequency-domain sums on the tensor cores (bgemm_tc.cu)
    float2* X = nullptr;  // memo: image spectra of the layer input [B*f][bins]
    float2* K = nullptr;  // memo: kernel spectra [fo*f][bins] (own buffer; null when pooled)
    float* dil = nullptr; // dilated kernels [fo*f][e^3]
    std::shared_ptr<kpool> pool;  // shared kernel-spectrum buffer (recomputed in bwd if clobbered)
    bool k_valid = false;         // own K holds the spectra of the current weights
    transform_counts cnt;
};

kpool::~kpool() { cudaFree(buf); }
float2* kpool::get(int64_t need) {
    if (need > bytes) {
        owner = nullptr;
        if (buf) {
            float2* old = buf;
            buf = nullptr;  // consistent state even if the new allocation fails
            bytes = 0;
            ZNN_CUDA_CHECK(cudaFree(old));
        }
        znn_gpu::dmalloc(&buf, size_t(need));
        bytes = need;
    }
    return buf;
}

void plan_deleter::operator()(plan* p) const {
    if (!p) return;
    cudaFree(p->X);
    cudaFree(p->K);
    cudaFree(p->dil);
    if (p->pool && p->pool->owner == p) p->pool->owner = nullptr;
    delete p;
}

const transform_counts& counts(const plan& p) { return p.cnt; }
void pad_dims(const plan& p, int64_t out[3]) { out[0] = p.P.x, out[1] = p.P.y, out[2] = p.P.z; }

namespace {

constexpr int64_t kMaxSpectrumBytes = int64_t(64) << 30;  // kernel spectra per layer (c5 conv2 at P = 96: 52 GB)

int64_t pad_axis(int64_t n) { return n <= 1 ? 1 : good_size(n); }

// Any pad >= n per axis is exact (the circular wrap only touches zeros,
// conv_fft.hpp:67-71). x and y share one pad (square xy planes, one compiled
// plane kernel per size) unless the volume is 2-D (x = 1).
// A dilated convolution is s_x s_y s_z undilated ones on the phase
// sub-volumes: with o = s q + r, y[s q + r] = sum_w x[s (q + w) + r] k[w] =
// conv_valid(x_r, k)[q], x_r[p] = x[s p + r] (conv_direct.hpp:39-68 with the
// dilated kernel of conv_direct.hpp:137-151). The adjoint and the kernel
// gradient split the same way (the kernel gradient sums over the phases).
// So the FFT engine transforms the phases at pad >= ceil(n / s) and the
// UNDILATED kernel: kernel spectra shrink by s^3 (c5 conv2: 52 -> 6.6 GB,
// conv3-5: 30 / 16 / 6.6 GB -> 0.5 / 0.3 / 0.1 GB) and the frequency-domain
// sums over converging edges reuse each kernel-spectrum bin for B s^3 phase
// images instead of B patches. ZNN_FFT_POLY=0 keeps the dilated-kernel path.
bool use_poly(const conv_shape& c) {
    if (c.s.x == 1 && c.s.y == 1 && c.s.z == 1) return false;
    const char* e = std::getenv("ZNN_FFT_POLY");
    return !(e && std::string(e) == "0");
}
conv_shape effective(const conv_shape& c) {
    if (!use_poly(c)) return c;
    const dims3 nr{ceil_div(c.n.x, c.s.x), ceil_div(c.n.y, c.s.y), ceil_div(c.n.z, c.s.z)};
    return conv_shape::make(c.B * c.s.x * c.s.y * c.s.z, c.f_in, c.f_out, nr, c.k, dims3{1, 1, 1});
}

dims3 pads_for_eff(const conv_shape& c) {
    dims3 P{pad_axis(c.n.x), pad_axis(c.n.y), pad_axis(c.n.z)};
    if (P.x > 1) P.x = P.y = std::max(P.x, P.y);
    if (P.z % 2) P.z = good_size(P.z + 1);  // R2C axis must be even
    return P;
}
dims3 pads_for(const conv_shape& c) { return pads_for_eff(effective(c)); }

// z passes: twiddles + per-line exchange buffers + the half-spectrum stash
size_t smem_for(int P) { return sizeof(float2) * (size_t(P) + size_t(LINES) * size_t(xpitch(P)) + size_t(LINES) * size_t(P / 2 + 2)); }
// xy passes: twiddles + exchange buffers + the [PX][PY+1] plane
size_t smem_xy(int PX, int PY) {
    const int PM = xpitch(PX) > xpitch(PY) ? xpitch(PX) : xpitch(PY);
    return sizeof(float2) * (size_t(PX + PY) + size_t(LINES) * size_t(PM) + size_t(PX) * size_t(PY + 1));
}

// compile-time pad dispatch: f(std::integral_constant<int, P>) for P in kPads
template <typename F>
void dispatch_pad(int P, F&& f) {
    switch (P) {
        case 2: f(std::integral_constant<int, 2>{}); break;
        case 4: f(std::integral_constant<int, 4>{}); break;
        case 8: f(std::integral_constant<int, 8>{}); break;
        case 12: f(std::integral_constant<int, 12>{}); break;
        case 16: f(std::integral_constant<int, 16>{}); break;
        case 20: f(std::integral_constant<int, 20>{}); break;
        case 24: f(std::integral_constant<int, 24>{}); break;
        case 32: f(std::integral_constant<int, 32>{}); break;
        case 40: f(std::integral_constant<int, 40>{}); break;
        case 48: f(std::integral_constant<int, 48>{}); break;
        case 64: f(std::integral_constant<int, 64>{}); break;
        case 72: f(std::integral_constant<int, 72>{}); break;
        case 80: f(std::integral_constant<int, 80>{}); break;
        case 96: f(std::integral_constant<int, 96>{}); break;
        case 128: f(std::integral_constant<int, 128>{}); break;
        default: throw znn_gpu::shape_error("fft: no compiled transform for pad " + std::to_string(P));
    }
}

// persistent double-buffered xy passes: twiddles + exchange buffers + 2 planes
size_t smem_pipe(int P) {
    return sizeof(float2) * (size_t(P) + size_t(LINES) * size_t(xpitch(P)) + 2 * size_t(P) * size_t(P + 2));
}
// as many CTAs as fit on the 148 SMs at once (never more than planes)
unsigned pipe_grid(int64_t planes, size_t smem) {
    int64_t per_sm = int64_t(220 * 1024) / int64_t(smem + 1024);
    if (per_sm < 1) per_sm = 1;
    if (per_sm > 8) per_sm = 8;
    const int64_t g = 148 * per_sm;
    return unsigned(planes < g ? planes : g);
}

template <typename K>
void allow_smem(K* k, size_t bytes) {
    ZNN_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
}

template <bool CONJ, int TB>
void cmac_ss_launch(cudaStream_t st, const float2* S, const float2* K, float2* O, int B, int nr, int nn, int64_t kn,
                    int64_t kr, int64_t bins) {
    constexpr size_t smem = cmac_smem<TB>();
    const int64_t nblk = ceil_div(nn, CNB) * ceil_div(B, 4 * TB) * ceil_div(bins, CBINS);
    require(nblk < (int64_t(1) << 31), "fft cmac: grid exceeds 2^31 blocks");
    const dim3 grid(unsigned(nblk), 1u, 1u);
    allow_smem(cmac_ss_k<CONJ, TB>, smem);
    cmac_ss_k<CONJ, TB><<<grid, C_THREADS, smem, st>>>(S, K, O, B, nr, nn, kn, kr, bins);
}

void cmac_ss(cudaStream_t st, const float2* S, const float2* K, float2* O, int B, int nr, int nn, int64_t kn,
             int64_t kr, int64_t bins, bool conj) {
    require(bins % 2 == 0, "fft cmac: odd bin count");
    // patch tile 4*TB: the smallest that covers B (whole batch per CTA up to 16)
    auto go = [&](auto tb) {
        constexpr int TB = decltype(tb)::value;
        if (conj)
            cmac_ss_launch<true, TB>(st, S, K, O, B, nr, nn, kn, kr, bins);
        else
            cmac_ss_launch<false, TB>(st, S, K, O, B, nr, nn, kn, kr, bins);
    };
    if (B <= 4)
        go(std::integral_constant<int, 1>{});
    else if (B <= 8)
        go(std::integral_constant<int, 2>{});
    else
        go(std::integral_constant<int, 4>{});
}

void cmac_upd(cudaStream_t st, const float2* X, const float2* G, float2* DK, int B, int f, int fo, int64_t bins) {
    require(bins % 2 == 0, "fft cmac: odd bin count");
    const int64_t nblk = ceil_div(f, UI) * ceil_div(fo, UO) * ceil_div(bins, CBINS);
    require(nblk < (int64_t(1) << 31), "fft cmac: grid exceeds 2^31 blocks");
    allow_smem(cmac_upd_ss_k, kUpdSmem);
    cmac_upd_ss_k<<<unsigned(nblk), C_THREADS, kUpdSmem, st>>>(X, G, DK, B, f, fo, bins);
}

// forward 3D R2C of imgs real volumes (valid dims n, image stride in floats):
// z pass (transposed store) + fused xy pass
// bias gradient of a fused transfer edge from the spectra (transfer.hpp:
// 108-121): sum over patches and voxels of the gated gradient = the DC term,
// here the sum over the valid (x, y) lines of the z pass's zb = 0 plane
__global__ void __launch_bounds__(1024) dc_bias_k(const float2* __restrict__ spec, int B, int fo, int64_t img_stride,
                                                 int nx, int ny, int py, float* __restrict__ dbias, int gF) {
    const int o = blockIdx.x;
    double acc = 0.0;
    const int64_t per = int64_t(nx) * ny, total = int64_t(B) * per;
    for (int64_t i = threadIdx.x; i < total; i += blockDim.x) {
        const int64_t b = i / per, r = i - b * per;
        const int x = int(r / ny), y = int(r - (r / ny) * ny);
        acc += double(spec[spec_at(gF, b * fo + o, img_stride, int64_t(x) * py + y)].x);
    }
    __shared__ double red[1024];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int w = int(blockDim.x) / 2; w > 0; w >>= 1) {
        if (int(threadIdx.x) < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) dbias[o] = float(red[0]);
}

// gate: optional ReLU output gating the input (fused transfer backward);
// dbias (with gate): receives the per-map sum over the batch (imgs = B * dmaps)
bool small_cube(const plan& p) {
    return p.P.x == p.P.y && p.P.y == p.P.z && p.P.x > 1 && p.P.x <= SMALLP && !std::getenv("ZNN_FFT_NO_CUBE");
}

// ph: the images are the phases of an original tensor (polyphase plan, small
// cubes only): read in place, no split pass
void forward3d(cudaStream_t st, const plan& p, const float* in, int64_t in_img_stride, dims3 n, int64_t imgs,
               float2* spec, bool z_only = false, const float* gate = nullptr, float* dbias = nullptr,
               int64_t dmaps = 1, const phase_geom* ph = nullptr, int64_t maps = 0) {
    // tensor-core plans keep every spectrum row-bin-major with F = maps
    const int quad = p.tc ? int(maps) : 0;
    require(!p.tc || (maps > 0 && imgs % maps == 0), "fft: row-bin-major spectrum needs its map count");
    if (!z_only && small_cube(p)) {
        cube_io a{};
        a.src = in, a.gate = gate, a.img_stride = in_img_stride;
        a.nx = int(n.x), a.ny = int(n.y), a.nz = int(n.z);
        a.phased = ph ? 1 : 0;
        if (ph) a.ph = *ph;
        a.gF = quad;
        a.vec4 = !ph && n.z % 4 == 0 && in_img_stride % 4 == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0 &&
                 (reinterpret_cast<uintptr_t>(gate) & 15) == 0;
        require(imgs < (int64_t(1) << 31), "fft: too many images");
        dispatch_pad(int(p.P.x), [&](auto pc) {
            constexpr int PP = decltype(pc)::value;
            if constexpr (PP <= REGP) {
                if (quad) {  // row-bin-major: NI images per CTA (use_tc keeps these plans on this path)
                    auto run = [&](auto ni) {
                        constexpr int NI = decltype(ni)::value;
                        require(imgs % NI == 0, "fft: row-bin-major images not a multiple of the CTA's images");
                        allow_smem(fft3_fwd_reg_k<PP, NI, true>, cube_reg_smem<PP, NI>());
                        fft3_fwd_reg_k<PP, NI, true><<<unsigned(imgs / NI), cube_threads<NI>(), cube_reg_smem<PP, NI>(), st>>>(
                            a, spec);
                    };
                    const int ni = cube_grp_ni<PP>();
                    if (ni == 1) run(std::integral_constant<int, 1>{});
                    else if (ni == 2) run(std::integral_constant<int, 2>{});
                    else run(std::integral_constant<int, 4>{});
                    return;
                }
                if (!std::getenv("ZNN_FFT_CUBE_LINES")) {
                    allow_smem(fft3_fwd_reg_k<PP, 1>, cube_reg_smem<PP, 1>());
                    fft3_fwd_reg_k<PP, 1><<<unsigned(imgs), RTHREADS, cube_reg_smem<PP, 1>(), st>>>(a, spec);
                    return;
                }
            }
            if constexpr (PP <= SMALLP) {
                require(!quad, "fft: row-bin-major layout needs the register cube kernels (pad <= 24)");
                allow_smem(fft3_fwd_small_k<PP>, cube_fwd_smem<PP>());
                fft3_fwd_small_k<PP><<<unsigned(imgs), THREADS, cube_fwd_smem<PP>(), st>>>(a, spec);
            }
        });
        launch_check("fft3_fwd_small");
        if (dbias) {  // the DC bin of each image's spectrum is its voxel sum
            dc_bias_k<<<unsigned(dmaps), 1024, 0, st>>>(spec, int(imgs / dmaps), int(dmaps), p.Zh * p.P.x * p.P.y, 1, 1,
                                                       int(p.P.y), dbias, quad);
            launch_check("fft_dc_bias");
        }
        return;
    }
    require(ph == nullptr || !z_only, "fft: phase addressing with a z-only pass");
    const int64_t nlines = imgs * n.x * n.y;
    require(nlines < (int64_t(1) << 32), "fft: too many transform lines");
    dispatch_pad(int(p.P.z), [&](auto pc) {
        constexpr int PP = decltype(pc)::value;
        if constexpr (PP >= 8 && PP <= 64) {
            if (!std::getenv("ZNN_FFT_Z_LINES")) {  // line pairs in registers (ZNN_FFT_Z_LINES=1: 8 threads per line)
                allow_smem(fft_z_fwd_reg_k<PP>, zr_smem<PP>(true));
                fft_z_fwd_reg_k<PP><<<unsigned(ceil_div(nlines, ZR_LINES)), ZR_THREADS, zr_smem<PP>(gate != nullptr), st>>>(
                    in, in_img_stride, int(n.x), int(n.y), int(n.z), nlines, spec, int(p.P.x), int(p.P.y), gate,
                    ph ? *ph : phase_geom{}, ph ? 1 : 0, quad);
                return;
            }
        }
        allow_smem(fft_z_fwd_k<PP>, smem_for(PP));
        fft_z_fwd_k<PP><<<unsigned(ceil_div(nlines, LINES)), THREADS, smem_for(PP), st>>>(
            in, in_img_stride, int(n.x), int(n.y), int(n.z), nlines, spec, int(p.P.x), int(p.P.y), gate,
            ph ? *ph : phase_geom{}, ph ? 1 : 0, quad);
    });
    launch_check("fft_z_fwd");
    if (dbias) {
        dc_bias_k<<<unsigned(dmaps), 1024, 0, st>>>(spec, int(imgs / dmaps), int(dmaps), p.Zh * p.P.x * p.P.y,
                                                   int(n.x), int(n.y), int(p.P.y), dbias, quad);
        launch_check("fft_dc_bias");
    }
    if (z_only) return;
    const int64_t planes = imgs * p.Zh;
    dispatch_pad(int(p.P.y), [&](auto pc) {
        constexpr int PY = decltype(pc)::value;
        if (p.P.x == 1) {
            allow_smem(fft_xy_fwd_k<1, PY>, smem_xy(1, PY));
            fft_xy_fwd_k<1, PY><<<unsigned(planes), THREADS, smem_xy(1, PY), st>>>(spec, planes, int(n.x), int(n.y));
        } else if (quad) {  // row-bin-major layout: the planes of 4 maps per CTA
            if constexpr (PY <= 64) {
                require(planes % XP_NI == 0 && quad % XP_NI == 0, "fft: row-bin-major maps not a multiple of 4");
                allow_smem(fft_xy_fwd_pair_k<PY>, smem_xy_pair<PY>());
                fft_xy_fwd_pair_k<PY><<<unsigned(planes / XP_NI), xp_threads<PY>(), smem_xy_pair<PY>(), st>>>(
                    spec, int(n.x), int(n.y), int(p.Zh), quad);
            }
        } else if (smem_pipe(PY) > size_t(220) * 1024 || !std::getenv("ZNN_FFT_XY_PIPE")) {
            // one plane per CTA, two CTAs per SM: faster than the persistent
            // double-buffered pass for the forward (c5: 9.1 vs 10.5 ms at P = 96,
            // 5.9 vs 7.0 at 80); the inverse keeps the persistent pass
            allow_smem(fft_xy_fwd_k<PY, PY>, smem_xy(PY, PY));
            fft_xy_fwd_k<PY, PY><<<unsigned(planes), THREADS, smem_xy(PY, PY), st>>>(spec, planes, int(n.x),
                                                                                      int(n.y));
        } else {
            const size_t sm = smem_pipe(PY);
            allow_smem(fft_xy_fwd_pipe_k<PY>, sm);
            fft_xy_fwd_pipe_k<PY><<<pipe_grid(planes, sm), THREADS, sm, st>>>(spec, planes, int(n.x), int(n.y));
        }
    });
    launch_check("fft_xy_fwd");
}

void inverse_z(cudaStream_t st, const plan& p, int64_t imgs, dims3 step, dims3 cnt, float* out, int64_t out_img_stride,
               const float* bias, int bias_mod, int act, const float2* cbuf, const phase_geom* ph = nullptr);

// inverse 3D C2R keeping voxels (x,y,z) = (step*i) for i < cnt per axis,
// written as a dense box [imgs][cnt.x][cnt.y][cnt.z] (image stride given);
// cbuf holds the compact kept planes between the two passes
void inverse3d(cudaStream_t st, const plan& p, const float2* spec, int64_t imgs, dims3 step, dims3 cnt, float* out,
               int64_t out_img_stride, const float* bias, int bias_mod, int act, float2* cbuf,
               const phase_geom* ph = nullptr, int64_t maps = 0) {
    require(step.x * (cnt.x - 1) < p.P.x && step.y * (cnt.y - 1) < p.P.y && step.z * (cnt.z - 1) < p.P.z,
            "fft: kept voxels outside the padded volume");
    const int quad = p.tc ? int(maps) : 0;  // row-bin-major spectra: F = maps
    require(!p.tc || (maps > 0 && imgs % maps == 0), "fft: row-bin-major spectrum needs its map count");
    if (small_cube(p)) {
        cube_io a{};
        a.dst = out, a.img_stride = out_img_stride;
        a.xs = int(step.x), a.xc = int(cnt.x), a.ys = int(step.y), a.yc = int(cnt.y), a.zs = int(step.z),
        a.zc = int(cnt.z);
        a.oy = int(cnt.y), a.oz = int(cnt.z);
        a.bias_mod = bias_mod > 0 ? bias_mod : 1;
        a.act = act;
        a.scale = float(1.0 / double(p.P.x * p.P.y * p.P.z));
        a.phased = ph ? 1 : 0;
        if (ph) a.ph = *ph;
        a.gF = quad;
        require(imgs < (int64_t(1) << 31), "fft: too many images");
        const bool unit = a.xs == 1 && a.ys == 1 && a.zs == 1;
        a.vec4 = !ph && unit && cnt.z % 4 == 0 && out_img_stride % 4 == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
        dispatch_pad(int(p.P.x), [&](auto pc) {
            constexpr int PP = decltype(pc)::value;
            auto go = [&](auto k, int64_t ctas, int threads, size_t sm) {
                allow_smem(k, sm);
                k<<<unsigned(ctas), threads, sm, st>>>(spec, a, bias);
            };
            if constexpr (PP <= REGP) {
                if (quad) {
                    auto run = [&](auto ni) {
                        constexpr int NI = decltype(ni)::value;
                        require(imgs % NI == 0, "fft: row-bin-major images not a multiple of the CTA's images");
                        if (unit)
                            go(fft3_inv_reg_k<PP, NI, true, true>, imgs / NI, cube_threads<NI>(), cube_reg_smem<PP, NI>());
                        else
                            go(fft3_inv_reg_k<PP, NI, false, true>, imgs / NI, cube_threads<NI>(), cube_reg_smem<PP, NI>());
                    };
                    const int ni = cube_grp_ni<PP>(true);
                    if (ni == 1) run(std::integral_constant<int, 1>{});
                    else if (ni == 2) run(std::integral_constant<int, 2>{});
                    else run(std::integral_constant<int, 4>{});
                    return;
                }
                if (!std::getenv("ZNN_FFT_CUBE_LINES")) {
                    if (unit)
                        go(fft3_inv_reg_k<PP, 1, true>, imgs, RTHREADS, cube_reg_smem<PP, 1>());
                    else
                        go(fft3_inv_reg_k<PP, 1, false>, imgs, RTHREADS, cube_reg_smem<PP, 1>());
                    return;
                }
            }
            if constexpr (PP <= SMALLP) {
                require(!quad, "fft: row-bin-major layout needs the register cube kernels (pad <= 24)");
                if (unit)
                    go(fft3_inv_small_k<PP, true>, imgs, THREADS, cube_smem<PP>());
                else
                    go(fft3_inv_small_k<PP, false>, imgs, THREADS, cube_smem<PP>());
            }
        });
        launch_check("fft3_inv_small");
        return;
    }

    const int64_t planes = imgs * p.Zh;
    dispatch_pad(int(p.P.y), [&](auto pc) {
        constexpr int PY = decltype(pc)::value;
        if (p.P.x == 1) {
            allow_smem(fft_xy_inv_k<1, PY>, smem_xy(1, PY));
            fft_xy_inv_k<1, PY><<<unsigned(planes), THREADS, smem_xy(1, PY), st>>>(
                spec, cbuf, planes, int(step.x), int(cnt.x), int(step.y), int(cnt.y));
        } else if (quad) {  // row-bin-major layout: the planes of 4 maps per CTA
            if constexpr (PY <= 64) {
                require(planes % XP_NI == 0 && quad % XP_NI == 0, "fft: row-bin-major maps not a multiple of 4");
                auto go = [&](auto kern) {
                    allow_smem(kern, smem_xy_pair<PY>());
                    kern<<<unsigned(planes / XP_NI), xp_threads<PY>(), smem_xy_pair<PY>(), st>>>(
                        spec, cbuf, int(step.x), int(cnt.x), int(step.y), int(cnt.y), int(p.Zh), quad);
                };
                if (step.x == 1 && step.y == 1)
                    go(fft_xy_inv_pair_k<PY, true>);
                else
                    go(fft_xy_inv_pair_k<PY, false>);
            }
        } else if (smem_pipe(PY) > size_t(220) * 1024) {  // two 128^2 planes do not fit: single buffer
            allow_smem(fft_xy_inv_k<PY, PY>, smem_xy(PY, PY));
            fft_xy_inv_k<PY, PY><<<unsigned(planes), THREADS, smem_xy(PY, PY), st>>>(
                spec, cbuf, planes, int(step.x), int(cnt.x), int(step.y), int(cnt.y));
        } else {
            const size_t sm = smem_pipe(PY);
            allow_smem(fft_xy_inv_pipe_k<PY>, sm);
            fft_xy_inv_pipe_k<PY><<<pipe_grid(planes, sm), THREADS, sm, st>>>(spec, cbuf, planes, int(step.x),
                                                                              int(cnt.x), int(step.y), int(cnt.y));
        }
    });
    launch_check("fft_xy_inv");
    inverse_z(st, p, imgs, step, cnt, out, out_img_stride, bias, bias_mod, act, cbuf, ph);
}

// z pass of an inverse: C2R of the compact kept planes in cbuf
void inverse_z(cudaStream_t st, const plan& p, int64_t imgs, dims3 step, dims3 cnt, float* out, int64_t out_img_stride,
               const float* bias, int bias_mod, int act, const float2* cbuf, const phase_geom* ph) {
    zinv_args g;
    g.phased = ph ? 1 : 0;
    g.ph = ph ? *ph : phase_geom{};
    g.xc = int(cnt.x), g.yc = int(cnt.y);
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
        if constexpr (PP >= 8 && PP <= 64) {
            if (!std::getenv("ZNN_FFT_Z_LINES")) {
                allow_smem(fft_z_inv_reg_k<PP>, zr_smem<PP>());
                fft_z_inv_reg_k<PP><<<unsigned(ceil_div(g.nlines, ZR_LINES)), ZR_THREADS, zr_smem<PP>(), st>>>(
                    cbuf, g, bias, out);
                return;
            }
        }
        allow_smem(fft_z_inv_k<PP>, smem_for(PP));
        fft_z_inv_k<PP><<<unsigned(ceil_div(g.nlines, LINES)), THREADS, smem_for(PP), st>>>(cbuf, g, bias, out);
    });
    launch_check("fft_z_inv");
}

// f_in = 1 fused paths need a square plane kernel with one plane buffer
bool fused1_ok(const plan& p, const conv_shape& c) {
    return c.f_in == 1 && p.P.x == p.P.y && p.P.x > 1 && p.P.x <= 96 && !std::getenv("ZNN_FFT_NOFUSE1");
}
size_t smem_plane1(int P) {
    return sizeof(float2) * (size_t(P) + size_t(LINES) * size_t(xpitch(P)) + size_t(P) * size_t(P + 2));
}

float2* carve(char*& cur, int64_t count) {
    float2* p = reinterpret_cast<float2*>(cur);
    cur += ((sizeof(float2) * size_t(count) + 255) / 256) * 256;
    return p;
}

}  // namespace

int64_t kernel_spectrum_bytes(const conv_shape& c) {
    const dims3 P = pads_for(c);
    return c.f_in * c.f_out * P.x * P.y * (P.z / 2 + 1) * int64_t(sizeof(float2));
}

int64_t image_spectrum_bytes(const conv_shape& c0) {
    const conv_shape c = effective(c0);
    const dims3 P = pads_for(c);
    return c.B * c.f_in * P.x * P.y * (P.z / 2 + 1) * int64_t(sizeof(float2));
}

// phase-split tensors of a polyphase plan: input side [B S f nr] and output side [B S f' mr]
int64_t split_bytes(const conv_shape& c0) {
    if (!use_poly(c0)) return 0;
    const conv_shape c = effective(c0);
    const int64_t a = c.B * c.f_in * c.n.vol(), b = c.B * c.f_out * c.m.vol();
    return ((int64_t(sizeof(float)) * (a + b) + 1024 + 4095) / 4096) * 4096;
}

// the CMACs run as per-bin tensor-core GEMMs when every kernel-spectrum bin
// is reused by enough images (polyphase plans: B s^3); ZNN_FFT_TC=0 keeps the
// register-tiled FMA kernels
// (square xy planes of at most 64: the row-bin-major transforms)
bool use_tc(const conv_shape& c0) {
    const char* e = std::getenv("ZNN_FFT_TC");
    if (e && std::string(e) == "0") return false;
    const conv_shape c = effective(c0);
    const dims3 P = pads_for_eff(c);
    const bool cube = P.x == P.z && P.x <= SMALLP && !std::getenv("ZNN_FFT_NO_CUBE");
    if (cube && (P.x > REGP || std::getenv("ZNN_FFT_CUBE_LINES"))) return false;
    return P.x == P.y && P.x > 1 && P.x <= 64 && znn_gpu::tc_cmac_supported(c.B, c.f_in, c.f_out);
}

// the engine arena of a plan: explicit phase split tensors
int64_t phase_bytes(const conv_shape& c0) { return split_bytes(c0); }

// the scratch-arena bytes conv_fwd / conv_bwd ask for (the larger of the two)
int64_t workspace_bytes(const conv_shape& c0) {
    const conv_shape c = effective(c0);
    const dims3 P = pads_for(c);
    const int64_t Zh = P.z / 2 + 1, bins = P.x * P.y * Zh, c8 = int64_t(sizeof(float2));
    const int64_t fwd = c8 * (c.B * c.f_out * bins + c.B * c.f_out * Zh * c.m.x * c.m.y) + 1024;
    const int64_t cc = std::max(c.B * c.f_in * Zh * c.n.x * c.n.y, c.f_out * c.f_in * Zh * c.k.x * c.k.y);
    const int64_t bwd = c8 * (c.B * c.f_out * bins + c.B * c.f_in * bins + cc) + 2048;
    return std::max(fwd, bwd);
}

bool supported(const conv_shape& c) {
    const dims3 P = pads_for(c);
    if (P.x > MAXP || P.y > MAXP || P.z > MAXP) return false;
    if ((P.x != P.y && P.x != 1) || P.y < 2) return false;  // compiled xy planes: square, or 2-D (x = 1)
    if (kernel_spectrum_bytes(c) > kMaxSpectrumBytes) return false;
    return true;
}

plan_ptr make_plan(const conv_shape& c0, std::shared_ptr<kpool> pool, std::shared_ptr<znn_gpu::scratch> phase_ws) {
    require(supported(c0), "fft engine: layer unsupported (pad > 128 or spectra exceed the memory budget)");
    const conv_shape c = effective(c0);
    plan_ptr p(new plan);
    if (use_poly(c0)) {
        p->poly = true;
        p->ce = c;
        p->S = c0.s.x * c0.s.y * c0.s.z;
    }
    p->tc = use_tc(c0);
    p->ph_bytes = split_bytes(c0);
    if (p->poly || p->tc) {
        p->phase_ws = phase_ws ? std::move(phase_ws) : std::make_shared<znn_gpu::scratch>();
        p->phase_ws->get(size_t(phase_bytes(c0)));  // sized now: a step never grows it
    }
    p->P = pads_for(c);
    p->Zh = p->P.z / 2 + 1;
    p->bins = p->P.x * p->P.y * p->Zh;
    p->B = c.B, p->f = c.f_in, p->fo = c.f_out;
    const dims3 e{c.s.x * (c.k.x - 1) + 1, c.s.y * (c.k.y - 1) + 1, c.s.z * (c.k.z - 1) + 1};
    znn_gpu::dmalloc(&p->X, sizeof(float2) * size_t(c.B * c.f_in * p->bins));
    p->pool = std::move(pool);
    if (!p->pool) znn_gpu::dmalloc(&p->K, sizeof(float2) * size_t(c.f_out * c.f_in * p->bins));
    (void)e;  // the dilated-kernel buffer is allocated on first use (dense-kernel path only)
    return p;
}

namespace {

// the kernel-spectrum buffer of a plan (own, or the shared pool's)
float2* kbuf(plan& p) {
    return p.pool ? p.pool->get(int64_t(sizeof(float2)) * p.f * p.fo * p.bins) : p.K;
}
bool k_current(const plan& p) { return p.pool ? p.pool->owner == &p : p.k_valid; }
void k_clobbered(plan& p) {
    if (p.pool) {
        if (p.pool->owner == &p) p.pool->owner = nullptr;
    } else {
        p.k_valid = false;
    }
}

// sparse-tap plane DFTs apply: square xy planes, <= KMAX taps per axis
bool sparse_taps(const plan& p, const conv_shape& c) {
    return p.P.x == p.P.y && p.P.x > 1 && c.k.x <= KMAX && c.k.y <= KMAX && c.k.z <= KMAX &&
           !std::getenv("ZNN_FFT_DENSE_KERNELS");
}

// kernel spectra of the dilated kernels into kbuf(p)
void kernel_spectra(cudaStream_t st, plan& p, const conv_shape& c, const float* w) {
    const dims3 e{c.s.x * (c.k.x - 1) + 1, c.s.y * (c.k.y - 1) + 1, c.s.z * (c.k.z - 1) + 1};
    const int64_t nker = c.f_out * c.f_in;
    float2* K = kbuf(p);
    if (sparse_taps(p, c)) {  // straight from the weights: one streaming write of K
        const int64_t planes = nker * p.Zh;
        dispatch_pad(int(p.P.y), [&](auto pc) {
            constexpr int PY = decltype(pc)::value;
            constexpr int G0 = ks_planes(PY);
            const int G = p.tc ? (G0 / 8) * 8 : G0;
            kspec_k<PY><<<unsigned(std::min<int64_t>((planes + G - 1) / G, 148 * 8)), KS_THREADS, 0, st>>>(
                w, planes, int(p.Zh), int(p.P.z), int(c.k.x), int(c.k.y), int(c.k.z), int(c.s.x), int(c.s.y),
                int(c.s.z), K, p.tc ? int(c.f_in) : 0);
        });
        launch_check("fft_kspec");
        if (p.pool)
            p.pool->owner = &p;
        else
            p.k_valid = true;
        return;
    }
    if (!p.dil) znn_gpu::dmalloc(&p.dil, sizeof(float) * size_t(nker * e.vol()));
    ZNN_CUDA_CHECK(cudaMemsetAsync(p.dil, 0, sizeof(float) * size_t(nker * e.vol()), st));
    const int64_t ntaps = nker * c.k.vol();
    dilate_k<<<unsigned(std::min<int64_t>(ceil_div(ntaps, 256), 148 * 16)), 256, 0, st>>>(
        w, ntaps, int(c.k.x), int(c.k.y), int(c.k.z), int(c.s.x), int(c.s.y), int(c.s.z), p.dil);
    launch_check("fft_dilate");
    forward3d(st, p, p.dil, e.vol(), e, nker, K, false, nullptr, nullptr, 1, nullptr, c.f_in);
    if (p.pool)
        p.pool->owner = &p;
    else
        p.k_valid = true;
}

}  // namespace

namespace {
std::string lbl(const char* k, const conv_shape& c, const plan& p) {
    return std::string(k) + " f=" + std::to_string(c.f_in) + "->" + std::to_string(c.f_out) + " B=" +
           std::to_string(c.B) + " P=" + std::to_string(p.P.y) + " bins=" + std::to_string(p.bins);
}
double cmac_bytes(const conv_shape& c, const plan& p) {
    return 8.0 * double(p.bins) * double(c.f_in * c.f_out + c.B * c.f_in + c.B * c.f_out);
}
double cmac_flops(const conv_shape& c, const plan& p) { return 8.0 * double(c.B * c.f_in * c.f_out) * double(p.bins); }
}  // namespace

static void conv_fwd_core(cudaStream_t st, plan& p, const conv_shape& c, const float* x, const float* w,
                          const float* bias, int act, float* y, znn_gpu::scratch& ws,
                          const phase_geom* ph_in = nullptr, const phase_geom* ph_out = nullptr) {
    require(p.B == c.B && p.f == c.f_in && p.fo == c.f_out, "fft engine: plan/layer mismatch");
    const int64_t nker = c.f_out * c.f_in;
    // image spectra (memoised for the backward / update passes)
    {
        znn_gpu::prof_scope ps(st, lbl("fft_image_fwd", c, p), double(c.B * c.f_in) * (4.0 * c.n.vol() + 8.0 * p.bins), 0);
        forward3d(st, p, x, c.n.vol(), c.n, c.B * c.f_in, p.X, false, nullptr, nullptr, 1, ph_in, c.f_in);
    }
    p.cnt.fwd_image += c.B * c.f_in;
    // kernel spectra of the dilated kernels (memoised for the backward pass)
    {
        znn_gpu::prof_scope ps(st, lbl("fft_kspec", c, p), 8.0 * double(nker) * double(p.bins), 0);
        kernel_spectra(st, p, c, w);
    }
    p.cnt.fwd_kernel += nker;
    const float2* K = kbuf(p);
    // Y = sum_i X * conj(K), one inverse per output node, crop + bias + transfer
    const int64_t ccount = c.B * c.f_out * p.Zh * c.m.x * c.m.y;  // compact kept planes
    if (fused1_ok(p, c)) {  // f_in = 1: Y = X * conj(K) formed inside the inverse xy pass
        float2* CB = static_cast<float2*>(ws.get(sizeof(float2) * size_t(ccount) + 256));
        const int64_t planes = c.B * c.f_out * p.Zh;
        dispatch_pad(int(p.P.y), [&](auto pc) {
            constexpr int PY = decltype(pc)::value;
            if constexpr (PY <= 96) {
                const size_t sm = smem_plane1(PY);
                allow_smem(fft_xy_inv_mul1_k<PY>, sm);
                fft_xy_inv_mul1_k<PY><<<pipe_grid(planes, sm), THREADS, sm, st>>>(
                    p.X, K, CB, planes, int(c.f_out), int(p.Zh), 1, int(c.m.x), 1, int(c.m.y));
            }
        });
        launch_check("fft_xy_inv_mul1");
        inverse_z(st, p, c.B * c.f_out, dims3{1, 1, 1}, c.m, y, c.m.vol(), bias, int(c.f_out), act, CB);
        p.cnt.fwd_inverse += c.B * c.f_out;
        return;
    }
    char* cur = static_cast<char*>(ws.get(sizeof(float2) * size_t(c.B * c.f_out * p.bins + ccount) + 1024));
    float2* Y = carve(cur, c.B * c.f_out * p.bins);
    float2* CB = carve(cur, ccount);
    {
        znn_gpu::prof_scope ps(st, lbl("fft_cmac_fwd", c, p), cmac_bytes(c, p), cmac_flops(c, p));
        if (p.tc)
            znn_gpu::tc_cmac_fwd(st, p.X, K, Y, c.B, c.f_in, c.f_out, p.bins);
        else
            cmac_ss(st, p.X, K, Y, int(c.B), int(c.f_in), int(c.f_out), int64_t(c.f_in), 1, p.bins, true);
    }
    launch_check("fft_cmac_fwd");
    {
        znn_gpu::prof_scope ps(st, lbl("fft_image_inv", c, p), double(c.B * c.f_out) * (8.0 * p.bins + 4.0 * c.m.vol()), 0);
        inverse3d(st, p, Y, c.B * c.f_out, dims3{1, 1, 1}, c.m, y, c.m.vol(), bias, int(c.f_out), act, CB, ph_out,
                  c.f_out);
    }
    p.cnt.fwd_inverse += c.B * c.f_out;
}

// kernel-gradient inverse: dK spectra -> gw[o][i] taps (scaled), sampled at s*w
void kernel_gradient_inverse(cudaStream_t st, const plan& p, const conv_shape& c, const float2* DK, float* gw,
                             float2* CB) {
    const int64_t nker = c.f_out * c.f_in;
    if (sparse_taps(p, c)) {
        const int64_t planes = nker * p.Zh;
        dispatch_pad(int(p.P.y), [&](auto pc) {
            constexpr int PY = decltype(pc)::value;
            constexpr int G0 = ks_planes(PY);
            const int G = p.tc ? (G0 / 8) * 8 : G0;
            const int64_t steps = (planes + G - 1) / G;
            dkinv_xy_k<PY><<<unsigned(std::min<int64_t>(steps, 148 * 8)), KS_THREADS, 0, st>>>(
                DK, planes, int(c.k.x), int(c.k.y), int(c.s.x), int(c.s.y), CB, int(p.Zh), p.tc ? int(c.f_in) : 0);
        });
        launch_check("fft_dkinv_xy");
        inverse_z(st, p, nker, c.s, c.k, gw, c.taps(), nullptr, 1, 3, CB);
        return;
    }
    inverse3d(st, p, DK, nker, c.s, c.k, gw, c.taps(), nullptr, 1, 3, CB, nullptr, c.f_in);
}

static void conv_bwd_core(cudaStream_t st, plan& p, const conv_shape& c, const float* g, const float* w, float* gw,
              float* gin, znn_gpu::scratch& ws, const float* relu_y, float* dbias,
              const phase_geom* ph_g = nullptr, const phase_geom* ph_dx = nullptr) {
    const int64_t nB = c.B;
    const int64_t ccount = std::max(nB * c.f_in * p.Zh * c.n.x * c.n.y, c.f_out * c.f_in * p.Zh * c.k.x * c.k.y);
    const size_t need = sizeof(float2) * size_t(nB * c.f_out * p.bins + (gin ? nB * c.f_in * p.bins : 0) + ccount) +
                        2048;
    char* cur = static_cast<char*>(ws.get(need));
    float2* G = carve(cur, nB * c.f_out * p.bins);
    float2* DX = gin ? carve(cur, nB * c.f_in * p.bins) : nullptr;
    float2* CB = carve(cur, ccount);
    // the data gradient needs this layer's kernel spectra: recompute them if a
    // layer sharing the buffer overwrote them after this layer's forward
    if (gin && !k_current(p)) {
        kernel_spectra(st, p, c, w);
        p.cnt.bwd_kernel += c.f_out * c.f_in;
    }
    const float2* K = kbuf(p);
    // dK (product spectra of the update) reuse the kernel-spectrum buffer
    float2* DK = kbuf(p);
    // backward image spectra, padded to the tail dims (engine.hpp:757-759)
    if (!gin && fused1_ok(p, c)) {
        // f_in = 1, no input gradient: the xy pass of every G[b][o] feeds
        // dK[o] = sum_b X[b] * conj(G[b][o]) directly (G never reaches HBM)
        forward3d(st, p, g, c.m.vol(), c.m, nB * c.f_out, G, /*z_only=*/true, relu_y, dbias, c.f_out);
        p.cnt.bwd_image += nB * c.f_out;
        const int64_t planes = c.f_out * p.Zh;
        dispatch_pad(int(p.P.y), [&](auto pc) {
            constexpr int PY = decltype(pc)::value;
            if constexpr (PY <= 96) {
                const size_t sm = smem_plane1(PY);
                allow_smem(fft_xy_fwd_upd1_k<PY>, sm);
                fft_xy_fwd_upd1_k<PY><<<pipe_grid(planes, sm), THREADS, sm, st>>>(
                    G, p.X, DK, planes, int(nB), int(c.f_out), int(p.Zh), int(c.m.x), int(c.m.y));
            }
        });
        launch_check("fft_xy_fwd_upd1");
        k_clobbered(p);
        kernel_gradient_inverse(st, p, c, DK, gw, CB);
        p.cnt.upd_inverse += c.f_out * c.f_in;
        return;
    }
    {
        znn_gpu::prof_scope ps(st, lbl("fft_grad_fwd", c, p), double(nB * c.f_out) * (4.0 * c.m.vol() + 8.0 * p.bins), 0);
        forward3d(st, p, g, c.m.vol(), c.m, nB * c.f_out, G, false, relu_y, dbias, c.f_out, ph_g, c.f_out);
    }
    p.cnt.bwd_image += nB * c.f_out;
    if (gin) {
        {
            znn_gpu::prof_scope ps(st, lbl("fft_cmac_dgrad", c, p), cmac_bytes(c, p), cmac_flops(c, p));
            if (p.tc)
                znn_gpu::tc_cmac_dgrad(st, G, K, DX, nB, c.f_in, c.f_out, p.bins);
            else
                cmac_ss(st, G, K, DX, int(nB), int(c.f_out), int(c.f_in), 1, int64_t(c.f_in), p.bins, false);
        }
        launch_check("fft_cmac_bwd");
        {
            znn_gpu::prof_scope ps(st, lbl("fft_dgrad_inv", c, p), double(nB * c.f_in) * (8.0 * p.bins + 4.0 * c.n.vol()), 0);
            inverse3d(st, p, DX, nB * c.f_in, dims3{1, 1, 1}, c.n, gin, c.n.vol(), nullptr, 1, 3, CB, ph_dx, c.f_in);
        }
        p.cnt.bwd_inverse += nB * c.f_in;
    }
    // kernel gradient: one gradient-specific inverse per edge, sampled at s*w
    {
        znn_gpu::prof_scope ps(st, lbl("fft_cmac_upd", c, p), cmac_bytes(c, p), cmac_flops(c, p));
        if (p.tc)
            znn_gpu::tc_cmac_upd(st, p.X, G, DK, nB, c.f_in, c.f_out, p.bins);
        else
            cmac_upd(st, p.X, G, DK, int(nB), int(c.f_in), int(c.f_out), p.bins);
    }
    launch_check("fft_cmac_upd");
    k_clobbered(p);
    {
        znn_gpu::prof_scope ps(st, lbl("fft_dkinv", c, p), 8.0 * double(c.f_out * c.f_in) * double(p.bins), 0);
        kernel_gradient_inverse(st, p, c, DK, gw, CB);
    }
    p.cnt.upd_inverse += c.f_out * c.f_in;
}

namespace {

// space-to-batch: x [B][f][n] -> xp [B][S][f][nr] with xp[(b S + r) f + i][q] =
// x[b][i][s q + r] (r = (rx sy + ry) sz + rz), optionally gated by a ReLU
// output (g * (y > 0), the fused transfer backward). Block = 8 z-lines
// (threadIdx.y) of one (image, x); lanes walk z: coalesced 128-byte reads,
// each store instruction fills sz phase lines with runs of 32 / sz floats.
// All index math is 32-bit except the two line bases. Voxels of a ragged
// phase beyond its valid length are never written (the caller zero-fills).
__global__ void __launch_bounds__(256) phase_split_k(const float* __restrict__ x, const float* __restrict__ gate,
                                                     phase_geom G, float* __restrict__ xp) {
    const int yy = blockIdx.x * 8 + threadIdx.y;
    if (yy >= G.ny) return;
    const int xx = blockIdx.y, img = blockIdx.z;
    const int b = img / G.f, i = img - b * G.f;
    const int qx = xx / G.sx, rx = xx - qx * G.sx, qy = yy / G.sy, ry = yy - qy * G.sy;
    const int S = G.sx * G.sy * G.sz;
    const int64_t src = ((int64_t(img) * G.nx + xx) * G.ny + yy) * G.nz;
    const int rb = (b * S + (rx * G.sy + ry) * G.sz) * G.f + i;  // phase image of rz = 0
    const int64_t pl = int64_t(G.nrx) * G.nry * G.nrz;            // phase image volume
    const int64_t dst0 = (int64_t(qx) * G.nry + qy) * G.nrz;
    for (int z = threadIdx.x; z < G.nz; z += 32) {
        float v = __ldcs(x + src + z);
        if (gate && !(__ldcs(gate + src + z) > 0.f)) v = 0.f;
        int qz, rz;
        zsplit(z, G.sz, G.zsh, qz, rz);
        xp[int64_t(rb + rz * G.f) * pl + dst0 + qz] = v;
    }
}

// batch-to-space: yp [B][S][f][mr] -> y [B][f][m], y[b][o][s q + r] =
// yp[(b S + r) f + o][q]; same block shape, coalesced stores.
__global__ void __launch_bounds__(256) phase_merge_k(const float* __restrict__ yp, phase_geom G,
                                                     float* __restrict__ y) {
    const int yy = blockIdx.x * 8 + threadIdx.y;
    if (yy >= G.ny) return;
    const int xx = blockIdx.y, img = blockIdx.z;
    const int b = img / G.f, o = img - b * G.f;
    const int qx = xx / G.sx, rx = xx - qx * G.sx, qy = yy / G.sy, ry = yy - qy * G.sy;
    const int S = G.sx * G.sy * G.sz;
    const int64_t dst = ((int64_t(img) * G.nx + xx) * G.ny + yy) * G.nz;
    const int rb = (b * S + (rx * G.sy + ry) * G.sz) * G.f + o;
    const int64_t pl = int64_t(G.nrx) * G.nry * G.nrz;
    const int64_t src0 = (int64_t(qx) * G.nry + qy) * G.nrz;
    for (int z = threadIdx.x; z < G.nz; z += 32) {
        int qz, rz;
        zsplit(z, G.sz, G.zsh, qz, rz);
        __stcs(y + dst + z, __ldcs(yp + int64_t(rb + rz * G.f) * pl + src0 + qz));
    }
}

phase_geom geom(const conv_shape& c, int64_t maps, dims3 n, dims3 nr) {
    phase_geom G;
    G.f = int(maps), G.nx = int(n.x), G.ny = int(n.y), G.nz = int(n.z);
    G.sx = int(c.s.x), G.sy = int(c.s.y), G.sz = int(c.s.z);
    G.zsh = -1;
    for (int k = 0; k < 8; ++k)
        if ((1 << k) == G.sz) G.zsh = k;
    G.nrx = int(nr.x), G.nry = int(nr.y), G.nrz = int(nr.z);
    return G;
}

void phase_split(cudaStream_t st, const plan& p, const conv_shape& c, const float* x, const float* gate, int64_t maps,
                 dims3 n, dims3 nr, float* xp) {
    const bool ragged = nr.x * c.s.x != n.x || nr.y * c.s.y != n.y || nr.z * c.s.z != n.z;
    if (ragged)  // phases shorter than nr: the missing voxels are the zero padding
        ZNN_CUDA_CHECK(cudaMemsetAsync(xp, 0, sizeof(float) * size_t(c.B * p.S * maps * nr.vol()), st));
    require(c.B * maps < 65536 && n.x < 65536, "fft phase split: grid exceeds 65535");
    const dim3 grid(unsigned(ceil_div(n.y, 8)), unsigned(n.x), unsigned(c.B * maps));
    phase_split_k<<<grid, dim3(32, 8, 1), 0, st>>>(x, gate, geom(c, maps, n, nr), xp);
    launch_check("fft_phase_split");
}

void phase_merge(cudaStream_t st, const conv_shape& c, const float* yp, int64_t maps, dims3 m, dims3 mr, float* y) {
    require(c.B * maps < 65536 && m.x < 65536, "fft phase merge: grid exceeds 65535");
    const dim3 grid(unsigned(ceil_div(m.y, 8)), unsigned(m.x), unsigned(c.B * maps));
    phase_merge_k<<<grid, dim3(32, 8, 1), 0, st>>>(yp, geom(c, maps, m, mr), y);
    launch_check("fft_phase_merge");
}

}  // namespace

// A dilated layer's tensors may be phase-major ([B s^3][maps][n / s], the
// dense images of the polyphase plan) instead of the natural [B][maps][n]:
// a convolution with sparsity s maps phase r of its input to phase r of its
// output, so a chain of FFT layers with one sparsity never needs the
// interleaved order in between (the executor decides, net.cpp)
bool phase_major_ok(const conv_shape& c) {
    if (!use_poly(c) || c.f_in == 1 || std::getenv("ZNN_FFT_PHASE_SPLIT")) return false;
    return c.n.x % c.s.x == 0 && c.n.y % c.s.y == 0 && c.n.z % c.s.z == 0 && c.m.x % c.s.x == 0 &&
           c.m.y % c.s.y == 0 && c.m.z % c.s.z == 0;
}

// phase-major input pays off for a producer that has to scatter into it (the
// max-filters) only where the strided in-place phase reads are the bound: the
// fused small-cube transforms (the z passes at larger pads already read whole
// sectors by pairing the z-phases of a line)
bool phase_major_pays(const conv_shape& c) {
    if (!phase_major_ok(c)) return false;
    const dims3 P = pads_for(c);
    return P.x == P.y && P.y == P.z && P.x > 1 && P.x <= REGP;
}

void conv_fwd(cudaStream_t st, plan& p, const conv_shape& c, const float* x, const float* w, const float* bias,
              int act, float* y, znn_gpu::scratch& ws, bool x_pm, bool y_pm) {
    require(p.B == c.B * p.S && p.f == c.f_in && p.fo == c.f_out, "fft engine: plan/layer mismatch");
    require((!x_pm && !y_pm) || (p.poly && phase_major_ok(c)), "fft engine: phase-major tensors need a polyphase plan");
    if (!p.poly) {
        conv_fwd_core(st, p, c, x, w, bias, act, y, ws);
        return;
    }
    const conv_shape& e = p.ce;
    // phases read / written in place by the transforms (no split / merge
    // pass); ZNN_FFT_PHASE_SPLIT=1 keeps the explicit split / merge kernels
    if (!fused1_ok(p, e) && !std::getenv("ZNN_FFT_PHASE_SPLIT")) {
        const phase_geom gi = geom(c, c.f_in, c.n, e.n), go = geom(c, c.f_out, c.m, e.m);
        conv_fwd_core(st, p, e, x, w, bias, act, y, ws, x_pm ? nullptr : &gi, y_pm ? nullptr : &go);
        return;
    }
    float* xp = static_cast<float*>(p.phase_ws->get(size_t(p.ph_bytes)));
    float* yp = xp + ((e.B * e.f_in * e.n.vol() + 63) / 64) * 64;
    {
        znn_gpu::prof_scope ps(st, lbl("fft_phase_split", c, p), 8.0 * double(c.B * c.f_in * c.n.vol()), 0);
        phase_split(st, p, c, x, nullptr, c.f_in, c.n, e.n, xp);
    }
    conv_fwd_core(st, p, e, xp, w, bias, act, yp, ws);  // bias + transfer per output map: phase-invariant
    znn_gpu::prof_scope ps(st, lbl("fft_phase_merge", c, p), 8.0 * double(c.B * c.f_out * c.m.vol()), 0);
    phase_merge(st, c, yp, c.f_out, c.m, e.m, y);
}

void conv_bwd(cudaStream_t st, plan& p, const conv_shape& c, const float*, const float* g, const float* w, float* gw,
              float* gin, znn_gpu::scratch& ws, const float* relu_y, float* dbias, bool x_pm, bool y_pm) {
    require((!x_pm && !y_pm) || (p.poly && phase_major_ok(c)), "fft engine: phase-major tensors need a polyphase plan");
    if (!p.poly) {
        conv_bwd_core(st, p, c, g, w, gw, gin, ws, relu_y, dbias);
        return;
    }
    const conv_shape& e = p.ce;
    if (!fused1_ok(p, e) && !std::getenv("ZNN_FFT_PHASE_SPLIT")) {
        // g and the gate relu_y share the output tensor's order, gin the input's
        const phase_geom gg = geom(c, c.f_out, c.m, e.m), gx = geom(c, c.f_in, c.n, e.n);
        conv_bwd_core(st, p, e, g, w, gw, gin, ws, relu_y, dbias, y_pm ? nullptr : &gg, x_pm ? nullptr : &gx);
        return;
    }
    float* dxp = static_cast<float*>(p.phase_ws->get(size_t(p.ph_bytes)));
    float* gp = dxp + ((e.B * e.f_in * e.n.vol() + 63) / 64) * 64;
    {
        // the gradient's phases, gated by the fused ReLU (its bias gradient is
        // then the DC term of the gated phases' spectra, summed over B s^3)
        znn_gpu::prof_scope ps(st, lbl("fft_phase_split", c, p),
                               (relu_y ? 12.0 : 8.0) * double(c.B * c.f_out * c.m.vol()), 0);
        phase_split(st, p, c, g, relu_y, c.f_out, c.m, e.m, gp);
    }
    conv_bwd_core(st, p, e, gp, w, gw, gin ? dxp : nullptr, ws, nullptr, dbias);
    if (gin) {
        znn_gpu::prof_scope ps(st, lbl("fft_phase_merge", c, p), 8.0 * double(c.B * c.f_in * c.n.vol()), 0);
        phase_merge(st, c, dxp, c.f_in, c.n, e.n, gin);
    }
}

float time_cmac(cudaStream_t st, int which, const conv_shape& c0, int reps, int64_t* bins_out) {
    require(which >= 0 && which <= 2 && reps > 0, "fft cmac probe: bad arguments");
    require(supported(c0), "fft cmac probe: layer unsupported by the FFT engine");
    const conv_shape c = effective(c0);  // dilated layers: the phase images of the polyphase plan
    const dims3 P = pads_for(c);
    const int64_t bins = P.x * P.y * (P.z / 2 + 1), B = c.B, f = c.f_in, fo = c.f_out;
    if (bins_out) *bins_out = bins;
    float2 *X = nullptr, *G = nullptr, *K = nullptr;
    ZNN_CUDA_CHECK(cudaMalloc(&X, sizeof(float2) * size_t(B * f * bins)));
    ZNN_CUDA_CHECK(cudaMalloc(&G, sizeof(float2) * size_t(B * fo * bins)));
    ZNN_CUDA_CHECK(cudaMalloc(&K, sizeof(float2) * size_t(f * fo * bins)));
    // small finite values (0x3c3c3c3c = 0.0115f); the FMA rate is value-independent
    ZNN_CUDA_CHECK(cudaMemsetAsync(X, 0x3c, sizeof(float2) * size_t(B * f * bins), st));
    ZNN_CUDA_CHECK(cudaMemsetAsync(G, 0x3c, sizeof(float2) * size_t(B * fo * bins), st));
    ZNN_CUDA_CHECK(cudaMemsetAsync(K, 0x3c, sizeof(float2) * size_t(f * fo * bins), st));
    auto launch = [&] {
        if (which == 0) {
            cmac_ss(st, X, K, G, int(B), int(f), int(fo), f, 1, bins, true);
        } else if (which == 1) {
            cmac_ss(st, G, K, X, int(B), int(fo), int(f), 1, f, bins, false);
        } else {
            cmac_upd(st, X, G, K, int(B), int(f), int(fo), bins);
        }
        launch_check("fft_cmac_probe");
    };
    launch();
    cudaEvent_t a, b;
    ZNN_CUDA_CHECK(cudaEventCreate(&a));
    ZNN_CUDA_CHECK(cudaEventCreate(&b));
    ZNN_CUDA_CHECK(cudaEventRecord(a, st));
    for (int r = 0; r < reps; ++r) launch();
    ZNN_CUDA_CHECK(cudaEventRecord(b, st));
    ZNN_CUDA_CHECK(cudaEventSynchronize(b));
    float ms = 0.f;
    ZNN_CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(X);
    cudaFree(G);
    cudaFree(K);
    return ms / float(reps);
}

namespace {
// FP32 FMA issue-rate probe: 16 independent chains per thread of the form the
// CMACs issue, d = a * b + c with all three operands in registers (runtime
// values, so no immediate form: 3-register FFMA issues at ~2/3 the rate of
// the immediate form on this GPU, 49.5 vs 71.9 TFLOP/s in tests/micro/mma_rate.cu)
__global__ void fma_probe_k(float* out, const float* __restrict__ in, int iters) {
    float x[16], y[4], z[4];
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = threadIdx.x * 1e-3f + j;
#pragma unroll
    for (int j = 0; j < 4; ++j) y[j] = in[j], z[j] = in[4 + j];
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 16; ++j) x[j] = fmaf(x[j], y[j & 3], z[(j >> 2) & 3]);
    }
    float sum = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) sum += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = sum;
}
}  // namespace

float fma_peak_tflops(cudaStream_t st) {
    int sms = 0, dev = 0;
    ZNN_CUDA_CHECK(cudaGetDevice(&dev));
    ZNN_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int blocks = sms * 2, threads = 1024, iters = 20000;
    float* out = nullptr;
    ZNN_CUDA_CHECK(cudaMalloc(&out, sizeof(float) * (size_t(blocks) * threads + 8)));
    float* in = out + size_t(blocks) * threads;
    const float h[8] = {0.9999f, 0.9998f, 0.9997f, 0.9996f, 1e-4f, 2e-4f, 3e-4f, 4e-4f};
    ZNN_CUDA_CHECK(cudaMemcpyAsync(in, h, sizeof(h), cudaMemcpyHostToDevice, st));
    fma_probe_k<<<blocks, threads, 0, st>>>(out, in, 100);
    cudaEvent_t a, b;
    ZNN_CUDA_CHECK(cudaEventCreate(&a));
    ZNN_CUDA_CHECK(cudaEventCreate(&b));
    ZNN_CUDA_CHECK(cudaEventRecord(a, st));
    fma_probe_k<<<blocks, threads, 0, st>>>(out, in, iters);
    ZNN_CUDA_CHECK(cudaEventRecord(b, st));
    ZNN_CUDA_CHECK(cudaEventSynchronize(b));
    float ms = 0.f;
    ZNN_CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    return float(2.0 * 16.0 * double(iters) * blocks * threads / (double(ms) * 1e-3) / 1e12);
}

}  // namespace znn_fft

