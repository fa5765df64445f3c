// Direct 3D valid (dilated) convolution, SIMT fp32 implicit GEMM.
//
// This is the exact-fp32 engine used for layers the tensor-core kernel does
// not cover (tiny channel counts, e.g. the 1^3 -> 3 output layers) and as the
// ZNN_CONV_DIRECT_SIMT reference engine. The convergent-edge sum of the
// reference (engine.hpp:345-353) is the GEMM K-loop: each output voxel's
// accumulator runs over (input map, tap) in registers; no atomics, no locks.
//
//   fwd   : y[b,o,v]   = act(bias[o] + sum_{i,w} W[o,i,w] x[b,i,v + s*w])      (conv_direct.hpp:39-68)
//   dgrad : dx[b,i,t]  = sum_{o,w} W[o,i,w] g[b,o,t - s*w]  (g zero outside)   (conv_direct.hpp:74-101 w/ reflect)
//   wgrad : dW[o,i,w]  = scale * sum_{b,v} g[b,o,v] x[b,i,v + s*w]             (conv_direct.hpp:108-132)
//
// 64x64 output tile per 256-thread block, 4x4 register micro-tile, BK = 16.
#include "ops.hpp"

namespace znn_gpu {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

struct geom {
    int nx, ny, nz;  // input (tail) dims
    int mx, my, mz;  // output (head) dims
    int kx, ky, kz;
    int sx, sy, sz;
};

__device__ __forceinline__ void tap_decode(const geom& g, int t, int& wx, int& wy, int& wz) {
    const int kyz = g.ky * g.kz;
    wx = t / kyz;
    const int r = t - wx * kyz;
    wy = r / g.kz;
    wz = r - wy * g.kz;
}

__device__ __forceinline__ void mma_tile(const float (&As)[BK][BM], const float (&Bs)[BK][BN],
                                         int ty, int tx, float (&acc)[4][4]) {
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
        const float4 a = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
        const float4 b = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
        const float av[4] = {a.x, a.y, a.z, a.w};
        const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
}

__global__ void __launch_bounds__(NT) conv_fwd_k(const float* __restrict__ x,
                                                 const float* __restrict__ w,
                                                 const float* __restrict__ bias, int act,
                                                 float* __restrict__ y, int f_in, int f_out,
                                                 geom g) {
    __shared__ __align__(16) float As[BK][BM];
    __shared__ __align__(16) float Bs[BK][BN];
    const int64_t mvol = int64_t(g.mx) * g.my * g.mz;
    const int64_t nvol = int64_t(g.nx) * g.ny * g.nz;
    const int T = g.kx * g.ky * g.kz;
    const int K = f_in * T;
    const int b = blockIdx.z;
    const int co0 = blockIdx.y * BM;
    const int64_t v0 = int64_t(blockIdx.x) * BN;
    const int tid = threadIdx.x;

    const int lv = tid % BN, lk = tid / BN;
    const int64_t vox = v0 + lv;
    const bool vok = vox < mvol;
    int64_t base = 0;
    if (vok) {
        const int ox = int(vox / (int64_t(g.my) * g.mz));
        const int oy = int((vox / g.mz) % g.my);
        const int oz = int(vox % g.mz);
        base = (int64_t(ox) * g.ny + oy) * g.nz + oz;
    }
    const int la_co = tid / 4, la_k = (tid % 4) * 4;
    const float* xb = x + int64_t(b) * f_in * nvol;

    float acc[4][4] = {};
    const int ty = tid / 16, tx = tid % 16;
    for (int k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int k = k0 + la_k + i;
            const int co = co0 + la_co;
            As[la_k + i][la_co] = (k < K && co < f_out) ? w[int64_t(co) * K + k] : 0.f;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int kk = lk * 4 + i;
            const int k = k0 + kk;
            float val = 0.f;
            if (k < K && vok) {
                const int ci = k / T;
                int wx, wy, wz;
                tap_decode(g, k - ci * T, wx, wy, wz);
                val = xb[int64_t(ci) * nvol + base +
                         (int64_t(g.sx * wx) * g.ny + g.sy * wy) * g.nz + g.sz * wz];
            }
            Bs[kk][lv] = val;
        }
        __syncthreads();
        mma_tile(As, Bs, ty, tx, acc);
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int co = co0 + ty * 4 + i;
        if (co >= f_out) continue;
        const float bv = bias ? bias[co] : 0.f;
        float* yr = y + (int64_t(b) * f_out + co) * mvol;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t v = v0 + tx * 4 + j;
            if (v < mvol) yr[v] = act_value(act, acc[i][j] + bv);
        }
    }
}

__global__ void __launch_bounds__(NT) conv_dgrad_k(const float* __restrict__ gr,
                                                   const float* __restrict__ w,
                                                   float* __restrict__ dx, int f_in, int f_out,
                                                   geom g) {
    __shared__ __align__(16) float As[BK][BM];
    __shared__ __align__(16) float Bs[BK][BN];
    const int64_t mvol = int64_t(g.mx) * g.my * g.mz;
    const int64_t nvol = int64_t(g.nx) * g.ny * g.nz;
    const int T = g.kx * g.ky * g.kz;
    const int K = f_out * T;
    const int b = blockIdx.z;
    const int ci0 = blockIdx.y * BM;
    const int64_t t0 = int64_t(blockIdx.x) * BN;
    const int tid = threadIdx.x;

    const int lv = tid % BN, lk = tid / BN;
    const int64_t tv = t0 + lv;
    const bool tok = tv < nvol;
    int tx_ = 0, ty_ = 0, tz_ = 0;
    if (tok) {
        tx_ = int(tv / (int64_t(g.ny) * g.nz));
        ty_ = int((tv / g.nz) % g.ny);
        tz_ = int(tv % g.nz);
    }
    const int la_ci = tid / 4, la_k = (tid % 4) * 4;
    const float* gb = gr + int64_t(b) * f_out * mvol;

    float acc[4][4] = {};
    const int ty = tid / 16, tx = tid % 16;
    for (int k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int k = k0 + la_k + i;
            const int ci = ci0 + la_ci;
            float val = 0.f;
            if (k < K && ci < f_in) {
                const int co = k / T;
                val = w[(int64_t(co) * f_in + ci) * T + (k - co * T)];
            }
            As[la_k + i][la_ci] = val;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int kk = lk * 4 + i;
            const int k = k0 + kk;
            float val = 0.f;
            if (k < K && tok) {
                const int co = k / T;
                int wx, wy, wz;
                tap_decode(g, k - co * T, wx, wy, wz);
                const int gx = tx_ - g.sx * wx, gy = ty_ - g.sy * wy, gz = tz_ - g.sz * wz;
                if (gx >= 0 && gx < g.mx && gy >= 0 && gy < g.my && gz >= 0 && gz < g.mz)
                    val = gb[int64_t(co) * mvol + (int64_t(gx) * g.my + gy) * g.mz + gz];
            }
            Bs[kk][lv] = val;
        }
        __syncthreads();
        mma_tile(As, Bs, ty, tx, acc);
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int ci = ci0 + ty * 4 + i;
        if (ci >= f_in) continue;
        float* dr = dx + (int64_t(b) * f_in + ci) * nvol;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t t = t0 + tx * 4 + j;
            if (t < nvol) dr[t] = acc[i][j];
        }
    }
}

// Split-K over output voxels: block z = b * splits + split. Partial tiles go
// to ws[z][f_out][f_in*T]; a fixed-order reduction sums them (deterministic).
__global__ void __launch_bounds__(NT) conv_wgrad_k(const float* __restrict__ x,
                                                   const float* __restrict__ gr,
                                                   float* __restrict__ ws, int f_in, int f_out,
                                                   geom g, int splits, int64_t chunk) {
    __shared__ __align__(16) float As[BK][BM];
    __shared__ __align__(16) float Bs[BK][BN];
    const int64_t mvol = int64_t(g.mx) * g.my * g.mz;
    const int64_t nvol = int64_t(g.nx) * g.ny * g.nz;
    const int T = g.kx * g.ky * g.kz;
    const int N = f_in * T;
    const int b = blockIdx.z / splits;
    const int sp = blockIdx.z - b * splits;
    const int64_t kb = int64_t(sp) * chunk;
    const int64_t ke = min(mvol, kb + chunk);
    const int co0 = blockIdx.y * BM;
    const int n0 = blockIdx.x * BN;
    const int tid = threadIdx.x;

    const int lk = tid % BK, lg = tid / BK;  // 16 groups x 4 columns
    int64_t noff[4];
    bool nok[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int n = n0 + lg * 4 + i;
        nok[i] = n < N;
        noff[i] = 0;
        if (nok[i]) {
            const int ci = n / T;
            int wx, wy, wz;
            tap_decode(g, n - ci * T, wx, wy, wz);
            noff[i] = int64_t(ci) * nvol + (int64_t(g.sx * wx) * g.ny + g.sy * wy) * g.nz +
                      g.sz * wz;
        }
    }
    const float* xb = x + int64_t(b) * f_in * nvol;
    const float* gb = gr + int64_t(b) * f_out * mvol;

    float acc[4][4] = {};
    const int ty = tid / 16, tx = tid % 16;
    for (int64_t k0 = kb; k0 < ke; k0 += BK) {
        const int64_t o = k0 + lk;
        const bool ook = o < ke;
        int64_t base = 0;
        if (ook) {
            const int ox = int(o / (int64_t(g.my) * g.mz));
            const int oy = int((o / g.mz) % g.my);
            const int oz = int(o % g.mz);
            base = (int64_t(ox) * g.ny + oy) * g.nz + oz;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int co = co0 + lg * 4 + i;
            As[lk][lg * 4 + i] = (ook && co < f_out) ? gb[int64_t(co) * mvol + o] : 0.f;
            Bs[lk][lg * 4 + i] = (ook && nok[i]) ? xb[noff[i] + base] : 0.f;
        }
        __syncthreads();
        mma_tile(As, Bs, ty, tx, acc);
        __syncthreads();
    }
    float* wsz = ws + int64_t(blockIdx.z) * f_out * N;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int co = co0 + ty * 4 + i;
        if (co >= f_out) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + tx * 4 + j;
            if (n < N) wsz[int64_t(co) * N + n] = acc[i][j];
        }
    }
}

__global__ void sum_partials_k(const float* __restrict__ ws, int64_t parts, int64_t len,
                               float scale, float* __restrict__ out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < len;
         i += int64_t(gridDim.x) * blockDim.x) {
        float acc = 0.f;
        for (int64_t p = 0; p < parts; ++p) acc += ws[p * len + i];
        out[i] = scale * acc;
    }
}

geom make_geom(const conv_shape& c) {
    geom g;
    g.nx = int(c.n.x), g.ny = int(c.n.y), g.nz = int(c.n.z);
    g.mx = int(c.m.x), g.my = int(c.m.y), g.mz = int(c.m.z);
    g.kx = int(c.k.x), g.ky = int(c.k.y), g.kz = int(c.k.z);
    g.sx = int(c.s.x), g.sy = int(c.s.y), g.sz = int(c.s.z);
    return g;
}

}  // namespace

conv_shape conv_shape::make(int64_t B, int64_t f_in, int64_t f_out, dims3 n, dims3 k, dims3 s) {
    conv_shape c;
    c.B = B, c.f_in = f_in, c.f_out = f_out, c.n = n, c.k = k, c.s = s;
    require(B > 0 && f_in > 0 && f_out > 0, "conv: batch and map counts must be positive");
    require(k.x > 0 && k.y > 0 && k.z > 0 && s.x > 0 && s.y > 0 && s.z > 0,
            "conv: kernel and sparsity must be positive");
    c.m = dims3{n.x - s.x * (k.x - 1), n.y - s.y * (k.y - 1), n.z - s.z * (k.z - 1)};
    require(c.m.x > 0 && c.m.y > 0 && c.m.z > 0,
            "conv_valid_direct: effective window exceeds image");
    require(f_in * k.vol() < (int64_t(1) << 31) && n.vol() < (int64_t(1) << 31),
            "conv: layer too large for 32-bit tap indexing");
    return c;
}

void conv_fwd_simt(cudaStream_t st, const conv_shape& c, const float* x, const float* w,
                   const float* bias, int act, float* y) {
    const dim3 grid(unsigned(ceil_div(c.m.vol(), BN)), unsigned(ceil_div(c.f_out, BM)),
                    unsigned(c.B));
    conv_fwd_k<<<grid, NT, 0, st>>>(x, w, bias, act, y, int(c.f_in), int(c.f_out),
                                    make_geom(c));
    launch_check("conv_fwd_simt");
}

void conv_dgrad_simt(cudaStream_t st, const conv_shape& c, const float* g, const float* w,
                     float* dx) {
    const dim3 grid(unsigned(ceil_div(c.n.vol(), BN)), unsigned(ceil_div(c.f_in, BM)),
                    unsigned(c.B));
    conv_dgrad_k<<<grid, NT, 0, st>>>(g, w, dx, int(c.f_in), int(c.f_out), make_geom(c));
    launch_check("conv_dgrad_simt");
}

void conv_wgrad_simt(cudaStream_t st, const conv_shape& c, const float* x, const float* g,
                     float* dw, float scale, scratch& ws) {
    const int64_t N = c.f_in * c.taps();
    const int64_t tiles = ceil_div(N, BN) * ceil_div(c.f_out, BM) * c.B;
    const int64_t mvol = c.m.vol();
    int64_t splits = ceil_div(148 * 4, tiles);
    const int64_t max_splits = ceil_div(mvol, 1024);
    if (splits > max_splits) splits = max_splits;
    if (splits < 1) splits = 1;
    const int64_t chunk = ceil_div(ceil_div(mvol, splits), BK) * BK;
    splits = ceil_div(mvol, chunk);
    const int64_t parts = c.B * splits;
    const int64_t len = c.f_out * N;
    float* part = static_cast<float*>(ws.get(sizeof(float) * size_t(parts * len)));
    const dim3 grid(unsigned(ceil_div(N, BN)), unsigned(ceil_div(c.f_out, BM)), unsigned(parts));
    conv_wgrad_k<<<grid, NT, 0, st>>>(x, g, part, int(c.f_in), int(c.f_out), make_geom(c),
                                      int(splits), chunk);
    launch_check("conv_wgrad_simt");
    int64_t rb = ceil_div(len, 256);
    if (rb > 148 * 8) rb = 148 * 8;
    sum_partials_k<<<unsigned(rb), 256, 0, st>>>(part, parts, len, scale, dw);
    launch_check("conv_wgrad_reduce");
}

}  // namespace znn_gpu
