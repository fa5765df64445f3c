// Max-pooling and dense (dilated) max-filtering with argmax masks
// (maxops.hpp:32-182). HBM-bound; a thread per output voxel forward and per
// input voxel backward (gather formulation: deterministic, no atomics).
// Mask = int32 flat index into the per-map input volume (the reference's
// record), or, for the executor's internal max-filters, a one-byte window
// code (a ky + b) kz + c: a quarter of the mask traffic (HBM-bound passes).
//
// Tie rule: the reference resolves ties to the lexicographically smallest
// (x,y,z) source, i.e. the lowest flat index (maxops.hpp:79-82 strict '>'
// scan; maxops.hpp:106-110 for the separable filter). A direct window scan
// in lexicographic order with strict '>' selects the same source, so masks
// are bit-identical on identical inputs.
#include <algorithm>
#include <cstdlib>
#include <string>

#include "ops.hpp"

namespace znn_gpu {

namespace {

// Volume grid (no per-element index division): a block is 32 z-lanes x 8
// y-rows of one x-plane of one map; blockIdx = (y tile, x, map). A thread
// walks its row along z in steps of 32 (coalesced along the contiguous axis).
constexpr int ZL = 32, YR = 8;
inline dim3 vgrid(int64_t y, int64_t x, int64_t maps) {
    require(x < 65536 && maps < 65536, "maxops: volume grid exceeds 65535 planes / maps");
    return dim3(unsigned(ceil_div(y, YR)), unsigned(x), unsigned(maps));
}
inline dim3 vblock() { return dim3(ZL, YR, 1); }

// phase-major addressing of an output volume [maps = B f][mx][my][mz] stored
// as [B S][f][mx / sx][my / sy][mz / sz] (ops.hpp pm_order)
struct pm_dev {
    int on, f, sx, sy, sz, zsh;
    int qy, qz;        // phase image dims (y, z)
    int64_t qvol;      // voxels of one phase image
};
// offset of row (i, j) of map `map`, z-phase 0, q = 0; voxel l of the row is at
// + (l & (sz - 1)) * f * qvol + (l >> zsh)
__device__ __forceinline__ int64_t pm_row(const pm_dev& P, int64_t map, int i, int j) {
    const int64_t b = map / P.f, c = map - b * P.f;
    const int rx = i % P.sx, ry = j % P.sy;
    const int64_t img = (b * (P.sx * P.sy * P.sz) + (rx * P.sy + ry) * P.sz) * P.f + c;
    return img * P.qvol + (int64_t(i / P.sx) * P.qy + j / P.sy) * P.qz;
}

// KX/KY/KZ > 0: compile-time window (fully unrolled, the common 2^3 and
// 1x2x2 filters); 0: runtime window.
// gate (window codes only): a window whose maximum is not > 0 gets code bit 7
// set, so the backward passes no gradient through it: the ReLU backward of
// the layer feeding the filter (ReLU'(0) = 0, transfer.hpp:99-106), folded in
// exactly because the argmax voxel holds the window's maximum
template <int KX, int KY, int KZ, typename M, bool PM = false>
__global__ void __launch_bounds__(ZL * YR) maxfilter_fwd_k(const float* __restrict__ x, int nx, int ny, int nz,
                                                           int mx, int my, int mz, int kx_, int ky_, int kz_, int sx,
                                                           int sy, int sz, float* __restrict__ y,
                                                           M* __restrict__ mask, int gate, pm_dev pm) {
    constexpr bool CODE = sizeof(M) == 1;
    const int kx = KX ? KX : kx_, ky = KY ? KY : ky_, kz = KZ ? KZ : kz_;
    const int j = blockIdx.x * YR + threadIdx.y, i = blockIdx.y;
    if (j >= my) return;
    const int64_t map = blockIdx.z;
    const float* xm = x + map * (int64_t(nx) * ny * nz);
    const int64_t orow = map * (int64_t(mx) * my * mz) + (int64_t(i) * my + j) * mz;
    // phase-major output: voxel l of the row goes to its z-phase's image; a
    // thread's voxels l = lane + 32 t share one z-phase (sz divides 32), so it
    // keeps one pointer into that image, advanced 32 / sz per step
    float* ypm = nullptr;
    int ypm_step = 0;
    if constexpr (PM) {
        ypm = y + pm_row(pm, map, i, j) + int64_t(threadIdx.x & (pm.sz - 1)) * pm.f * pm.qvol + (threadIdx.x >> pm.zsh);
        ypm_step = ZL >> pm.zsh;
    }
    auto put = [&](float* yr_, int l, float v) {
        if constexpr (PM) {
            __stcs(ypm, v);
            ypm += ypm_step;
        } else {
            __stcs(yr_ + l, v);
        }
    };
    const int dx = sx * ny * nz, dy = sy * nz;
    const int rbase = (i * ny + j) * nz;
    const float* xr = xm + rbase;
    float* yr = y + orow;
    M* mr = mask + orow;
    if constexpr (KX > 0) {
        // one 64-bit pointer per window row (a, b), advanced along z: the
        // loads need no per-element 64-bit index arithmetic
        const float* q[KX][KY];
#pragma unroll
        for (int a = 0; a < KX; ++a)
#pragma unroll
            for (int b = 0; b < KY; ++b) q[a][b] = xr + a * dx + b * dy + threadIdx.x;
        for (int l = threadIdx.x; l < mz; l += ZL) {
            float v[KX][KY][KZ];
#pragma unroll
            for (int a = 0; a < KX; ++a)
#pragma unroll
                for (int b = 0; b < KY; ++b)
#pragma unroll
                    for (int c = 0; c < KZ; ++c) v[a][b][c] = __ldg(q[a][b] + c * sz);
            float best = v[0][0][0];
            int best_off = 0, best_code = 0;
#pragma unroll
            for (int a = 0; a < KX; ++a)
#pragma unroll
                for (int b = 0; b < KY; ++b)
#pragma unroll
                    for (int c = 0; c < KZ; ++c)
                        if (v[a][b][c] > best) {  // strict: ties keep the lexicographically first source
                            best = v[a][b][c];
                            best_off = a * dx + b * dy + c * sz;
                            best_code = (a * KY + b) * KZ + c;
                        }
            put(yr, l, best);
            if constexpr (CODE)
                mr[l] = M(best_code | ((gate && !(best > 0.f)) ? 0x80 : 0));
            else
                __stcs(mr + l, M(rbase + l + best_off));
#pragma unroll
            for (int a = 0; a < KX; ++a)
#pragma unroll
                for (int b = 0; b < KY; ++b) q[a][b] += ZL;
        }
    } else {
        for (int l = threadIdx.x; l < mz; l += ZL) {
            const int base = rbase + l;
            int best_idx = base, best_code = 0;
            float best = __ldg(xm + base);
            for (int a = 0; a < kx; ++a)
                for (int b = 0; b < ky; ++b)
                    for (int c = 0; c < kz; ++c) {
                        const int idx = base + a * dx + b * dy + c * sz;
                        const float v = __ldg(xm + idx);
                        if (v > best) {  // strict: ties keep the lexicographically first source
                            best = v;
                            best_idx = idx;
                            best_code = (a * ky + b) * kz + c;
                        }
                    }
            put(yr, l, best);
            if constexpr (CODE)
                mr[l] = M(best_code | ((gate && !(best > 0.f)) ? 0x80 : 0));
            else
                __stcs(mr + l, M(best_idx));
        }
    }
}

// Forward of the 2^3 max-filter with one-byte codes and x-stride SX (1 or 2):
// a thread owns one (y, z) column of the output and walks its x-planes; input
// plane i + SX's four window-row values are loaded once and serve output
// planes i (a = 1) and i + SX (a = 0): half the loads of maxfilter_fwd_k.
// Block = whole z rows (up to 128 lanes) x y-rows, grid = (y tiles, maps).
// Same scan order (a, b, c) and strict '>' as maxfilter_fwd_k: same codes.
template <int SX, bool PM>
__global__ void __launch_bounds__(ZL * YR) maxfilter2_fwd_k(const float* __restrict__ x, int nx, int ny, int nz, int mx,
                                                            int my, int mz, int sy, int sz, float* __restrict__ y,
                                                            uint8_t* __restrict__ code, int gate, pm_dev pm) {
    const int j = blockIdx.x * blockDim.y + threadIdx.y;
    if (j >= my) return;
    const int64_t map = blockIdx.y;
    const int64_t pin = int64_t(ny) * nz, pout = int64_t(my) * mz;
    const float* xm = x + map * (pin * nx);
    const int64_t pxs = PM ? int64_t(pm.sy) * pm.sz * pm.f * pm.qvol : 0;
    const int64_t pwrap = PM ? int64_t(pm.qy) * pm.qz - (pm.sx - 1) * pxs : 0;
    for (int l = threadIdx.x; l < mz; l += blockDim.x) {
        const float* xp = xm + j * nz + l;  // window row (b, c) of a plane at xp + b sy nz + c sz
        const int o01 = sz, o10 = sy * nz, o11 = sy * nz + sz;
        constexpr int D = SX == 1 ? 2 : 1;  // planes loaded ahead of use (measured: n = 91 5.2 -> 4.9 ms with 2; the x-stride-2 ring gets too wide)
        float v[SX + 1 + D][4];  // planes i .. i + SX + D
#pragma unroll
        for (int k = 0; k < SX + D; ++k) {
            if (k < nx) {
                v[k][0] = __ldg(xp), v[k][1] = __ldg(xp + o01), v[k][2] = __ldg(xp + o10), v[k][3] = __ldg(xp + o11);
                xp += pin;
            }
        }
        uint8_t* cp = code + map * (pout * mx) + j * mz + l;
        float* yp;
        int rxp = 0;
        if constexpr (PM)
            yp = y + pm_row(pm, map, 0, j) + int64_t(l & (pm.sz - 1)) * pm.f * pm.qvol + (l >> pm.zsh);
        else
            yp = y + map * (pout * mx) + j * mz + l;
        for (int i = 0; i < mx; ++i) {
            if (i + SX + D < nx) {
                v[SX + D][0] = __ldg(xp), v[SX + D][1] = __ldg(xp + o01), v[SX + D][2] = __ldg(xp + o10),
                          v[SX + D][3] = __ldg(xp + o11);
                xp += pin;
            }
            float best = v[0][0];
            int bc = 0;
#pragma unroll
            for (int q = 1; q < 4; ++q)
                if (v[0][q] > best) best = v[0][q], bc = q;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (v[SX][q] > best) best = v[SX][q], bc = 4 + q;
            __stcs(yp, best);
            *cp = uint8_t(bc | ((gate && !(best > 0.f)) ? 0x80 : 0));
            cp += pout;
            if constexpr (PM) {
                if (++rxp == pm.sx) rxp = 0, yp += pwrap;
                else yp += pxs;
            } else {
                yp += pout;
            }
#pragma unroll
            for (int k = 0; k < SX + D; ++k)
#pragma unroll
                for (int q = 0; q < 4; ++q) v[k][q] = v[k + 1][q];
        }
    }
}

// dx[t] = sum over windows o whose argmax is t of g[o]; windows visited in
// ascending flat order of o, the order the reference accumulates in
// (maxops.hpp:176-181), so fp32 sums match it bit for bit.
template <int KX, int KY, int KZ, typename M>
__global__ void __launch_bounds__(ZL * YR) maxfilter_bwd_k(const float* __restrict__ g,
                                                           const M* __restrict__ mask, int nx, int ny, int nz,
                                                           int mx, int my, int mz, int kx_, int ky_, int kz_, int sx,
                                                           int sy, int sz, float* __restrict__ dx) {
    constexpr bool CODE = sizeof(M) == 1;
    const int kx = KX ? KX : kx_, ky = KY ? KY : ky_, kz = KZ ? KZ : kz_;
    const int tj = blockIdx.x * YR + threadIdx.y, ti = blockIdx.y;
    if (tj >= ny) return;
    const int64_t map = blockIdx.z;
    const int64_t mv = int64_t(mx) * my * mz;
    const float* gm = g + map * mv;
    const M* mm = mask + map * mv;
    float* drow = dx + map * (int64_t(nx) * ny * nz) + (int64_t(ti) * ny + tj) * nz;
    // rows whose every window origin t - s*w is inside the output volume skip
    // the per-window bounds tests (the common case away from the faces)
    const bool row_in = ti >= sx * (kx - 1) && ti < mx && tj >= sy * (ky - 1) && tj < my;
    for (int tl = threadIdx.x; tl < nz; tl += ZL) {
        const int tr = (ti * ny + tj) * nz + tl;
        float acc = 0.f;
        if (KX && row_in && tl >= sz * (kz - 1) && tl < mz) {
            const int o0 = (ti * my + tj) * mz + tl;
#pragma unroll
            for (int a = kx - 1; a >= 0; --a)
#pragma unroll
                for (int b = ky - 1; b >= 0; --b)
#pragma unroll
                    for (int c = kz - 1; c >= 0; --c) {
                        // both loads issued together: no mask -> g dependent round trip
                        const int o = o0 - (sx * a * my + sy * b) * mz - sz * c;
                        const int mv = int(__ldg(mm + o));
                        const float gv = __ldg(gm + o);
                        acc += (mv == (CODE ? (a * ky + b) * kz + c : tr)) ? gv : 0.f;
                    }
            __stcs(drow + tl, acc);
            continue;
        }
#pragma unroll
        for (int a = kx - 1; a >= 0; --a) {
            const int oi = ti - sx * a;
            if (oi < 0 || oi >= mx) continue;
#pragma unroll
            for (int b = ky - 1; b >= 0; --b) {
                const int oj = tj - sy * b;
                if (oj < 0 || oj >= my) continue;
#pragma unroll
                for (int c = kz - 1; c >= 0; --c) {
                    const int ol = tl - sz * c;
                    if (ol < 0 || ol >= mz) continue;
                    const int o = (oi * my + oj) * mz + ol;
                    if (int(__ldg(mm + o)) == (CODE ? (a * ky + b) * kz + c : tr)) acc += __ldg(gm + o);
                }
            }
        }
        __stcs(drow + tl, acc);
    }
}

// Backward of the 2^3 max-filter with x-stride SX (1 or 2): a thread owns one
// (y, z) column of the input and walks its x-planes; output plane oi's
// window-row (mask, g) pairs are loaded once (one plane ahead of use) and
// serve input planes oi and oi + SX, half the loads of maxfilter_bwd_k.
// Block = 32 z-lanes x 8 y-rows, grid = (y tiles, maps). Sums in ascending
// window order like maxfilter_bwd_k.
template <int SX, typename M, bool PM, bool SUM>
__device__ __forceinline__ void maxfilter2_bwd_body(const float* __restrict__ g, const M* __restrict__ mask, int nx,
                                                    int ny, int nz, int mx, int my, int mz, int sy, int sz,
                                                    float* __restrict__ dx, pm_dev pm, float* __restrict__ part,
                                                    int part_f) {
    constexpr bool CODE = sizeof(M) == 1;
    const int tj = blockIdx.x * blockDim.y + threadIdx.y;
    const int64_t map = blockIdx.y;
    // part: per-warp partial sums of dx in fixed order, part[(c * B + b) * cols + blockIdx.x * warps + warp]
    // with map = b f + c (a warp is one z-row segment: its lanes share tj and leave together)
    const int nwarp = (blockDim.x * blockDim.y) >> 5, warp = (threadIdx.y * blockDim.x + threadIdx.x) >> 5;
    float* pslot = nullptr;
    if (SUM && part) {
        const int64_t b = map / part_f, c = map - b * part_f, B = gridDim.y / part_f;
        pslot = part + (c * B + b) * (int64_t(gridDim.x) * nwarp) + blockIdx.x * nwarp + warp;
    }
    if (tj >= ny) {
        if (pslot && (threadIdx.x & 31) == 0) *pslot = 0.f;
        return;
    }
    float tsum = 0.f;
    const int64_t pin = int64_t(ny) * nz, pout = int64_t(my) * mz;
    // phase-major gradient: plane oi of map (b, c) starts at gpm0 + (oi % sx) * pxs + (oi / sx) * qy * qz,
    // its voxel (oj, ol) at + goff[q]
    const float* gm = PM ? g + pm_row(pm, map, 0, 0) : g + map * (pout * mx);
    // plane oi -> oi + 1: the next x-phase's images, or back to x-phase 0 one phase-image plane on
    const int64_t pxs = PM ? int64_t(pm.sy) * pm.sz * pm.f * pm.qvol : 0;
    const int64_t pwrap = PM ? int64_t(pm.qy) * pm.qz - (pm.sx - 1) * pxs : 0;
    const M* mm = mask + map * (pout * mx);
    float* dm = dx + map * (pin * nx);
    for (int tl = threadIdx.x; tl < nz; tl += blockDim.x) {
        // window rows (b, c) in descending order = ascending output index
        int roff[4];
        int goff[4];
        bool rok[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int b = 1 - (q >> 1), c = 1 - (q & 1);
            const int oj = tj - sy * b, ol = tl - sz * c;
            rok[q] = oj >= 0 && oj < my && ol >= 0 && ol < mz;
            roff[q] = rok[q] ? oj * mz + ol : 0;
            goff[q] = roff[q];
            if (PM && rok[q])
                goff[q] = ((oj % pm.sy) * pm.sz + (ol & (pm.sz - 1))) * pm.f * int(pm.qvol) + (oj / pm.sy) * pm.qz +
                          (ol >> pm.zsh);
        }
        // ring[k]: (mask, g) of output plane ti - SX + k, k <= SX + D (the
        // last D are the next iterations' planes, loaded ahead of use)
        constexpr int D = 1;  // (two planes ahead measured slower here: 5.2 vs 4.6 ms at n = 91)
        int rm[SX + 1 + D][4];
        float rg[SX + 1 + D][4];
#pragma unroll
        for (int k = 0; k < SX; ++k)
#pragma unroll
            for (int q = 0; q < 4; ++q) rm[k][q] = -1, rg[k][q] = 0.f;
        const M* mp = mm;
        const float* gp = gm;
        int rxp = 0;  // x-phase of the plane gp points at
        auto fetch = [&](int oi, int slot) {
            const bool pok = oi < mx;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const bool ok = pok && rok[q];
                rm[slot][q] = ok ? int(__ldg(mp + roff[q])) : -1;
                rg[slot][q] = ok ? __ldg(gp + goff[q]) : 0.f;
            }
            mp += pout;
            if constexpr (PM) {
                if (++rxp == pm.sx) rxp = 0, gp += pwrap;
                else gp += pxs;
            } else {
                gp += pout;
            }
        };
#pragma unroll
        for (int k = 0; k < D; ++k) fetch(k, SX + k);
        float* dp = dm + tj * nz + tl;
        int tr = tj * nz + tl;
        for (int ti = 0; ti < nx; ++ti) {
            fetch(ti + D, SX + D);
            float acc = 0.f;
            // window (a, b, c) with b = 1 - (q >> 1), c = 1 - (q & 1): code (2 a + b) 2 + c
#pragma unroll
            for (int q = 0; q < 4; ++q)  // a = 1: plane ti - SX
                acc += (rm[0][q] == (CODE ? 4 + 2 * (1 - (q >> 1)) + (1 - (q & 1)) : tr)) ? rg[0][q] : 0.f;
#pragma unroll
            for (int q = 0; q < 4; ++q)  // a = 0: plane ti
                acc += (rm[SX][q] == (CODE ? 2 * (1 - (q >> 1)) + (1 - (q & 1)) : tr)) ? rg[SX][q] : 0.f;
            __stcs(dp, acc);
            if constexpr (SUM) tsum += acc;
            dp += pin;
            tr += int(pin);
#pragma unroll
            for (int k = 0; k < SX + D; ++k)
#pragma unroll
                for (int q = 0; q < 4; ++q) rm[k][q] = rm[k + 1][q], rg[k][q] = rg[k + 1][q];
        }
    }
    if (SUM && pslot) {
        for (int o = 16; o > 0; o >>= 1) tsum += __shfl_xor_sync(0xffffffffu, tsum, o);
        if ((threadIdx.x & 31) == 0) *pslot = tsum;
    }
}
template <int SX, typename M, bool PM = false>
__global__ void __launch_bounds__(ZL * YR) maxfilter2_bwd_k(const float* __restrict__ g, const M* __restrict__ mask,
                                                            int nx, int ny, int nz, int mx, int my, int mz, int sy,
                                                            int sz, float* __restrict__ dx, pm_dev pm) {
    maxfilter2_bwd_body<SX, M, PM, false>(g, mask, nx, ny, nz, mx, my, mz, sy, sz, dx, pm, nullptr, 1);
}
// + per-warp partial sums of dx (64 registers: four blocks per SM as the plain kernel)
template <int SX, typename M>
__global__ void __launch_bounds__(ZL * YR, 4) maxfilter2_bwd_sum_k(const float* __restrict__ g,
                                                                   const M* __restrict__ mask, int nx, int ny, int nz,
                                                                   int mx, int my, int mz, int sy, int sz,
                                                                   float* __restrict__ dx, float* __restrict__ part,
                                                                   int part_f) {
    maxfilter2_bwd_body<SX, M, false, true>(g, mask, nx, ny, nz, mx, my, mz, sy, sz, dx, pm_dev{}, part, part_f);
}

__global__ void __launch_bounds__(ZL * YR) maxpool_fwd_k(const float* __restrict__ x, int nx, int ny, int nz, int px,
                                                         int py, int pz, float* __restrict__ y,
                                                         int32_t* __restrict__ mask) {
    const int mx = nx / px, my = ny / py, mz = nz / pz;
    const int bj = blockIdx.x * YR + threadIdx.y, bi = blockIdx.y;
    if (bj >= my) return;
    const int64_t map = blockIdx.z;
    const float* xm = x + map * (int64_t(nx) * ny * nz);
    const int64_t orow = map * (int64_t(mx) * my * mz) + (int64_t(bi) * my + bj) * mz;
    for (int bl = threadIdx.x; bl < mz; bl += ZL) {
        const int base = ((bi * px) * ny + bj * py) * nz + bl * pz;
        int best_idx = base;
        float best = __ldg(xm + base);
        for (int a = 0; a < px; ++a)
            for (int b = 0; b < py; ++b)
                for (int c = 0; c < pz; ++c) {
                    const int idx = base + (a * ny + b) * nz + c;
                    const float v = __ldg(xm + idx);
                    if (v > best) {
                        best = v;
                        best_idx = idx;
                    }
                }
        y[orow + bl] = best;
        mask[orow + bl] = best_idx;
    }
}

__global__ void __launch_bounds__(ZL * YR) maxpool_bwd_k(const float* __restrict__ g, const int32_t* __restrict__ mask,
                                                         int mx, int my, int mz, int px, int py, int pz,
                                                         float* __restrict__ dx) {
    const int nx = mx * px, ny = my * py, nz = mz * pz;
    const int tj = blockIdx.x * YR + threadIdx.y, ti = blockIdx.y;
    if (tj >= ny) return;
    const int64_t map = blockIdx.z;
    const int64_t mv = int64_t(mx) * my * mz;
    const int64_t orow = map * mv + (int64_t(ti / px) * my + (tj / py)) * mz;
    float* drow = dx + map * (int64_t(nx) * ny * nz) + (int64_t(ti) * ny + tj) * nz;
    for (int tl = threadIdx.x; tl < nz; tl += ZL) {
        const int tr = (ti * ny + tj) * nz + tl;
        const int64_t o = orow + tl / pz;
        drow[tl] = (__ldg(mask + o) == tr) ? __ldg(g + o) : 0.f;
    }
}

}  // namespace

namespace {
pm_dev pm_device(const pm_order& pm, int64_t maps, dims3 m) {
    pm_dev d{};
    if (!pm.on) return d;
    int zsh = -1;
    for (int b = 0; b < 8; ++b)
        if ((int64_t(1) << b) == pm.s.z) zsh = b;
    require(zsh >= 0 && pm.f > 0 && maps % pm.f == 0 && m.x % pm.s.x == 0 && m.y % pm.s.y == 0 && m.z % pm.s.z == 0,
            "maxfilter: phase-major order needs dims divisible by the sparsity (power-of-two along z)");
    d.on = 1, d.f = pm.f, d.sx = int(pm.s.x), d.sy = int(pm.s.y), d.sz = int(pm.s.z), d.zsh = zsh;
    d.qy = int(m.y / pm.s.y), d.qz = int(m.z / pm.s.z);
    d.qvol = (m.x / pm.s.x) * int64_t(d.qy) * d.qz;
    require(pm.s.vol() * pm.f * d.qvol < (int64_t(1) << 31), "maxfilter: phase-major patch exceeds the int32 offset range");
    return d;
}

template <typename M>
void maxfilter_fwd_t(cudaStream_t st, const float* x, int64_t maps, dims3 n, dims3 k, dims3 s, float* y, M* mask,
                     int gate = 0, pm_order pm = {}) {
    const dims3 m{n.x - s.x * (k.x - 1), n.y - s.y * (k.y - 1), n.z - s.z * (k.z - 1)};
    require(m.x > 0 && m.y > 0 && m.z > 0, "maxfilter_forward: effective window exceeds input");
    prof_scope ps(st, "maxfilter_fwd n=" + std::to_string(n.x) + " maps=" + std::to_string(maps),
                  double(maps) * (4.0 * double(n.vol()) + (4.0 + sizeof(M)) * double(m.vol())), 0);
    require(n.vol() < (int64_t(1) << 31), "maxfilter_forward: map exceeds int32 mask range");
    require(sizeof(M) == 4 || k.vol() <= (gate ? 128 : 256), "maxfilter_forward: window too large for one-byte codes");
    const pm_dev pd = pm_device(pm, maps, m);
    require(!pm.on || (k.x == 2 && k.y == 2 && k.z == 2 && ZL % pm.s.z == 0),
            "maxfilter_forward: phase-major output is written by the 2^3 kernel only");
    if constexpr (sizeof(M) == 1) {
        // one-byte codes, 2^3 window: the x-walking kernel (ZNN_MAXFILTER_WALK=0: a thread per output voxel)
        const char* e = std::getenv("ZNN_MAXFILTER_WALK");
        if (k.x == 2 && k.y == 2 && k.z == 2 && (s.x == 1 || s.x == 2) && maps < 65536 && m.x > s.x &&
            !(e && std::string(e) == "0")) {
            const unsigned bx = unsigned(std::min<int64_t>(4, ceil_div(m.z, ZL))) * ZL, by = (ZL * YR) / bx;
            const dim3 grid(unsigned(ceil_div(m.y, int64_t(by))), unsigned(maps));
            auto* kw = pm.on ? (s.x == 1 ? maxfilter2_fwd_k<1, true> : maxfilter2_fwd_k<2, true>)
                             : (s.x == 1 ? maxfilter2_fwd_k<1, false> : maxfilter2_fwd_k<2, false>);
            kw<<<grid, dim3(bx, by, 1), 0, st>>>(x, int(n.x), int(n.y), int(n.z), int(m.x), int(m.y), int(m.z), int(s.y),
                                                 int(s.z), y, mask, gate, pd);
            launch_check("maxfilter_fwd");
            return;
        }
    }
    auto* kf = pm.on                                ? maxfilter_fwd_k<2, 2, 2, M, true>
               : (k.x == 2 && k.y == 2 && k.z == 2) ? maxfilter_fwd_k<2, 2, 2, M>
               : (k.x == 1 && k.y == 2 && k.z == 2) ? maxfilter_fwd_k<1, 2, 2, M>
                                                    : maxfilter_fwd_k<0, 0, 0, M>;
    kf<<<vgrid(m.y, m.x, maps), vblock(), 0, st>>>(x, int(n.x), int(n.y), int(n.z), int(m.x), int(m.y), int(m.z),
                                                  int(k.x), int(k.y), int(k.z), int(s.x), int(s.y), int(s.z), y,
                                                  mask, gate, pd);
    launch_check("maxfilter_fwd");
}

}  // namespace
int64_t maxfilter_bwd_sum_cols(dims3 m, dims3 k, dims3 s);
namespace {
template <typename M>
void maxfilter_bwd_t(cudaStream_t st, const float* g, const M* mask, int64_t maps, dims3 m, dims3 k, dims3 s,
                     float* dx, pm_order pm = {}, float* part = nullptr, int part_f = 1) {
    const dims3 n{m.x + s.x * (k.x - 1), m.y + s.y * (k.y - 1), m.z + s.z * (k.z - 1)};
    prof_scope ps(st, "maxfilter_bwd n=" + std::to_string(n.x) + " maps=" + std::to_string(maps),
                  double(maps) * ((4.0 + sizeof(M)) * double(m.vol()) + 4.0 * double(n.vol())), 0);
    if (k.x == 2 && k.y == 2 && k.z == 2 && (s.x == 1 || s.x == 2) && maps < 65536) {
        // a block spans whole z rows (up to 128 lanes) so one walk along x reads
        // every sector of a gradient / code plane once: with 32-lane blocks the
        // three z chunks of a 91-voxel row walked the planes one after another
        // and re-read the sectors they share from DRAM (2.6x the read traffic)
        const unsigned bx = unsigned(std::min<int64_t>(4, ceil_div(n.z, ZL))) * ZL, by = (ZL * YR) / bx;
        const dim3 grid(unsigned(ceil_div(n.y, int64_t(by))), unsigned(maps));
        require(!part || (part_f > 0 && maps % part_f == 0 &&
                          int64_t(grid.x) * ((bx * by) / 32) == maxfilter_bwd_sum_cols(m, k, s)),
                "maxfilter_backward: bias partials need maps = B f");
        require(!part || !pm.on, "maxfilter_backward: bias partials come with natural-order gradients only");
        if (part) {
            auto* ks = s.x == 1 ? maxfilter2_bwd_sum_k<1, M> : maxfilter2_bwd_sum_k<2, M>;
            ks<<<grid, dim3(bx, by, 1), 0, st>>>(g, mask, int(n.x), int(n.y), int(n.z), int(m.x), int(m.y), int(m.z),
                                                 int(s.y), int(s.z), dx, part, part_f);
            launch_check("maxfilter_bwd");
            return;
        }
        auto* kk = pm.on ? (s.x == 1 ? maxfilter2_bwd_k<1, M, true> : maxfilter2_bwd_k<2, M, true>)
                         : (s.x == 1 ? maxfilter2_bwd_k<1, M> : maxfilter2_bwd_k<2, M>);
        kk<<<grid, dim3(bx, by, 1), 0, st>>>(g, mask, int(n.x), int(n.y), int(n.z), int(m.x), int(m.y), int(m.z),
                                             int(s.y), int(s.z), dx, pm_device(pm, maps, m));
        launch_check("maxfilter_bwd");
        return;
    }
    require(!pm.on && !part, "maxfilter_backward: phase-major gradients / bias partials need the 2^3 kernel");
    auto* kb = (k.x == 2 && k.y == 2 && k.z == 2)   ? maxfilter_bwd_k<2, 2, 2, M>
               : (k.x == 1 && k.y == 2 && k.z == 2) ? maxfilter_bwd_k<1, 2, 2, M>
                                                    : maxfilter_bwd_k<0, 0, 0, M>;
    kb<<<vgrid(n.y, n.x, maps), vblock(), 0, st>>>(g, mask, int(n.x), int(n.y), int(n.z), int(m.x), int(m.y),
                                                  int(m.z), int(k.x), int(k.y), int(k.z), int(s.x), int(s.y),
                                                  int(s.z), dx);
    launch_check("maxfilter_bwd");
}
}  // namespace

void maxfilter_fwd(cudaStream_t st, const float* x, int64_t maps, dims3 n, dims3 k, dims3 s, float* y,
                   int32_t* mask) {
    maxfilter_fwd_t(st, x, maps, n, k, s, y, mask);
}
void maxfilter_fwd(cudaStream_t st, const float* x, int64_t maps, dims3 n, dims3 k, dims3 s, float* y,
                   uint8_t* code, bool relu_gate, pm_order pm) {
    maxfilter_fwd_t(st, x, maps, n, k, s, y, code, relu_gate ? 1 : 0, pm);
}
void maxfilter_bwd(cudaStream_t st, const float* g, const int32_t* mask, int64_t maps, dims3 m, dims3 k, dims3 s,
                   float* dx) {
    maxfilter_bwd_t(st, g, mask, maps, m, k, s, dx);
}
void maxfilter_bwd(cudaStream_t st, const float* g, const uint8_t* code, int64_t maps, dims3 m, dims3 k, dims3 s,
                   float* dx, pm_order pm, float* sum_part, int sum_f) {
    maxfilter_bwd_t(st, g, code, maps, m, k, s, dx, pm, sum_part, sum_f);
}

int64_t maxfilter_bwd_sum_cols(dims3 m, dims3 k, dims3 s) {
    if (!(k.x == 2 && k.y == 2 && k.z == 2 && (s.x == 1 || s.x == 2))) return 0;
    const dims3 n{m.x + s.x, m.y + s.y, m.z + s.z};
    const int64_t bx = std::min<int64_t>(4, ceil_div(n.z, ZL)) * ZL, by = (ZL * YR) / bx;
    return ceil_div(n.y, by) * ((bx * by) / 32);  // y tiles x warps per block
}

void maxpool_fwd(cudaStream_t st, const float* x, int64_t maps, dims3 n, dims3 p, float* y,
                 int32_t* mask) {
    require(p.x > 0 && p.y > 0 && p.z > 0 && n.x % p.x == 0 && n.y % p.y == 0 && n.z % p.z == 0,
            "maxpool_forward: dims not divisible by window");
    const dims3 m{n.x / p.x, n.y / p.y, n.z / p.z};
    maxpool_fwd_k<<<vgrid(m.y, m.x, maps), vblock(), 0, st>>>(x, int(n.x), int(n.y), int(n.z), int(p.x), int(p.y),
                                                             int(p.z), y, mask);
    launch_check("maxpool_fwd");
}

void maxpool_bwd(cudaStream_t st, const float* g, const int32_t* mask, int64_t maps, dims3 m,
                 dims3 p, float* dx) {
    maxpool_bwd_k<<<vgrid(m.y * p.y, m.x * p.x, maps), vblock(), 0, st>>>(g, mask, int(m.x), int(m.y), int(m.z),
                                                                         int(p.x), int(p.y), int(p.z), dx);
    launch_check("maxpool_bwd");
}

}  // namespace znn_gpu
