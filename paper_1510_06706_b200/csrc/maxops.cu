// Max-pooling and dense (dilated) max-filtering with argmax masks
// (maxops.hpp:32-182). HBM-bound; one thread per output voxel forward, one
// thread per input voxel backward (gather formulation: deterministic, no
// atomics). Mask = int32 flat index into the per-map input volume.
//
// Tie rule: the reference resolves ties to the lexicographically smallest
// (x,y,z) source, i.e. the lowest flat index (maxops.hpp:79-82 strict '>'
// scan; maxops.hpp:106-110 for the separable filter). A direct window scan
// in lexicographic order with strict '>' selects the same source, so masks
// are bit-identical on identical inputs.
#include "ops.hpp"

namespace znn_gpu {

namespace {

constexpr int kThreads = 256;

// Grid: x covers the voxels of one map (32-bit index math only — 64-bit
// division per voxel made these kernels issue-bound at ~15% of HBM), y the
// maps.
inline dim3 grid2(int64_t per_map, int64_t maps) {
    const int64_t gx = ceil_div(per_map, kThreads);
    const int64_t gy = maps < 65535 ? (maps < 1 ? 1 : maps) : 65535;
    return dim3(unsigned(gx < 1 ? 1 : gx), unsigned(gy), unsigned(ceil_div(maps < 1 ? 1 : maps, gy)));
}
// map of this block (y, z fold the map count past 65535): no per-thread loop,
// whose 64-bit trip-count division cost more than the voxel's work
__device__ __forceinline__ int64_t block_map() { return blockIdx.y + int64_t(blockIdx.z) * gridDim.y; }

// KX/KY/KZ > 0: compile-time window (fully unrolled, the common 2^3 and
// 1x2x2 filters); 0: runtime window.
template <int KX, int KY, int KZ>
__global__ void __launch_bounds__(kThreads) maxfilter_fwd_k(const float* __restrict__ x, int64_t maps, int nx, int ny,
                                                            int nz, int mx, int my, int mz, int kx_, int ky_, int kz_,
                                                            int sx, int sy, int sz, float* __restrict__ y,
                                                            int32_t* __restrict__ mask) {
    const int kx = KX ? KX : kx_, ky = KY ? KY : ky_, kz = KZ ? KZ : kz_;
    const unsigned mv = unsigned(mx) * unsigned(my) * unsigned(mz);
    const unsigned r = blockIdx.x * kThreads + threadIdx.x;
    if (r >= mv) return;
    const unsigned myz = unsigned(my) * unsigned(mz);
    const int i = int(r / myz);
    const unsigned r2 = r - unsigned(i) * myz;
    const int j = int(r2 / unsigned(mz));
    const int l = int(r2 - unsigned(j) * unsigned(mz));
    const int base = (i * ny + j) * nz + l;
    const int dx = sx * ny * nz, dy = sy * nz;
    {
        const int64_t map = block_map();
        if (map >= maps) return;
        const float* xm = x + map * (int64_t(nx) * ny * nz);
        int best_idx = base;
        float best = __ldg(xm + base);
#pragma unroll
        for (int a = 0; a < kx; ++a)
#pragma unroll
            for (int b = 0; b < ky; ++b)
#pragma unroll
                for (int c = 0; c < kz; ++c) {
                    const int idx = base + a * dx + b * dy + c * sz;
                    const float v = __ldg(xm + idx);
                    if (v > best) {  // strict: ties keep the lexicographically first source
                        best = v;
                        best_idx = idx;
                    }
                }
        y[map * int64_t(mv) + r] = best;
        mask[map * int64_t(mv) + r] = best_idx;
    }
}

// dx[t] = sum over windows o whose argmax is t of g[o]; windows visited in
// ascending flat order of o, the order the reference accumulates in
// (maxops.hpp:176-181), so fp32 sums match it bit for bit.
template <int KX, int KY, int KZ>
__global__ void __launch_bounds__(kThreads) maxfilter_bwd_k(const float* __restrict__ g,
                                                            const int32_t* __restrict__ mask, int64_t maps, int nx,
                                                            int ny, int nz, int mx, int my, int mz, int kx_, int ky_,
                                                            int kz_, int sx, int sy, int sz, float* __restrict__ dx) {
    const int kx = KX ? KX : kx_, ky = KY ? KY : ky_, kz = KZ ? KZ : kz_;
    const unsigned nv = unsigned(nx) * unsigned(ny) * unsigned(nz);
    const unsigned tr = blockIdx.x * kThreads + threadIdx.x;
    if (tr >= nv) return;
    const unsigned nyz = unsigned(ny) * unsigned(nz);
    const int ti = int(tr / nyz);
    const unsigned r2 = tr - unsigned(ti) * nyz;
    const int tj = int(r2 / unsigned(nz));
    const int tl = int(r2 - unsigned(tj) * unsigned(nz));
    const int64_t mv = int64_t(mx) * my * mz;
    {
        const int64_t map = block_map();
        if (map >= maps) return;
        const float* gm = g + map * mv;
        const int32_t* mm = mask + map * mv;
        float acc = 0.f;
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
                    if (__ldg(mm + o) == int(tr)) acc += __ldg(gm + o);
                }
            }
        }
        dx[map * int64_t(nv) + tr] = acc;
    }
}

__global__ void __launch_bounds__(kThreads) maxpool_fwd_k(const float* __restrict__ x, int64_t maps, int nx, int ny,
                                                          int nz, int px, int py, int pz, float* __restrict__ y,
                                                          int32_t* __restrict__ mask) {
    const int mx = nx / px, my = ny / py, mz = nz / pz;
    const unsigned mv = unsigned(mx) * unsigned(my) * unsigned(mz);
    const unsigned r = blockIdx.x * kThreads + threadIdx.x;
    if (r >= mv) return;
    const unsigned myz = unsigned(my) * unsigned(mz);
    const int bi = int(r / myz);
    const unsigned r2 = r - unsigned(bi) * myz;
    const int bj = int(r2 / unsigned(mz));
    const int bl = int(r2 - unsigned(bj) * unsigned(mz));
    const int base = ((bi * px) * ny + bj * py) * nz + bl * pz;
    {
        const int64_t map = block_map();
        if (map >= maps) return;
        const float* xm = x + map * (int64_t(nx) * ny * nz);
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
        y[map * int64_t(mv) + r] = best;
        mask[map * int64_t(mv) + r] = best_idx;
    }
}

__global__ void __launch_bounds__(kThreads) maxpool_bwd_k(const float* __restrict__ g, const int32_t* __restrict__ mask,
                                                          int64_t maps, int mx, int my, int mz, int px, int py, int pz,
                                                          float* __restrict__ dx) {
    const int nx = mx * px, ny = my * py, nz = mz * pz;
    const unsigned nv = unsigned(nx) * unsigned(ny) * unsigned(nz);
    const unsigned tr = blockIdx.x * kThreads + threadIdx.x;
    if (tr >= nv) return;
    const unsigned nyz = unsigned(ny) * unsigned(nz);
    const int ti = int(tr / nyz);
    const unsigned r2 = tr - unsigned(ti) * nyz;
    const int tj = int(r2 / unsigned(nz));
    const int tl = int(r2 - unsigned(tj) * unsigned(nz));
    const int o = ((ti / px) * my + (tj / py)) * mz + (tl / pz);
    const int64_t mv = int64_t(mx) * my * mz;
    const int64_t map = block_map();
    if (map < maps)
        dx[map * int64_t(nv) + tr] = (__ldg(mask + map * mv + o) == int(tr)) ? __ldg(g + map * mv + o) : 0.f;
}

}  // namespace

void maxfilter_fwd(cudaStream_t st, const float* x, int64_t maps, dims3 n, dims3 k, dims3 s,
                   float* y, int32_t* mask) {
    const dims3 m{n.x - s.x * (k.x - 1), n.y - s.y * (k.y - 1), n.z - s.z * (k.z - 1)};
    require(m.x > 0 && m.y > 0 && m.z > 0, "maxfilter_forward: effective window exceeds input");
    require(n.vol() < (int64_t(1) << 31), "maxfilter_forward: map exceeds int32 mask range");
    auto* kf = (k.x == 2 && k.y == 2 && k.z == 2)   ? maxfilter_fwd_k<2, 2, 2>
               : (k.x == 1 && k.y == 2 && k.z == 2) ? maxfilter_fwd_k<1, 2, 2>
                                                    : maxfilter_fwd_k<0, 0, 0>;
    kf<<<grid2(m.vol(), maps), kThreads, 0, st>>>(x, maps, int(n.x), int(n.y), int(n.z), int(m.x), int(m.y),
                                                 int(m.z), int(k.x), int(k.y), int(k.z), int(s.x), int(s.y),
                                                 int(s.z), y, mask);
    launch_check("maxfilter_fwd");
}

void maxfilter_bwd(cudaStream_t st, const float* g, const int32_t* mask, int64_t maps, dims3 m,
                   dims3 k, dims3 s, float* dx) {
    const dims3 n{m.x + s.x * (k.x - 1), m.y + s.y * (k.y - 1), m.z + s.z * (k.z - 1)};
    auto* kb = (k.x == 2 && k.y == 2 && k.z == 2)   ? maxfilter_bwd_k<2, 2, 2>
               : (k.x == 1 && k.y == 2 && k.z == 2) ? maxfilter_bwd_k<1, 2, 2>
                                                    : maxfilter_bwd_k<0, 0, 0>;
    kb<<<grid2(n.vol(), maps), kThreads, 0, st>>>(g, mask, maps, int(n.x), int(n.y), int(n.z), int(m.x), int(m.y),
                                                 int(m.z), int(k.x), int(k.y), int(k.z), int(s.x), int(s.y),
                                                 int(s.z), dx);
    launch_check("maxfilter_bwd");
}

void maxpool_fwd(cudaStream_t st, const float* x, int64_t maps, dims3 n, dims3 p, float* y,
                 int32_t* mask) {
    require(p.x > 0 && p.y > 0 && p.z > 0 && n.x % p.x == 0 && n.y % p.y == 0 && n.z % p.z == 0,
            "maxpool_forward: dims not divisible by window");
    const dims3 m{n.x / p.x, n.y / p.y, n.z / p.z};
    maxpool_fwd_k<<<grid2(m.vol(), maps), kThreads, 0, st>>>(
        x, maps, int(n.x), int(n.y), int(n.z), int(p.x), int(p.y), int(p.z), y, mask);
    launch_check("maxpool_fwd");
}

void maxpool_bwd(cudaStream_t st, const float* g, const int32_t* mask, int64_t maps, dims3 m,
                 dims3 p, float* dx) {
    const int64_t nvol = m.vol() * p.vol();
    maxpool_bwd_k<<<grid2(nvol, maps), kThreads, 0, st>>>(
        g, mask, maps, int(m.x), int(m.y), int(m.z), int(p.x), int(p.y), int(p.z), dx);
    launch_check("maxpool_bwd");
}

}  // namespace znn_gpu
