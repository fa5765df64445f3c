// Weight gradient of the 3D (dilated) valid convolution as a split-K
// tcgen05 implicit GEMM, 3xTF32 (kernel_gradient_direct, conv_direct.hpp:108-132,
// summed over the batch):
//   dW[o][i][w] = scale * sum_{b,v} g[b][o][v] * x[b][i][v + s*w]
// GEMM view: rows R = (i, w) (f_in*T of them, 128 per tile), columns = output
// maps o (<= 128 per tile), K = output voxels of every patch (32 per stage,
// never straddling a patch).
//   A (x rows, shifted windows) : in TMEM. Each producer warp owns 32 rows (its
//       TMEM lane quarter): it gathers them with coalesced row loads (lane =
//       voxel), transposes the 32x32 block through a private shared-memory
//       tile (conflict-free, pitch 33), splits hi/lo and writes its lanes with
//       tcgen05.st; the MMA reads A from TMEM (kind::tf32).
//   B (g rows)                  : pre-split into hi/lo tiles [B][map tile][K-block][nt][32]
//       by one memory-bound pass (each TMA box one contiguous block), then
//       TMA-loaded (SWIZZLE_128B), multicast to the 2 CTAs of a cluster.
// Each CTA owns a contiguous K range (split-K); partial tiles land in a
// workspace [split][o][R] and a fixed-order reduction sums them
// (deterministic).
//
// Warps: 0-7 producers (warps 0-3 even, 4-7 odd K-blocks; warp w owns A rows
// / TMEM lanes 32*(w%4)..+31) that also drain finished TMEM chunks (column
// half w / 4) and run the epilogue; 8 TMA producer; 9 TMEM alloc + MMA
// issuer; 10-11 idle (registers are granted per 4-warp group).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "ops.hpp"
#include "tc_common.cuh"

namespace znn_gpu {

CUtensorMap make_panel_map_rows(const float* ptr, int64_t cols, int64_t rows, int box_rows);

namespace {

using namespace znn_tc;

// NG producer warpgroups (one warp per TMEM lane quarter each) + one control
// warpgroup (TMA, MMA, 2 idle): 32 * 4 * (NG + 1) threads
template <int NG>
constexpr int threads_for() { return 128 * (NG + 1); }
constexpr uint32_t TMEM_COLS = 512;
constexpr int CHUNK_KB = 8;
constexpr int TP = 33;  // transpose tile pitch (floats)
constexpr int kPrefetch = 16;  // g tiles prefetched into L2 this many K-blocks ahead

struct wg_params {
    int f_in, f_out, T, nt;
    int mrows;  // f_in * T
    int stages, nbuf, bstride, na;
    int ntiles; // output-map tiles (grid y)
    int csize;  // CTAs per cluster along the row tiles: they share (multicast) every g tile
    int64_t kb_per_patch, kb_total, kb_per_split;
    int64_t nvol, mvol;
    int ny, nz, my, mz;
};

template <int NTMAX, bool PAIR, int NG>
__global__ void __launch_bounds__(threads_for<NG>(), 1)
wgrad_tc_kernel(const __grid_constant__ CUtensorMap tm_hi, const __grid_constant__ CUtensorMap tm_lo,
                const float* __restrict__ x, const int* __restrict__ rowoff_g, float* __restrict__ ws,
                wg_params p) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ int rowoff[BM];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* base_ptr = smem_raw + (base - raw);
    // PAIR: this CTA holds half of the g tile (nt/2 output maps); the pair MMA
    // reads both halves. Otherwise the whole tile (multicast to the cluster).
    const uint32_t b_bytes = uint32_t(PAIR ? p.nt / 2 : p.nt) * 128u;
    const uint32_t stage_bytes = 2u * b_bytes;
    const uint32_t bar_base = base + uint32_t(p.stages) * stage_bytes;
    auto full_bar = [&](int s) { return bar_base + 8u * uint32_t(s); };
    auto empty_bar = [&](int s) { return bar_base + 8u * uint32_t(p.stages + s); };
    const uint32_t accf0 = bar_base + 8u * uint32_t(2 * p.stages);
    const uint32_t acce0 = accf0 + 32u;
    const uint32_t af0 = acce0 + 32u;
    const uint32_t ae0 = af0 + 32u;
    uint8_t* tail = base_ptr + (bar_base - base) + 8u * uint32_t(2 * p.stages + 16);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tail);
    float* tpose = reinterpret_cast<float*>(tail + 16);  // producer warps x [32][TP]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r0 = blockIdx.x * BM;    // first (i, w) row of this tile
    const int n0 = blockIdx.y * p.nt;  // first output map
    const int64_t q0 = int64_t(blockIdx.z) * p.kb_per_split;
    const int64_t q1 = min(p.kb_total, q0 + p.kb_per_split);
    const int kblocks = int(q1 - q0);
    const int nchunks = (kblocks + CHUNK_KB - 1) / CHUNK_KB;

    // rows past f_in * T read a valid dummy offset: their D rows are never stored
    if (threadIdx.x < BM) rowoff[threadIdx.x] = (r0 + threadIdx.x < p.mrows) ? rowoff_g[r0 + threadIdx.x] : 0;
    if (threadIdx.x == 0) {
        // PAIR: the leader's full / A-written / drained barriers collect both
        // CTAs (elected remote arrives); every CTA's empty / A-free /
        // chunk-ready barriers receive the leader's multicast commits.
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(full_bar(s), PAIR ? 2u : 1u);
            mbar_init(empty_bar(s), PAIR ? 1u : uint32_t(p.csize));  // every CTA of the cluster consumed slot s
        }
        for (int b = 0; b < 4; ++b) {
            mbar_init(accf0 + 8u * b, 1);
            mbar_init(acce0 + 8u * b, PAIR ? 16u : 128u * NG);
            mbar_init(af0 + 8u * b, PAIR ? 8u : 128u);
            mbar_init(ae0 + 8u * b, 1);
        }
        fence_barrier_init();
    }
    constexpr int PW = 4 * NG;  // producer warps; then TMA warp PW, MMA warp PW + 1
    if (warp == PW + 1) {
        if constexpr (PAIR) tmem_alloc_pair(smem_u32(tmem_slot), TMEM_COLS);
        else tmem_alloc(smem_u32(tmem_slot), TMEM_COLS);
    }
    tc_fence_before();
    __syncthreads();
    if (p.csize > 1) cluster_sync();  // peers' barriers exist before any multicast lands
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t a_col0 = uint32_t(p.nbuf * p.bstride);
    const uint32_t rank = p.csize > 1 ? cluster_ctarank() : 0u;

    static_assert(NG == 2 || NG == 3, "2 or 3 producer warpgroups");
    if (warp < PW) setmaxnreg_inc<NG == 2 ? 224 : 152>();
    else setmaxnreg_dec<56>();
    if (warp < PW) {
        // group grp takes K-blocks grp, grp + NG, ...; the NG warps of one lane
        // quarter split its accumulator columns (NH each)
        constexpr int NH = ((NTMAX + NG - 1) / NG + 15) / 16 * 16;
        const int grp = warp >> 2;
        const int wq = warp & 3;    // rows / TMEM lanes 32*wq .. 32*wq + 31
        const int col0 = grp * NH;
        const int ncols = max(0, min(NH, p.nt - col0));
        const uint32_t lane_base = uint32_t(wq * 32) << 16;
        chunk_drainer<NH> D;
        D.init(accf0, acce0, tmem + lane_base + uint32_t(col0), p.nbuf, p.bstride, ncols, nchunks);
        if constexpr (PAIR) D.acce_leader = mapa_u32(acce0, 0);
        const uint32_t af_leader = PAIR ? mapa_u32(af0, 0) : 0u;
        const int mvol = int(p.mvol);
        const int myz = p.my * p.mz;
        float* tp = tpose + warp * (32 * TP);
        int a = grp;
        uint32_t u = 0;
        int64_t pb = (q0 + grp) / p.kb_per_patch;  // patch / K-block of the next gather, tracked incrementally
        int vkb = int(q0 + grp - pb * p.kb_per_patch);
        int ro[32];  // this warp's 32 row offsets (tap window starts), kept in registers
#pragma unroll
        for (int t = 0; t < 32; ++t) ro[t] = rowoff[wq * 32 + t];
        auto rowo = [&](int t) { return ro[t]; };
        auto gather = [&](float (&av)[32]) {
            const int v = vkb * BK + lane;
            const int64_t pcur = pb;
            for (vkb += NG; vkb >= p.kb_per_patch; vkb -= int(p.kb_per_patch)) ++pb;
            const bool vok = v < mvol;
            const float* xp = x;
            if (vok) {
                const int vx = v / myz;
                const int r2 = v - vx * myz;
                const int vy = r2 / p.mz;
                const int vz = r2 - vy * p.mz;
                xp = x + pcur * int64_t(p.f_in) * p.nvol + (vx * p.ny + vy) * p.nz + vz;
            }
            if (vok) {  // voxels past the patch (its last K-block) must contribute zeros
#pragma unroll
                for (int t = 0; t < 32; ++t) av[t] = __ldg(xp + rowo(t));
            } else {
#pragma unroll
                for (int t = 0; t < 32; ++t) av[t] = 0.f;
            }
        };
        auto put = [&](float (&av)[32]) {
            // 32x32 transpose through this warp's tile: row t, voxel lane -> lane t, column voxel
            __syncwarp();
#pragma unroll
            for (int t = 0; t < 32; ++t) tp[t * TP + lane] = av[t];
            __syncwarp();
#pragma unroll
            for (int c = 0; c < 32; ++c) av[c] = tp[lane * TP + c];
            D.wait_stage(ae0 + 8u * uint32_t(a), u ^ 1u);
            tc_fence_after();
            const uint32_t acol = tmem + lane_base + a_col0 + uint32_t(a) * 64u;
#pragma unroll
            for (int c = 0; c < BK / 8; ++c) {
                float h[8], l[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {  // lo is exact in fp32; the MMA keeps its top tf32 bits
                    h[e] = tf32_hi(av[8 * c + e]);
                    l[e] = av[8 * c + e] - h[e];
                }
                tmem_st8(acol + uint32_t(8 * c), h);
                tmem_st8(acol + 32u + uint32_t(8 * c), l);
            }
            tmem_wait_st();
            tc_fence_before();
            if constexpr (PAIR) {
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(af_leader + 8u * uint32_t(a));
            } else {
                mbar_arrive(af0 + 8u * uint32_t(a));
            }
            a += NG;
            if (a >= p.na) a = grp, u ^= 1u;
            D.poll();
        };
        // two K-blocks of gathers in flight per warp (registers from setmaxnreg)
        if constexpr (NG == 2) {  // two K-blocks of gathers in flight per warp
            float va[32], vb[32];
            if (grp < kblocks) gather(va);
            for (int kb = grp; kb < kblocks; kb += 2 * NG) {
                if (kb + NG < kblocks) gather(vb);
                put(va);
                if (kb + NG >= kblocks) break;
                if (kb + 2 * NG < kblocks) gather(va);
                put(vb);
            }
        } else {  // three groups already keep three K-blocks in flight
            float va[32];
            for (int kb = grp; kb < kblocks; kb += NG) {
                gather(va);
                put(va);
            }
        }
        // ---------------- remaining drains + epilogue (this warp's columns) ----------------
        D.finish();
        const int R = r0 + wq * 32 + lane;  // TMEM lane = tile row
        if (R < p.mrows) {
            float* wsz = ws + int64_t(blockIdx.z) * p.f_out * p.mrows;
#pragma unroll
            for (int qq = 0; qq < NH; ++qq) {
                const int o = n0 + col0 + qq;
                if (qq < ncols && o < p.f_out) wsz[int64_t(o) * p.mrows + R] = D.A.acc[qq];
            }
        }
    } else if (warp == PW) {
        // ---------------- TMA producer: g panels ----------------
        // Cluster rank r loads rows [r*nt/C, (r+1)*nt/C) of the g tile and
        // multicasts them to every CTA of the cluster (same K range, other
        // row tiles): each tile leaves L2 once per cluster.
        {  // converged warp, one elected lane issues
            const int C = p.csize;
            const int rows_per = p.nt / C;
            const uint32_t part = uint32_t(rows_per) * 128u;
            const uint16_t mask = uint16_t((1u << C) - 1u);
            int s = 0;
            uint32_t ph = 0;
            int64_t pb = q0 / p.kb_per_patch;
            int vkb = int(q0 - pb * p.kb_per_patch);
            for (int kb = 0; kb < kblocks; ++kb) {
                // g tiles are stored contiguously ([patch][map tile][K-block][nt rows][32]),
                // so a box is one 16 KB DRAM stream instead of nt scattered 128 B rows
                const int vcol = 0;
                const int row = int(((pb * p.ntiles + blockIdx.y) * p.kb_per_patch + vkb) * p.nt) + int(rank) * rows_per;
                if (kb + kPrefetch < kblocks && (kb % 2) == int(rank) && elect_one()) {
                    // pull the tile kPrefetch K-blocks ahead from HBM into L2 (the
                    // cluster ranks alternate), so the TMA below finds it there
                    int64_t ppb = pb;
                    int pvkb = vkb + kPrefetch;
                    while (pvkb >= p.kb_per_patch) pvkb -= int(p.kb_per_patch), ++ppb;
                    const int prow = int(((ppb * p.ntiles + blockIdx.y) * p.kb_per_patch + pvkb) * p.nt);
                    for (int h = 0; h < C; ++h) {  // the map's box is one rank's part of the tile
                        tma_prefetch_2d(&tm_hi, 0, prow + h * rows_per);
                        tma_prefetch_2d(&tm_lo, 0, prow + h * rows_per);
                    }
                }
                __syncwarp();
                mbar_wait(empty_bar(s), ph ^ 1u);
                const uint32_t b_hi = base + uint32_t(s) * stage_bytes;
                if constexpr (PAIR) {
                    // own half tile into own smem, bytes counted on the leader's barrier
                    const uint32_t fl = mapa_u32(full_bar(s), 0);
                    if (elect_one()) {
                        mbar_expect_tx_cluster(fl, 2u * b_bytes);
                        tma_load_2d_pair(b_hi, &tm_hi, fl, vcol, row);
                        tma_load_2d_pair(b_hi + b_bytes, &tm_lo, fl, vcol, row);
                    }
                    __syncwarp();
                } else if (C > 1) {
                    tma_pair_mc_w(full_bar(s), 2u * b_bytes, b_hi + rank * part, &tm_hi, b_hi + b_bytes + rank * part,
                                  &tm_lo, vcol, row, mask);
                } else {
                    tma_pair_w(full_bar(s), 2u * b_bytes, b_hi, &tm_hi, b_hi + b_bytes, &tm_lo, vcol, row);
                }
                if (++s == p.stages) s = 0, ph ^= 1u;
                if (++vkb == p.kb_per_patch) vkb = 0, ++pb;  // TMA side: one K-block per step
            }
        }
    } else if (warp == PW + 1) {
        // ---------------- MMA issuer ----------------
        if (!PAIR || rank == 0) {  // the whole warp runs the loop (converged); one elected lane issues
            const uint32_t idesc = idesc_tf32(PAIR ? 2 * BM : BM, p.nt);
            int b = 0, s = 0, a = 0, kc = 0;
            uint32_t bph = 0, sph = 0, aph = 0;
            for (int kb = 0; kb < kblocks; ++kb) {
                const bool first = kc == 0;
                if (first) {
                    mbar_wait(acce0 + 8u * uint32_t(b), bph ^ 1u);
                    tc_fence_after();
                }
                const uint32_t d = tmem + uint32_t(b * p.bstride);
                mbar_wait(full_bar(s), sph);
                mbar_wait(af0 + 8u * uint32_t(a), aph);
                tc_fence_after();
                const uint32_t a_hi = tmem + a_col0 + uint32_t(a) * 64u;
                const uint32_t b_hi = base + uint32_t(s) * stage_bytes;
                const uint32_t b_lo = b_hi + b_bytes;
#pragma unroll
                for (int kk = 0; kk < BK / 8; ++kk) {
                    const uint32_t ko = uint32_t(kk) * 32u;
                    const uint64_t bh = sw128_desc(b_hi + ko), bl = sw128_desc(b_lo + ko);
                    const uint32_t ah = a_hi + uint32_t(8 * kk), al = a_hi + 32u + uint32_t(8 * kk);
                    if constexpr (PAIR) {
                        mma_tf32_ts_pair_w(d, ah, bh, idesc, (first && kk == 0) ? 0u : 1u);
                        mma_tf32_ts_pair_w(d, ah, bl, idesc, 1u);
                        mma_tf32_ts_pair_w(d, al, bh, idesc, 1u);
                    } else {
                        mma_tf32_ts_w(d, ah, bh, idesc, (first && kk == 0) ? 0u : 1u);
                        mma_tf32_ts_w(d, ah, bl, idesc, 1u);
                        mma_tf32_ts_w(d, al, bh, idesc, 1u);
                    }
                }
                if constexpr (PAIR) {
                    mma_commit_pair_mc_w(empty_bar(s), 3);
                    mma_commit_pair_mc_w(ae0 + 8u * uint32_t(a), 3);
                    if (kc == CHUNK_KB - 1 || kb == kblocks - 1) mma_commit_pair_mc_w(accf0 + 8u * uint32_t(b), 3);
                } else {
                    if (p.csize > 1) mma_commit_mc_w(empty_bar(s), uint16_t((1u << p.csize) - 1u));
                    else mma_commit_w(empty_bar(s));
                    mma_commit_w(ae0 + 8u * uint32_t(a));
                    if (kc == CHUNK_KB - 1 || kb == kblocks - 1) mma_commit_w(accf0 + 8u * uint32_t(b));
                }
                if (++s == p.stages) s = 0, sph ^= 1u;
                if (++a == p.na) a = 0, aph ^= 1u;
                if (++kc == CHUNK_KB) {
                    kc = 0;
                    if (++b == p.nbuf) b = 0, bph ^= 1u;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (p.csize > 1) cluster_sync();  // no CTA leaves (or frees TMEM) while its peer still uses it
    if (warp == PW + 1) {
        __syncwarp();
        tc_fence_after();
        if constexpr (PAIR) tmem_dealloc_pair(tmem, TMEM_COLS);
        else tmem_dealloc(tmem, TMEM_COLS);
    }
}

__global__ void rowoff_k(int* __restrict__ out, int mrows, int T, int ky, int kz, int sx, int sy, int sz, int ny,
                         int nz, int64_t nvol) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < mrows; r += gridDim.x * blockDim.x) {
        const int i = r / T, t = r - i * T;
        const int wx = t / (ky * kz), wy = (t / kz) % ky, wz = t % kz;
        out[r] = int(int64_t(i) * nvol + (int64_t(sx * wx) * ny + sy * wy) * nz + sz * wz);
    }
}

// g [B][f_out][mvol] -> hi/lo tiles [B][map tile][K-block][R rows][32] (zero
// padded rows / columns): one TMA box per (patch, map tile, K-block) is a
// contiguous 128*R-byte block. grid: x = float4 in a tile, y = K-block,
// z = patch * map tiles + map tile.
__global__ void split_tiles_k(const float* __restrict__ g, int f_out, int64_t mvol, int R, int ntiles, int64_t kbpp,
                              float* __restrict__ hi, float* __restrict__ lo) {
    const int e4 = blockIdx.x * blockDim.x + threadIdx.x;
    if (e4 >= R * (BK / 4)) return;
    const int r = e4 / (BK / 4), c4 = e4 - r * (BK / 4);
    const int64_t q = blockIdx.y;
    const int64_t z = blockIdx.z;
    const int64_t pb = z / ntiles;
    const int o = int(z - pb * ntiles) * R + r;
    const int64_t col = q * BK + c4 * 4;
    float v[4], h[4], l[4];
    const float* src = g + (pb * f_out + o) * mvol;
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = (o < f_out && col + k < mvol) ? __ldg(src + col + k) : 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        h[k] = tf32_hi(v[k]);
        l[k] = tf32_rn(v[k] - h[k]);
    }
    const int64_t dst = ((z * kbpp + q) * R + r) * BK + c4 * 4;
    *reinterpret_cast<float4*>(hi + dst) = make_float4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<float4*>(lo + dst) = make_float4(l[0], l[1], l[2], l[3]);
}

// fixed-order sum of the split-K partials; with w != nullptr also the
// SGD+momentum update of those weights (the fused weight-gradient epilogue)
__global__ void reduce_splits_k(const float* __restrict__ ws, int64_t splits, int64_t len, float scale,
                                float* __restrict__ out, float* __restrict__ w, float* __restrict__ v, float lr,
                                float mu) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < len; i += int64_t(gridDim.x) * blockDim.x) {
        float acc = 0.f;
        for (int64_t s = 0; s < splits; ++s) acc += ws[s * len + i];
        const float g = scale * acc;
        out[i] = g;
        if (w) {
            const float nv = mu * v[i] + g;
            v[i] = nv;
            w[i] -= lr * nv;
        }
    }
}

template <int NTMAX, bool PAIR, int NG>
void launch_wgrad(dim3 grid, size_t smem, cudaStream_t st, const CUtensorMap& mhi, const CUtensorMap& mlo,
                  const float* x, const int* rowoff, float* ws, const wg_params& p) {
    auto* k = wgrad_tc_kernel<NTMAX, PAIR, NG>;
    ZNN_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(threads_for<NG>(), 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(p.csize);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ZNN_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k, mhi, mlo, x, rowoff, ws, p));
    launch_check("conv_wgrad_tc");
}

template <int NTMAX, bool PAIR, int NG>
const void* wgrad_kernel_ptr() {
    return reinterpret_cast<const void*>(wgrad_tc_kernel<NTMAX, PAIR, NG>);
}
template <bool PAIR, int NG>
const void* wgrad_kernel_ptr(int ntmax) {
    return ntmax == 32 ? wgrad_kernel_ptr<32, PAIR, NG>()
                       : (ntmax == 64 ? wgrad_kernel_ptr<64, PAIR, NG>() : wgrad_kernel_ptr<128, PAIR, NG>());
}

// CTAs resident at once (one per SM; clusters cannot use every SM of a GPC)
int64_t resident_ctas(int ntmax, size_t smem, int csize, bool pair, int ng) {
    static int64_t cache[3][3][2][2] = {};
    const int ti = ntmax == 32 ? 0 : (ntmax == 64 ? 1 : 2), ci = csize == 1 ? 0 : (csize == 2 ? 1 : 2);
    int64_t& slot = cache[ti][ci][pair][ng == 3];
    if (slot) return slot;
    int64_t r = 148;
    if (csize > 1) {
        const void* k = pair      ? wgrad_kernel_ptr<true, 2>(ntmax)
                         : ng == 3 ? wgrad_kernel_ptr<false, 3>(ntmax)
                                   : wgrad_kernel_ptr<false, 2>(ntmax);
        ZNN_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(csize) * 64, 1, 1);
        cfg.blockDim = dim3(unsigned(128 * (ng + 1)), 1, 1);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = unsigned(csize);
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, k, &cfg) == cudaSuccess && nc > 0) r = int64_t(nc) * csize;
        else cudaGetLastError();
    }
    slot = r;
    return r;
}

}  // namespace

void conv_wgrad_tc(cudaStream_t st, const conv_shape& c, const float* x, const float* g, float* dw, float scale,
                   scratch& ws, const sgd_fuse* upd) {
    prof_scope ps(st,
                  "conv_wgrad_tc f=" + std::to_string(c.f_in) + "->" + std::to_string(c.f_out) + " n=" +
                      std::to_string(c.n.x) + " k=" + std::to_string(c.k.x) + " s=" + std::to_string(c.s.x) +
                      " B=" + std::to_string(c.B),
                  4.0 * double(c.B) * double(c.f_in * c.n.vol() + c.f_out * c.m.vol()),
                  2.0 * double(c.B * c.f_in * c.f_out) * double(c.m.vol() * c.taps()));
    wg_params p;
    p.f_in = int(c.f_in);
    p.f_out = int(c.f_out);
    p.T = int(c.taps());
    p.mrows = p.f_in * p.T;
    const int64_t r16 = ceil_div(c.f_out, 16) * 16;
    p.nt = int(r16 <= 128 ? r16 : 128);
    const int ntiles = int(ceil_div(c.f_out, p.nt));
    const int ntmax = p.nt <= 32 ? 32 : (p.nt <= 64 ? 64 : 128);
    p.bstride = ntmax;
    p.nbuf = ntmax == 128 ? 2 : 4;  // + na x 64 A columns <= 512 TMEM columns
    // producer warpgroups: 3 measured ~7% faster than 2 on c5 (the gather +
    // transpose chain is latency-bound with one producer warp per SMSP)
    int ng = 3;
    if (const char* e = std::getenv("ZNN_WGRAD_NG")) ng = std::atoi(e) == 2 ? 2 : 3;
    p.nvol = c.n.vol();
    p.mvol = c.m.vol();
    p.ny = int(c.n.y), p.nz = int(c.n.z), p.my = int(c.m.y), p.mz = int(c.m.z);
    p.kb_per_patch = ceil_div(p.mvol, BK);
    p.kb_total = p.kb_per_patch * c.B;
    // clusters of csize row tiles share every g tile by TMA multicast (the
    // g panel is streamed once per cluster instead of once per row tile)
    int csize = 2;  // measured on c5: 2 beats 4 (cluster placement) and 1 (L2 misses)
    if (const char* e = std::getenv("ZNN_WGRAD_CLUSTER")) csize = std::atoi(e);
    while (csize > 1 && (p.nt % (8 * csize) != 0 || ceil_div(p.mrows, BM) < csize)) csize /= 2;
    if (csize != 1 && csize != 2 && csize != 4) csize = 1;
    p.csize = csize;
    // CTA pairs (cta_group::2, M = 256): each CTA stages half of the g tile
    // and the pair MMA reads both halves, halving B's shared-memory traffic.
    // Parity-green but measured slower on c5 (conv2 wgrad 232 vs 197 ms: the
    // pair MMA waits for the slower CTA's producers), so opt-in only.
    bool pair = false;
    if (const char* e = std::getenv("ZNN_WGRAD_PAIR")) pair = csize == 2 && p.nt % 32 == 0 && std::atoi(e) != 0;
    const int stage = 2 * (pair ? p.nt / 2 : p.nt) * 128;
    if (pair) ng = 2;
    p.na = ng == 3 ? 3 : 4;  // A buffers: a multiple of the producer groups
    const size_t fixed = 1024 + 8 * size_t(16) + 16 + sizeof(float) * 4 * ng * 32 * TP + 64;
    p.stages = int((size_t(220) * 1024 - fixed) / size_t(stage + 16));
    if (p.stages > 8) p.stages = 8;
    const int mtiles = int(ceil_div(ceil_div(p.mrows, BM), csize) * csize);
    // split-K factor: fill whole waves of 148 SMs (one CTA each). The first
    // split count >= 2 waves whose last wave is >= 97% full, else the best
    // fill up to max(32, 8 waves' worth) splits (a 2.4-wave grid idles 20% of the GPU in its tail).
    const int64_t tiles = int64_t(mtiles) * ntiles;
    const size_t smem = size_t(p.stages) * size_t(stage) + 8 * size_t(2 * p.stages + 16) + fixed;
    const int64_t wave = resident_ctas(ntmax, smem, csize, pair, ng);
    const int64_t max_splits = std::max<int64_t>(
        1, std::min<int64_t>(std::max<int64_t>(32, ceil_div(8 * 148, tiles)), ceil_div(p.kb_total, 4 * CHUNK_KB)));
    int64_t splits = 1;
    double best = -1.0;
    for (int64_t sp = 1; sp <= max_splits; ++sp) {
        const int64_t ctas = tiles * sp;
        const double eff = double(ctas) / double(ceil_div(ctas, wave) * wave);
        if (ctas >= 2 * wave && eff >= 0.97) {
            splits = sp;
            break;
        }
        if (eff > best + 1e-9) best = eff, splits = sp;
    }
    p.kb_per_split = ceil_div(p.kb_total, splits);
    splits = ceil_div(p.kb_total, p.kb_per_split);

    p.ntiles = ntiles;
    const int64_t gtiles = c.B * ntiles * p.kb_per_patch;  // (patch, map tile, K-block) tiles
    const size_t panel = size_t(gtiles) * size_t(p.nt) * BK;
    const size_t part = size_t(splits) * size_t(c.f_out) * size_t(p.mrows);
    char* wsp = static_cast<char*>(ws.get(sizeof(float) * (2 * panel + part) + sizeof(int) * size_t(p.mrows) + 4096));
    float* ghi = reinterpret_cast<float*>(wsp);
    float* glo = ghi + panel;
    float* partials = glo + panel;
    int* rowoff = reinterpret_cast<int*>((reinterpret_cast<uintptr_t>(partials + part) + 255) & ~uintptr_t(255));
    require(p.kb_per_patch < 65536 && c.B * ntiles < 65536, "wgrad: volume too large for the tile grid");
    const dim3 sgrid(unsigned(ceil_div(p.nt * (BK / 4), 256)), unsigned(p.kb_per_patch), unsigned(c.B * ntiles));
    split_tiles_k<<<sgrid, 256, 0, st>>>(g, int(c.f_out), p.mvol, p.nt, ntiles, p.kb_per_patch, ghi, glo);
    launch_check("conv_wgrad_tc_split");
    rowoff_k<<<unsigned(ceil_div(p.mrows, 256)), 256, 0, st>>>(rowoff, p.mrows, p.T, int(c.k.y), int(c.k.z),
                                                               int(c.s.x), int(c.s.y), int(c.s.z), p.ny, p.nz,
                                                               p.nvol);
    launch_check("conv_wgrad_tc_rowoff");
    const CUtensorMap mhi = make_panel_map_rows(ghi, BK, gtiles * p.nt, p.nt / csize);
    const CUtensorMap mlo = make_panel_map_rows(glo, BK, gtiles * p.nt, p.nt / csize);
    const dim3 grid{unsigned(mtiles), unsigned(ntiles), unsigned(splits)};
    if (pair) {
        if (ntmax == 32) launch_wgrad<32, true, 2>(grid, smem, st, mhi, mlo, x, rowoff, partials, p);
        else if (ntmax == 64) launch_wgrad<64, true, 2>(grid, smem, st, mhi, mlo, x, rowoff, partials, p);
        else launch_wgrad<128, true, 2>(grid, smem, st, mhi, mlo, x, rowoff, partials, p);
    } else if (ng == 3) {
        if (ntmax == 32) launch_wgrad<32, false, 3>(grid, smem, st, mhi, mlo, x, rowoff, partials, p);
        else if (ntmax == 64) launch_wgrad<64, false, 3>(grid, smem, st, mhi, mlo, x, rowoff, partials, p);
        else launch_wgrad<128, false, 3>(grid, smem, st, mhi, mlo, x, rowoff, partials, p);
    } else {
        if (ntmax == 32) launch_wgrad<32, false, 2>(grid, smem, st, mhi, mlo, x, rowoff, partials, p);
        else if (ntmax == 64) launch_wgrad<64, false, 2>(grid, smem, st, mhi, mlo, x, rowoff, partials, p);
        else launch_wgrad<128, false, 2>(grid, smem, st, mhi, mlo, x, rowoff, partials, p);
    }
    const int64_t len = c.f_out * int64_t(p.mrows);
    int64_t rb = ceil_div(len, 256);
    if (rb > 148 * 8) rb = 148 * 8;
    reduce_splits_k<<<unsigned(rb), 256, 0, st>>>(partials, splits, len, scale, dw, upd ? upd->w : nullptr,
                                                  upd ? upd->v : nullptr, upd ? upd->lr : 0.f,
                                                  upd ? upd->mu : 0.f);
    launch_check("conv_wgrad_tc_reduce");
}

}  // namespace znn_gpu
