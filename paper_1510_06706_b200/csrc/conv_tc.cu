// Direct 3D (dilated) convolution as a tcgen05 implicit GEMM, 3xTF32.
//
// GEMM view (one CTA = 128 output voxels x NT output maps):
//   D[v][n] = sum_k A[v][k] * B[n][k],   A[v][k] = src[b][c][v + s*w]
//   fwd   : src = x, B = W                         (conv_direct.hpp:39-68)
//   dgrad : src = g zero-haloed by s*(k-1) per side, B[i][(o, w')] = W[o][i][T-1-w']
//           i.e. conv_full_direct(g, reflect(k)) (conv_direct.hpp:74-101, engine.hpp:681)
//           computed as a valid convolution: no bounds tests in the hot loop.
// K order: k = ((wx*ky + wy)*f + c)*kz + wz — kernel rows (wx, wy) outermost,
// so a 32-wide K-block touches one or two (wx, wy) rows of taps. A tile whose
// voxels only see the zero halo through a tap row skips that K-block (dgrad of
// the sparse layers spends up to 70% of its taps in the halo otherwise); the
// inner (c, wz) order keeps a K-block's gathers on a few overlapping z-runs.
// The reference's convergent-edge sum (engine.hpp:345-353, sum_accumulator.hpp)
// is the K loop, accumulated in TMEM: no atomics, no locks. fp32 accuracy on
// tensor cores: operands split into hi = tf32(x), lo = tf32(x - hi) and
// D += Ahi*Bhi + Ahi*Blo + Alo*Bhi. TMEM accumulation is cut into chunks of
// CHUNK_KB K-blocks drained into fp32 registers (tensor-core accumulation
// error grows with the number of accumulating MMAs).
//
// Operands: A (the im2col tile, hi|lo) lives in TMEM — the producers write it
// with tcgen05.st and the MMA reads it from there (kind::tf32, A in TMEM), so
// shared memory only carries B (pre-split weight panels, TMA, SWIZZLE_128B).
// With both operands in shared memory the 3 MMAs per K-step read 8 KB per
// 64 cycles — the whole shared-memory bandwidth — before any operand is written.
//
// TMEM columns: [0, nbuf*bstride) accumulator chunks, then NA A buffers of
// 64 columns (32 hi + 32 lo).
// Warp roles (384 threads, 1 CTA per SM; warps 10-11 idle):
//   warps 0-7 : im2col producers: thread = one voxel row = one TMEM lane
//               (warp w owns lane quarter w % 4); warps 0-3 fill the even and
//               4-7 the odd active K-blocks; they also drain finished
//               accumulator chunks (warps 0-3 columns [0, NT/2), 4-7
//               [NT/2, NT)) and run the epilogue (bias + transfer, coalesced)
//   warp 8    : TMA producer for B
//   warp 9    : TMEM allocator + single-thread tcgen05.mma issuer
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "ops.hpp"
#include "tc_common.cuh"

namespace znn_gpu {

namespace {

using namespace znn_tc;

// NG producer warpgroups (one warp per TMEM lane quarter each) + one control
// warpgroup (TMA, MMA, K-block list, idle): 128 * (NG + 1) threads
template <int NG>
constexpr int conv_threads() { return 128 * (NG + 1); }
constexpr uint32_t TMEM_COLS = 512;
constexpr int CHUNK_KB = 8;

struct tc_params {
    int f_src;        // channels of the im2col source
    int n_real;       // real N (output maps of this GEMM)
    int nt;           // N tile (multiple of 16, <= NTMAX)
    int kblocks;
    int K;            // real K (f_src * T)
    int stages;
    int nbuf;         // TMEM accumulator buffers
    int bstride;      // TMEM columns per buffer
    int na;           // TMEM A buffers (64 columns each)
    int64_t rows;     // B * vox_out
    int64_t vox_out;  // voxels per output map
    int ox, oy, oz;   // output dims
    int sx, sy, sz;   // source dims
    int64_t src_vol;
    // tap-row skipping: K group = one (wx, wy) kernel row, gsize = f_src*kz
    int gsize, ky, dsx, dsy;
    int vx0, vx1, vy0, vy1;  // source region that can be nonzero (inclusive)
    // box tiles (dgrad): a tile is a bxs x bys x bzs box of output voxels and
    // K is tap-major (k = tap * f + c), so whole taps are skipped along all
    // three axes; box == 0: tiles are 128 consecutive voxels, K (wx, wy)-outer
    int box, bxs, bys, bzs, tnx, tny, tnz;
    int kz, dsz, vz0, vz1, taps;
};

template <int NTMAX, int NG>
__global__ void __launch_bounds__(conv_threads<NG>(), 1)
conv_tc_kernel(const __grid_constant__ CUtensorMap tm_hi, const __grid_constant__ CUtensorMap tm_lo,
               const float* __restrict__ src, const int* __restrict__ koff, float* __restrict__ out,
               const float* __restrict__ bias, int act, tc_params p) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ int s_nact;
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* base_ptr = smem_raw + (base - raw);
    const uint32_t b_bytes = uint32_t(p.nt) * 128u;
    const uint32_t stage_bytes = 2u * b_bytes;
    const uint32_t bar_base = base + uint32_t(p.stages) * stage_bytes;
    auto full_bar = [&](int s) { return bar_base + 8u * uint32_t(s); };
    auto empty_bar = [&](int s) { return bar_base + 8u * uint32_t(p.stages + s); };
    const uint32_t accf0 = bar_base + 8u * uint32_t(2 * p.stages);
    const uint32_t acce0 = accf0 + 32u;
    const uint32_t af0 = acce0 + 32u;  // A buffer written (128 producer arrivals)
    const uint32_t ae0 = af0 + 32u;    // A buffer consumed (MMA commit)
    uint8_t* tail = base_ptr + (bar_base - base) + 8u * uint32_t(2 * p.stages + 16);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tail);
    uint16_t* list = reinterpret_cast<uint16_t*>(tail + 16);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t m0 = int64_t(blockIdx.x) * BM;
    const int n0 = blockIdx.y * p.nt;

    if (threadIdx.x == 0) {
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), 1);
        }
        for (int b = 0; b < 4; ++b) {
            mbar_init(accf0 + 8u * b, 1);
            mbar_init(acce0 + 8u * b, 128u * NG);
            mbar_init(af0 + 8u * b, 128);
            mbar_init(ae0 + 8u * b, 1);
        }
        fence_barrier_init();
    }
    constexpr int PW = 4 * NG;  // producer warps; TMA warp PW, MMA warp PW + 1, list warp PW + 2
    if (warp == PW + 1) tmem_alloc(smem_u32(tmem_slot), TMEM_COLS);
    if (warp == PW + 2) {
        // active K-blocks of this tile: a (wx, wy) tap row is live iff the
        // tile's bounding box shifted by s*w meets the nonzero source region
        int x0 = 0, x1 = p.ox - 1, y0 = 0, y1 = p.oy - 1, z0 = 0, z1 = p.oz - 1;
        if (p.box) {
            const int t = blockIdx.x % (p.tnx * p.tny * p.tnz);
            const int ix = t / (p.tny * p.tnz), iy = (t / p.tnz) % p.tny, iz = t % p.tnz;
            x0 = ix * p.bxs, x1 = min(x0 + p.bxs, p.ox) - 1;
            y0 = iy * p.bys, y1 = min(y0 + p.bys, p.oy) - 1;
            z0 = iz * p.bzs, z1 = min(z0 + p.bzs, p.oz) - 1;
        } else {
            const int64_t va = m0, vb = min(m0 + BM, p.rows) - 1;
            const int64_t ba = va / p.vox_out, bb = vb / p.vox_out;
            if (ba == bb) {
                const int64_t ra = va - ba * p.vox_out, rb = vb - bb * p.vox_out;
                const int64_t plane = int64_t(p.oy) * p.oz;
                x0 = int(ra / plane), x1 = int(rb / plane);
                if (x0 == x1) y0 = int((ra / p.oz) % p.oy), y1 = int((rb / p.oz) % p.oy);
            }
        }
        int cnt = 0;
        for (int kb0 = 0; kb0 < p.kblocks; kb0 += 32) {
            const int kb = kb0 + lane;
            bool act_kb = false;
            if (kb < p.kblocks) {
                const int g0 = (kb * BK) / p.gsize, g1 = (min(kb * BK + BK, p.K) - 1) / p.gsize;
                for (int g = g0; g <= g1 && !act_kb; ++g) {
                    // group g: a (wx, wy) tap row, or (box tiles) a single tap (wx, wy, wz)
                    int wz = 0, gr = g;
                    if (p.box) {
                        const int t = g % p.taps;  // group = (channel block, tap)
                        wz = t % p.kz, gr = t / p.kz;
                    }
                    const int wx = gr / p.ky, wy = gr - (gr / p.ky) * p.ky;
                    act_kb = x0 + p.dsx * wx <= p.vx1 && x1 + p.dsx * wx >= p.vx0 && y0 + p.dsy * wy <= p.vy1 &&
                             y1 + p.dsy * wy >= p.vy0 && z0 + p.dsz * wz <= p.vz1 && z1 + p.dsz * wz >= p.vz0;
                }
            }
            const uint32_t m = __ballot_sync(0xffffffffu, act_kb);
            if (act_kb) list[cnt + __popc(m & ((1u << lane) - 1u))] = uint16_t(kb);
            cnt += __popc(m);
        }
        if (lane == 0) s_nact = cnt;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int nact = s_nact;
    const int nchunks = (nact + CHUNK_KB - 1) / CHUNK_KB;
    const uint32_t a_col0 = uint32_t(p.nbuf * p.bstride);

    if constexpr (NG == 3) {  // producers need the registers of a fourth warpgroup
        if (warp < PW) setmaxnreg_inc<152>();
        else setmaxnreg_dec<56>();
    }
    if (warp < PW) {
        // ---------------- im2col producers -> TMEM ----------------
        const int r = threadIdx.x & 127;
        const int half = threadIdx.x >> 7;  // producer group: active K-blocks half, half + NG, ...
        constexpr int NH = ((NTMAX + NG - 1) / NG + 15) / 16 * 16;
        const int col0 = half * NH;
        const int ncols = max(0, min(NH, p.nt - col0));
        const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
        chunk_drainer<NH> D;
        D.init(accf0, acce0, tmem + lane_base + uint32_t(col0), p.nbuf, p.bstride, ncols, nchunks);
        // this row's output voxel: patch vb, in-volume index vin
        bool vok;
        int64_t vb, vin;
        int tx, ty, tz;
        if (p.box) {
            const int per = p.tnx * p.tny * p.tnz;
            vb = blockIdx.x / per;
            const int t = blockIdx.x - int(vb) * per;
            const int ix = t / (p.tny * p.tnz), iy = (t / p.tnz) % p.tny, iz = t % p.tnz;
            tx = ix * p.bxs + r / (p.bys * p.bzs);
            ty = iy * p.bys + (r / p.bzs) % p.bys;
            tz = iz * p.bzs + r % p.bzs;
            vok = tx < p.ox && ty < p.oy && tz < p.oz;
            vin = (int64_t(tx) * p.oy + ty) * p.oz + tz;
        } else {
            const int64_t v = m0 + r;
            vok = v < p.rows;
            vb = vok ? v / p.vox_out : 0;
            vin = v - vb * p.vox_out;
            tx = int(vin / (int64_t(p.oy) * p.oz));
            ty = int((vin / p.oz) % p.oy);
            tz = int(vin % p.oz);
        }
        const float* sp = src;
        if (vok) sp = src + vb * int64_t(p.f_src) * p.src_vol + (int64_t(tx) * p.sy + ty) * p.sz + tz;
        // this group's A buffers: half, half + 2, ... (< na); (a, use parity) tracked incrementally
        int a = half;
        uint32_t u = 0;
        for (int j = half; j < nact; j += NG) {
            const int kb = list[j];
            const int4* tb = reinterpret_cast<const int4*>(koff + kb * BK);
            float v[BK];
#pragma unroll
            for (int q = 0; q < BK / 4; ++q) {
                const int4 e = __ldg(tb + q);
                v[4 * q + 0] = vok ? __ldg(sp + e.x) : 0.f;
                v[4 * q + 1] = vok ? __ldg(sp + e.y) : 0.f;
                v[4 * q + 2] = vok ? __ldg(sp + e.z) : 0.f;
                v[4 * q + 3] = vok ? __ldg(sp + e.w) : 0.f;
            }
            D.wait_stage(ae0 + 8u * uint32_t(a), u ^ 1u);
            tc_fence_after();
            const uint32_t acol = tmem + lane_base + a_col0 + uint32_t(a) * 64u;
#pragma unroll
            for (int c = 0; c < BK / 8; ++c) {
                float h[8], l[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {  // lo is exact in fp32; the MMA keeps its top tf32 bits
                    h[q] = tf32_hi(v[8 * c + q]);
                    l[q] = v[8 * c + q] - h[q];
                }
                tmem_st8(acol + uint32_t(8 * c), h);
                tmem_st8(acol + 32u + uint32_t(8 * c), l);
            }
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(af0 + 8u * uint32_t(a));
            a += NG;
            if (a >= p.na) a = half, u ^= 1u;
            D.poll();
        }
        // ---------------- remaining drains + epilogue (this warp's columns) ----------------
        D.finish();
        if (vok) {
            float* op = out + vb * int64_t(p.n_real) * p.vox_out + vin;
#pragma unroll
            for (int q = 0; q < NH; ++q) {
                const int n = n0 + col0 + q;
                if (q < ncols && n < p.n_real) {
                    const float val = act_value(act, D.A.acc[q] + (bias ? __ldg(bias + n) : 0.f));
                    op[int64_t(n) * p.vox_out] = val;
                }
            }
        }
    } else if (warp == PW) {
        // ---------------- TMA producer (pre-split weight panels) ----------------
        {  // converged warp, one elected lane issues
            int s = 0;
            uint32_t ph = 0;
            for (int j = 0; j < nact; ++j) {
                const int kb = list[j];
                mbar_wait(empty_bar(s), ph ^ 1u);
                const uint32_t b_hi = base + uint32_t(s) * stage_bytes;
                tma_pair_w(full_bar(s), 2u * b_bytes, b_hi, &tm_hi, b_hi + b_bytes, &tm_lo, kb * BK, n0);
                if (++s == p.stages) s = 0, ph ^= 1u;
            }
        }
    } else if (warp == PW + 1) {
        // ---------------- MMA issuer ----------------
        {  // the whole warp runs the loop (converged); one elected lane issues
            const uint32_t idesc = idesc_tf32(BM, p.nt);
            int b = 0, s = 0, a = 0, kc = 0;
            uint32_t bph = 0, sph = 0, aph = 0;
            for (int j = 0; j < nact; ++j) {
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
                    const uint32_t ko = uint32_t(kk) * 32u;  // 8 tf32 = 32 B along K
                    const uint64_t bh = sw128_desc(b_hi + ko), bl = sw128_desc(b_lo + ko);
                    const uint32_t ah = a_hi + uint32_t(8 * kk), al = a_hi + 32u + uint32_t(8 * kk);
                    mma_tf32_ts_w(d, ah, bh, idesc, (first && kk == 0) ? 0u : 1u);
                    mma_tf32_ts_w(d, ah, bl, idesc, 1u);
                    mma_tf32_ts_w(d, al, bh, idesc, 1u);
                }
                mma_commit_w(empty_bar(s));
                mma_commit_w(ae0 + 8u * uint32_t(a));
                if (kc == CHUNK_KB - 1 || j == nact - 1) mma_commit_w(accf0 + 8u * uint32_t(b));
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
    if (warp == PW + 1) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc(tmem, TMEM_COLS);
    }
}

// K index -> (source channel c, tap t): order 0 = (wx, wy)-outer with (c, wz)
// inner (k = ((wx*ky + wy)*f + c)*kz + wz); order CB > 0 = channel blocks of
// CB, taps, channels in the block (k = (cb*T + t)*CB + ci): a K-block covers
// one or two taps of one channel block, and consecutive K-blocks walk the taps
// of the same channels (their gathers overlap in L1)
__device__ __forceinline__ void k_decode(int k, int f, int T, int kz, int order, int& c, int& t) {
    if (order) {
        const int cb = k / (T * order), rem = k - cb * (T * order);
        t = rem / order;
        c = cb * order + (rem - t * order);
        return;
    }
    const int gsize = f * kz;
    const int g = k / gsize, rem = k - g * gsize;
    c = rem / kz;
    const int wz = rem - c * kz;
    t = g * kz + wz;  // g = wx*ky + wy, so t = (wx*ky + wy)*kz + wz
}

// Weight panels for the B operand, split hi/lo, zero padded to [npad][kpad].
//   mode 0 (fwd)  : B[n][(c, t)] = W[n][c][t]
//   mode 1 (dgrad): B[n][(o, t)] = W[o][n][T-1-t]   (transposed, reflected)
__global__ void split_weights_k(const float* __restrict__ w, int n_real, int f_src, int f_in, int T, int ky, int kz,
                                int K, int npad, int kpad, int mode, int order, float* __restrict__ hi,
                                float* __restrict__ lo) {
    const int64_t total = int64_t(npad) * kpad;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
        const int n = int(i / kpad), k = int(i - int64_t(n) * kpad);
        float v = 0.f;
        if (n < n_real && k < K) {
            int c, t;
            k_decode(k, f_src, T, kz, order, c, t);
            if (mode == 0) v = w[(int64_t(n) * f_src + c) * T + t];
            else v = w[(int64_t(c) * f_in + n) * T + (T - 1 - t)];
        }
        const float h = tf32_hi(v);
        hi[i] = h;
        lo[i] = tf32_rn(v - h);
    }
}

// im2col offsets: koff[k] = c*src_vol + linear(s*w) in source dims; padded
// k -> 0 (their weights are zero).
__global__ void koff_k(int* __restrict__ tab, int K, int kpad, int f_src, int kx, int ky, int kz, int order, int sx,
                       int sy, int sz, int64_t src_vol, int src_y, int src_z) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < kpad; k += gridDim.x * blockDim.x) {
        int e = 0;
        if (k < K) {
            int c, t;
            k_decode(k, f_src, ky * kz * kx, kz, order, c, t);
            const int wx = t / (ky * kz), wy = (t / kz) % ky, wz = t % kz;
            e = int(int64_t(c) * src_vol + (int64_t(sx * wx) * src_y + sy * wy) * src_z + sz * wz);
        }
        tab[k] = e;
    }
}

// g [maps][m] -> gp [maps][m + 2P] with a zero halo of P = s*(k-1) per side.
// block = 32 z-lanes x 8 padded y-rows; grid = (y tiles, padded x, maps).
__global__ void __launch_bounds__(256) pad_halo_k(const float* __restrict__ g, int mx, int my, int mz, int px, int py,
                                                  int pz, float* __restrict__ gp) {
    const int gx = mx + 2 * px, gy = my + 2 * py, gz = mz + 2 * pz;
    const int y = blockIdx.x * 8 + threadIdx.y, x = blockIdx.y;
    if (y >= gy) return;
    const int64_t map = blockIdx.z;
    float* dst = gp + map * (int64_t(gx) * gy * gz) + (int64_t(x) * gy + y) * gz;
    const int ux = x - px, uy = y - py;
    const bool rin = unsigned(ux) < unsigned(mx) && unsigned(uy) < unsigned(my);
    const float* src = g + map * (int64_t(mx) * my * mz) + (int64_t(ux) * my + uy) * mz;
    for (int z = threadIdx.x; z < gz; z += 32) {
        const int uz = z - pz;
        __stcs(dst + z, (rin && unsigned(uz) < unsigned(mz)) ? __ldcs(src + uz) : 0.f);
    }
}

typedef CUresult (*encode_fn_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

encode_fn_t encoder() {
    static encode_fn_t fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        ZNN_CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) throw cuda_error("cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<encode_fn_t>(p);
    }
    return fn;
}

CUtensorMap make_panel_map(const float* ptr, int kpad, int rows, int nt);

template <int NTMAX, int NG>
void launch_kernel(dim3 grid, size_t smem, cudaStream_t st, const CUtensorMap& mhi, const CUtensorMap& mlo,
                   const float* srcp, const int* tab, float* outp, const float* bias, int act, const tc_params& p,
                   const char* what) {
    auto* k = conv_tc_kernel<NTMAX, NG>;
    ZNN_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    k<<<grid, conv_threads<NG>(), smem, st>>>(mhi, mlo, srcp, tab, outp, bias, act, p);
    launch_check(what);
}

// Rows x taps computed along one axis when output tiles of extent L skip the
// taps whose shifted tile misses the nonzero source interval [v0, v0 + vn).
int64_t axis_work(int64_t n_out, int64_t L, int64_t s, int64_t k, int64_t v0, int64_t vn) {
    int64_t tot = 0;
    for (int64_t t0 = 0; t0 < n_out; t0 += L) {
        const int64_t t1 = std::min(t0 + L, n_out) - 1;
        int64_t act = 0;
        for (int64_t w = 0; w < k; ++w) act += (t0 + s * w <= v0 + vn - 1 && t1 + s * w >= v0) ? 1 : 0;
        tot += act * L;
    }
    return tot;
}

struct box_choice {
    int box = 0, bx = 0, by = 0, bz = 0;
};

// Box tiles (with tap-major K) for a convolution whose source has a zero halo,
// when they cut the computed MMA work by >= 8% against the flattened tiles
// (whose bounding box is ~1 x 2 x full-z voxels).
box_choice choose_box(dims3 od, dims3 k, dims3 s, dims3 v0, dims3 vn) {
    box_choice best;
    const double flat = double(axis_work(od.x, 1, s.x, k.x, v0.x, vn.x)) *
                        double(axis_work(od.y, 2, s.y, k.y, v0.y, vn.y)) * double(od.z * k.z);
    double bw = 0.92 * flat;
    static const int shapes[][3] = {{4, 4, 8}, {2, 8, 8}, {2, 4, 16}, {1, 8, 16}, {4, 8, 4}, {8, 4, 4}, {1, 4, 32}};
    for (const auto& sh : shapes) {
        const double w = double(axis_work(od.x, sh[0], s.x, k.x, v0.x, vn.x)) *
                         double(axis_work(od.y, sh[1], s.y, k.y, v0.y, vn.y)) *
                         double(axis_work(od.z, sh[2], s.z, k.z, v0.z, vn.z));
        if (w < bw) bw = w, best.box = 1, best.bx = sh[0], best.by = sh[1], best.bz = sh[2];
    }
    return best;
}

// One valid convolution src[B][f_src][sd] -> out[B][n_real][sd - s(k-1)] on
// the tensor cores. wmode selects how the B panel is built from w; only the
// source box [v0, v0 + vn) can be nonzero (the rest is zero halo).
void launch_valid(cudaStream_t st, int64_t Bn, int f_src, int n_real, int f_in_w, dims3 sd, dims3 k, dims3 s,
                  const float* srcp, const float* w, int wmode, const float* bias, int act, float* outp,
                  char* wsp, dims3 v0, dims3 vn, const char* what) {
    const int T = int(k.vol());
    const int K = f_src * T;
    const int kpad = int(ceil_div(K, BK) * BK);
    const int64_t r16 = ceil_div(n_real, 16) * 16;
    const int nt = int(r16 <= 128 ? r16 : 128);
    const int ntiles = int(ceil_div(n_real, nt));
    const int npad = ntiles * nt;
    const dims3 od{sd.x - s.x * (k.x - 1), sd.y - s.y * (k.y - 1), sd.z - s.z * (k.z - 1)};
    require(kpad / BK < 65536, "conv_tc: too many K-blocks");
    box_choice bc;
    const bool halo = v0.x > 0 || v0.y > 0 || v0.z > 0;
    // measured on c5's s = 4 layers: box tiles cut the MMAs by 15-25% but the
    // tap-major gathers lose the L1 reuse of the (wx, wy)-outer order and the
    // pass gets ~4% slower, so box tiles are opt-in (ZNN_CONV_BOX=1)
    if (halo && std::getenv("ZNN_CONV_BOX")) bc = choose_box(od, k, s, v0, vn);
    // box tiles skip single taps: channel-blocked tap-major K (block = the
    // largest divisor of f_src <= 32)
    int order = 0;
    if (bc.box) {
        order = 1;
        for (int cb = std::min(f_src, 32); cb >= 1; --cb)
            if (f_src % cb == 0) {
                order = cb;
                break;
            }
    }

    const size_t panel = size_t(npad) * size_t(kpad);
    float* hi = reinterpret_cast<float*>(wsp);
    float* lo = hi + panel;
    int* tab = reinterpret_cast<int*>((reinterpret_cast<uintptr_t>(lo + panel) + 255) & ~uintptr_t(255));

    int64_t blocks = ceil_div(int64_t(panel), 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    split_weights_k<<<unsigned(blocks), 256, 0, st>>>(w, n_real, f_src, f_in_w, T, int(k.y), int(k.z), K, npad, kpad,
                                                      wmode, order, hi, lo);
    launch_check("conv_tc_split_weights");
    koff_k<<<unsigned(ceil_div(kpad, 256)), 256, 0, st>>>(tab, K, kpad, f_src, int(k.x), int(k.y), int(k.z), order,
                                                           int(s.x),
                                                           int(s.y), int(s.z), sd.vol(), int(sd.y), int(sd.z));
    launch_check("conv_tc_koff");

    const CUtensorMap mhi = make_panel_map(hi, kpad, npad, nt);
    const CUtensorMap mlo = make_panel_map(lo, kpad, npad, nt);
    tc_params p;
    p.f_src = f_src;
    p.n_real = n_real;
    p.nt = nt;
    p.kblocks = kpad / BK;
    p.K = K;
    const int ntmax = nt <= 32 ? 32 : (nt <= 64 ? 64 : 128);
    p.bstride = ntmax;
    p.nbuf = ntmax == 128 ? 2 : 4;  // + na x 64 A columns <= 512 TMEM columns
    // producer warpgroups: 3 for short K (gathers dominate: c5's first layer
    // 9.0 -> 7.9 ms), 2 for long K (the MMA dominates; 3 measured ~1% slower)
    int ng = p.kblocks <= 64 ? 3 : 2;
    if (const char* e = std::getenv("ZNN_CONV_NG")) ng = std::atoi(e) == 3 ? 3 : 2;
    p.na = ng == 3 ? 3 : 4;  // A buffers: two per group (NG = 2) or one per group (NG = 3)
    p.vox_out = od.vol();
    p.rows = Bn * p.vox_out;
    p.ox = int(od.x), p.oy = int(od.y), p.oz = int(od.z);
    p.sx = int(sd.x), p.sy = int(sd.y), p.sz = int(sd.z);
    p.src_vol = sd.vol();
    p.gsize = order ? order : f_src * int(k.z);
    p.taps = T;
    p.ky = int(k.y), p.kz = int(k.z);
    p.dsx = int(s.x), p.dsy = int(s.y), p.dsz = int(s.z);
    p.vx0 = int(v0.x), p.vx1 = int(v0.x + vn.x - 1), p.vy0 = int(v0.y), p.vy1 = int(v0.y + vn.y - 1);
    p.vz0 = int(v0.z), p.vz1 = int(v0.z + vn.z - 1);
    p.box = bc.box, p.bxs = bc.bx, p.bys = bc.by, p.bzs = bc.bz;
    p.tnx = bc.box ? int(ceil_div(od.x, bc.bx)) : 0;
    p.tny = bc.box ? int(ceil_div(od.y, bc.by)) : 0;
    p.tnz = bc.box ? int(ceil_div(od.z, bc.bz)) : 0;
    const int stage = 2 * nt * 128;
    const size_t fixed = 1024 + 8 * size_t(16) + 16 + 2 * size_t(p.kblocks) + 64;
    p.stages = int((size_t(220) * 1024 - fixed) / size_t(stage + 16));
    if (p.stages > 8) p.stages = 8;
    require(p.stages >= 2, "conv_tc: K too long for the shared-memory budget");
    const size_t smem = size_t(p.stages) * size_t(stage) + 8 * size_t(2 * p.stages + 16) + fixed;
    const int64_t mtiles = bc.box ? Bn * p.tnx * p.tny * p.tnz : ceil_div(p.rows, BM);
    const dim3 grid{unsigned(mtiles), unsigned(ntiles), 1u};
    if (ng == 3) {
        if (ntmax == 32) launch_kernel<32, 3>(grid, smem, st, mhi, mlo, srcp, tab, outp, bias, act, p, what);
        else if (ntmax == 64) launch_kernel<64, 3>(grid, smem, st, mhi, mlo, srcp, tab, outp, bias, act, p, what);
        else launch_kernel<128, 3>(grid, smem, st, mhi, mlo, srcp, tab, outp, bias, act, p, what);
    } else {
        if (ntmax == 32) launch_kernel<32, 2>(grid, smem, st, mhi, mlo, srcp, tab, outp, bias, act, p, what);
        else if (ntmax == 64) launch_kernel<64, 2>(grid, smem, st, mhi, mlo, srcp, tab, outp, bias, act, p, what);
        else launch_kernel<128, 2>(grid, smem, st, mhi, mlo, srcp, tab, outp, bias, act, p, what);
    }
}

size_t panel_bytes(int f_src, int n_real, int64_t T) {
    const int64_t kpad = ceil_div(int64_t(f_src) * T, BK) * BK;
    const int64_t npad = ceil_div(n_real, 16) * 16 + 128;
    return sizeof(float) * size_t(npad * kpad) * 2 + sizeof(int) * size_t(kpad) + 512;
}

}  // namespace

// 2D TMA map over a row-major fp32 panel [rows][cols] (cols * 4 B a multiple
// of 16), box = 32 columns (one 128 B swizzle row) x box_rows rows, SWIZZLE_128B.
// the driver entry point of cuTensorMapEncodeTiled (shared with bgemm_tc.cu)
void* tensor_map_encoder() { return reinterpret_cast<void*>(encoder()); }

CUtensorMap make_panel_map_rows(const float* ptr, int64_t cols, int64_t rows, int box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    const cuuint64_t strides[1] = {cuuint64_t(cols) * sizeof(float)};
    const cuuint32_t box[2] = {cuuint32_t(BK), cuuint32_t(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    require(cols % 4 == 0, "tma panel: row pitch must be a multiple of 16 bytes");
    CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw cuda_error("cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
    return m;
}

namespace {
CUtensorMap make_panel_map(const float* ptr, int kpad, int rows, int nt) {
    return make_panel_map_rows(ptr, kpad, rows, nt);
}
}  // namespace

bool conv_tc_supported(const conv_shape& c, int pass) {
    if (pass == 0) return c.f_out >= 16 && c.f_in * c.n.vol() < (int64_t(1) << 31);
    if (pass == 1) {
        const int64_t pv = (c.m.x + 2 * c.s.x * (c.k.x - 1)) * (c.m.y + 2 * c.s.y * (c.k.y - 1)) *
                           (c.m.z + 2 * c.s.z * (c.k.z - 1));
        return c.f_in >= 16 && c.f_out * pv < (int64_t(1) << 31);
    }
    return c.f_out >= 16 && c.n.vol() * c.f_in < (int64_t(1) << 31);
}

namespace {
std::string tc_label(const char* k, const conv_shape& c) {
    return std::string(k) + " f=" + std::to_string(c.f_in) + "->" + std::to_string(c.f_out) + " n=" +
           std::to_string(c.n.x) + " k=" + std::to_string(c.k.x) + " s=" + std::to_string(c.s.x) + " B=" +
           std::to_string(c.B);
}
double tc_flops(const conv_shape& c) { return 2.0 * double(c.B * c.f_in * c.f_out) * double(c.m.vol() * c.taps()); }
}  // namespace

void conv_fwd_tc(cudaStream_t st, const conv_shape& c, const float* x, const float* w, const float* bias, int act,
                 float* y, scratch& ws) {
    prof_scope ps(st, tc_label("conv_fwd_tc", c), 4.0 * double(c.B) * double(c.f_in * c.n.vol() + c.f_out * c.m.vol()),
                  tc_flops(c));
    if (conv1_tc_supported(c) && !std::getenv("ZNN_CONV1_GENERIC")) {  // weights-resident single-input-map kernel
        conv1_fwd_tc(st, c, x, w, bias, act, y);
        return;
    }
    char* wsp = static_cast<char*>(ws.get(panel_bytes(int(c.f_in), int(c.f_out), c.taps())));
    launch_valid(st, c.B, int(c.f_in), int(c.f_out), int(c.f_in), c.n, c.k, c.s, x, w, 0, bias, act, y, wsp,
                 dims3{0, 0, 0}, c.n, "conv_fwd_tc");
}

void conv_dgrad_tc(cudaStream_t st, const conv_shape& c, const float* g, const float* w, float* dx, scratch& ws) {
    prof_scope ps(st, tc_label("conv_dgrad_tc", c), 4.0 * double(c.B) * double(c.f_in * c.n.vol() + c.f_out * c.m.vol()),
                  tc_flops(c));
    const dims3 P{c.s.x * (c.k.x - 1), c.s.y * (c.k.y - 1), c.s.z * (c.k.z - 1)};
    const dims3 gd{c.m.x + 2 * P.x, c.m.y + 2 * P.y, c.m.z + 2 * P.z};
    const size_t gbytes = sizeof(float) * size_t(c.B * c.f_out * gd.vol());
    const size_t gpad = (gbytes + 1023) & ~size_t(1023);
    char* wsp = static_cast<char*>(ws.get(gpad + panel_bytes(int(c.f_out), int(c.f_in), c.taps())));
    float* gp = reinterpret_cast<float*>(wsp);
    const int64_t pmaps = c.B * c.f_out;
    require(gd.x < 65536 && pmaps < 65536, "conv_dgrad_tc: halo grid exceeds 65535");
    const dim3 pgrid(unsigned(ceil_div(gd.y, 8)), unsigned(gd.x), unsigned(pmaps));
    pad_halo_k<<<pgrid, dim3(32, 8, 1), 0, st>>>(g, int(c.m.x), int(c.m.y), int(c.m.z), int(P.x), int(P.y), int(P.z),
                                                 gp);
    launch_check("conv_dgrad_tc_pad");
    launch_valid(st, c.B, int(c.f_out), int(c.f_in), int(c.f_in), gd, c.k, c.s, gp, w, 1, nullptr, 3, dx,
                 wsp + gpad, P, c.m, "conv_dgrad_tc");
}

}  // namespace znn_gpu
