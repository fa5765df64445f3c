// Direct 3D (dilated) convolution as a tcgen05 implicit GEMM, 3xTF32.
//
// GEMM view (one CTA = 128 output voxels x NT output maps):
//   D[v][n] = sum_k A[v][k] * B[n][k]
//   fwd   : v = output voxel (b, o_xyz), n = output map, k = (input map c, tap w),
//           A[v][k] = x[b][c][o + s*w]            (conv_direct.hpp:39-68)
//   dgrad : v = input voxel (b, t_xyz),  n = input map,  k = (output map o, tap w),
//           A[v][k] = g[b][o][t - s*w] (0 outside) (conv_direct.hpp:74-101 with reflect)
// The convergent-edge sum of the reference (engine.hpp:345-353,
// sum_accumulator.hpp) is the K loop, accumulated in TMEM: no atomics, no
// locks. fp32 accuracy with tensor cores: every operand is split into
// hi = tf32(x) and lo = tf32(x - hi) and D += Ahi*Bhi + Ahi*Blo + Alo*Bhi.
//
// Warp roles (192 threads, 1 CTA per SM):
//   warps 0-3 : im2col producers for A (one voxel row per thread, 32 k per
//               K-block, hi/lo split in registers, 128B-swizzled K-major
//               stores), then the epilogue (TMEM -> regs -> bias + transfer
//               -> coalesced global stores)
//   warp 4    : TMA producer for B (pre-split weight panels, SWIZZLE_128B)
//   warp 5    : TMEM allocator + single-thread tcgen05.mma issuer
// mbarrier ring: full[s] (128 producer arrivals + TMA tx bytes), empty[s]
// (tcgen05.commit), done (final commit -> epilogue).
#include <cuda.h>

#include "ops.hpp"
#include "tc_common.cuh"

namespace znn_gpu {

namespace {

using namespace znn_tc;

constexpr int THREADS = 320;     // 4 producer + 4 drain/epilogue + TMA + MMA warps
constexpr uint32_t TMEM_COLS = 512;
constexpr int CHUNK_KB = 8;      // K-blocks accumulated per TMEM buffer before a drain

struct tc_params {
    int f_src;        // channels of the im2col source
    int n_real;       // real N (output maps of this GEMM)
    int nt;           // N tile (multiple of 16, <= NTMAX)
    int kblocks;
    int stages;
    int nbuf;         // TMEM accumulator buffers
    int bstride;      // TMEM columns per buffer
    int64_t rows;     // B * vox_out
    int64_t vox_out;  // voxels per output map
    int ox, oy, oz;   // output dims
    int sx, sy, sz;   // source dims
    int64_t src_vol;
};

template <bool DGRAD, int NTMAX>
__global__ void __launch_bounds__(THREADS, 1)
conv_tc_kernel(const __grid_constant__ CUtensorMap tm_hi, const __grid_constant__ CUtensorMap tm_lo,
               const float* __restrict__ src, const int4* __restrict__ ktab,
               float* __restrict__ out, const float* __restrict__ bias, int act, tc_params p) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* base_ptr = smem_raw + (base - raw);
    const uint32_t b_bytes = uint32_t(p.nt) * 128u;
    const uint32_t stage_bytes = 2u * BM * 128u + 2u * b_bytes;
    const uint32_t bar_base = base + uint32_t(p.stages) * stage_bytes;
    auto full_bar = [&](int s) { return bar_base + 8u * uint32_t(s); };
    auto empty_bar = [&](int s) { return bar_base + 8u * uint32_t(p.stages + s); };
    auto accf_bar = [&](int b) { return bar_base + 8u * uint32_t(2 * p.stages + b); };
    auto acce_bar = [&](int b) { return bar_base + 8u * uint32_t(2 * p.stages + 4 + b); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base_ptr + (bar_base - base) + 8u * uint32_t(2 * p.stages + 8));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t m0 = int64_t(blockIdx.x) * BM;
    const int n0 = blockIdx.y * p.nt;
    const int nchunks = (p.kblocks + CHUNK_KB - 1) / CHUNK_KB;

    if (threadIdx.x == 0) {
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(full_bar(s), 128 + 1);
            mbar_init(empty_bar(s), 1);
        }
        for (int b = 0; b < 4; ++b) {
            mbar_init(accf_bar(b), 1);
            mbar_init(acce_bar(b), 128);
        }
        fence_barrier_init();
    }
    if (warp == 9) tmem_alloc(smem_u32(tmem_slot), TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < 4) {
        // ---------------- im2col producer (one voxel row per thread) ----------------
        const int r = threadIdx.x;
        const int64_t v = m0 + r;
        const bool vok = v < p.rows;
        int64_t sbase = 0;
        int tx = 0, ty = 0, tz = 0;
        if (vok) {
            const int64_t b = v / p.vox_out;
            const int64_t rem = v - b * p.vox_out;
            tx = int(rem / (int64_t(p.oy) * p.oz));
            ty = int((rem / p.oz) % p.oy);
            tz = int(rem % p.oz);
            sbase = b * int64_t(p.f_src) * p.src_vol;
            if (!DGRAD) sbase += (int64_t(tx) * p.sy + ty) * p.sz + tz;
        }
        const uint32_t row_off = uint32_t(r) * 128u;
        const uint32_t sw = uint32_t(r & 7);
        const float* sp = src + sbase;  // 32-bit offsets from here on (map * f_src < 2^31)
        const int syz = p.sy * p.sz;
        const int tlin = tx * syz + ty * p.sz + tz;
        for (int kb = 0; kb < p.kblocks; ++kb) {
            const int s = kb % p.stages;
            const uint32_t ph = uint32_t(kb / p.stages) & 1u;
            float vals[BK];
            const int4* tb = ktab + kb * BK;
#pragma unroll
            for (int j = 0; j < BK; ++j) {
                const int4 e = __ldg(tb + j);
                float val = 0.f;
                if (vok) {
                    if (!DGRAD) {
                        val = __ldg(sp + e.x);
                    } else {
                        // e = {map offset, s*wx, s*wy, s*wz}; in-bounds test per axis
                        const int gx = tx - e.y, gy = ty - e.z, gz = tz - e.w;
                        if (unsigned(gx) < unsigned(p.sx) && unsigned(gy) < unsigned(p.sy) &&
                            unsigned(gz) < unsigned(p.sz))
                            val = __ldg(sp + (e.x + tlin));
                    }
                }
                vals[j] = val;
            }
            mbar_wait(empty_bar(s), ph ^ 1u);
            const uint32_t a_hi = base + uint32_t(s) * stage_bytes;
            const uint32_t a_lo = a_hi + BM * 128u;
#pragma unroll
            for (int c = 0; c < BK / 4; ++c) {
                float h[4], l[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    h[q] = tf32_hi(vals[4 * c + q]);
                    l[q] = tf32_rn(vals[4 * c + q] - h[q]);
                }
                const uint32_t off = row_off + ((uint32_t(c) ^ sw) << 4);
                asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a_hi + off), "f"(h[0]), "f"(h[1]),
                             "f"(h[2]), "f"(h[3]));
                asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a_lo + off), "f"(l[0]), "f"(l[1]),
                             "f"(l[2]), "f"(l[3]));
            }
            fence_proxy_async();
            mbar_arrive(full_bar(s));
        }
    } else if (warp < 8) {
        // ---------------- accumulator drain + epilogue ----------------
        const int r = threadIdx.x - 128;
        const uint32_t lane_base = tmem + (uint32_t((warp - 4) * 32) << 16);
        drain_acc<NTMAX> A;
        A.zero();
        for (int ch = 0; ch < nchunks; ++ch) {
            const int b = ch % p.nbuf;
            mbar_wait(accf_bar(b), uint32_t(ch / p.nbuf) & 1u);
            tc_fence_after();
            A.add(lane_base + uint32_t(b * p.bstride), p.nt);
            tc_fence_before();
            mbar_arrive(acce_bar(b));
        }
        const int64_t v = m0 + r;
        if (v < p.rows) {
            const int64_t bb = v / p.vox_out;
            const int64_t vin = v - bb * p.vox_out;
            const int64_t obase = bb * int64_t(p.n_real) * p.vox_out + vin;
#pragma unroll
            for (int q = 0; q < NTMAX; ++q) {
                const int n = n0 + q;
                if (q < p.nt && n < p.n_real) {
                    float val = A.acc[q];
                    if (!DGRAD) val = act_value(act, val + (bias ? __ldg(bias + n) : 0.f));
                    out[obase + int64_t(n) * p.vox_out] = val;
                }
            }
        }
    } else if (warp == 8) {
        // ---------------- TMA producer (pre-split weight panels) ----------------
        if (lane == 0) {
            for (int kb = 0; kb < p.kblocks; ++kb) {
                const int s = kb % p.stages;
                const uint32_t ph = uint32_t(kb / p.stages) & 1u;
                mbar_wait(empty_bar(s), ph ^ 1u);
                const uint32_t b_hi = base + uint32_t(s) * stage_bytes + 2u * BM * 128u;
                mbar_expect_tx(full_bar(s), 2u * b_bytes);
                tma_load_2d(b_hi, &tm_hi, full_bar(s), kb * BK, n0);
                tma_load_2d(b_hi + b_bytes, &tm_lo, full_bar(s), kb * BK, n0);
            }
        }
    } else {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            const uint32_t idesc = idesc_tf32(BM, p.nt);
            for (int kb = 0; kb < p.kblocks; ++kb) {
                const int ch = kb / CHUNK_KB;
                const int b = ch % p.nbuf;
                const bool first = (kb % CHUNK_KB) == 0;
                if (first) {
                    mbar_wait(acce_bar(b), (uint32_t(ch / p.nbuf) & 1u) ^ 1u);
                    tc_fence_after();
                }
                const uint32_t d = tmem + uint32_t(b * p.bstride);
                const int s = kb % p.stages;
                const uint32_t ph = uint32_t(kb / p.stages) & 1u;
                mbar_wait(full_bar(s), ph);
                tc_fence_after();
                const uint32_t a_hi = base + uint32_t(s) * stage_bytes;
                const uint32_t a_lo = a_hi + BM * 128u;
                const uint32_t b_hi = a_hi + 2u * BM * 128u;
                const uint32_t b_lo = b_hi + b_bytes;
#pragma unroll
                for (int kk = 0; kk < BK / 8; ++kk) {
                    const uint32_t koff = uint32_t(kk) * 32u;  // 8 tf32 = 32 B along K
                    const uint64_t ah = sw128_desc(a_hi + koff), al = sw128_desc(a_lo + koff);
                    const uint64_t bh = sw128_desc(b_hi + koff), bl = sw128_desc(b_lo + koff);
                    mma_tf32(d, ah, bh, idesc, (first && kk == 0) ? 0u : 1u);
                    mma_tf32(d, ah, bl, idesc, 1u);
                    mma_tf32(d, al, bh, idesc, 1u);
                }
                mma_commit(empty_bar(s));
                if ((kb % CHUNK_KB) == CHUNK_KB - 1 || kb == p.kblocks - 1) mma_commit(accf_bar(b));
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 9) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc(tmem, TMEM_COLS);
    }
}

// Weight panels for the B operand, split hi/lo, zero padded to [npad][kpad].
//   fwd  : B[n][k] = W[n][k]                (k = c*T + w)
//   dgrad: B[n][k] = W[o][n][w], k = o*T + w
__global__ void split_weights_k(const float* __restrict__ w, int n_real, int other, int T, int K, int npad,
                                int kpad, int dgrad, float* __restrict__ hi, float* __restrict__ lo) {
    const int64_t total = int64_t(npad) * kpad;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
        const int n = int(i / kpad), k = int(i - int64_t(n) * kpad);
        float v = 0.f;
        if (n < n_real && k < K) {
            if (!dgrad) {
                v = w[int64_t(n) * K + k];
            } else {
                const int o = k / T, t = k - o * T;
                v = w[(int64_t(o) * other + n) * T + t];
            }
        }
        const float h = tf32_hi(v);
        hi[i] = h;
        lo[i] = tf32_rn(v - h);
    }
}

// K table: fwd {c*src_vol + tap offset, 0,0,0}; dgrad {c*src_vol, sx*wx, sy*wy, sz*wz};
// padded k: fwd -> offset 0 (weights are zero there), dgrad -> out of bounds.
__global__ void ktab_k(int4* __restrict__ tab, int K, int kpad, int T, int ky, int kz, int sx, int sy, int sz,
                       int64_t src_vol, int src_y, int src_z, int dgrad) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < kpad; k += gridDim.x * blockDim.x) {
        int4 e = make_int4(0, 0, 0, 0);
        if (k < K) {
            const int c = k / T, t = k - c * T;
            const int wx = t / (ky * kz), wy = (t / kz) % ky, wz = t % kz;
            if (!dgrad) {
                e.x = int(int64_t(c) * src_vol + (int64_t(sx * wx) * src_y + sy * wy) * src_z + sz * wz);
            } else {
                // map offset minus the linear tap shift: address = e.x + linear(t)
                e = make_int4(int(int64_t(c) * src_vol - (int64_t(sx * wx) * src_y + sy * wy) * src_z - sz * wz),
                              sx * wx, sy * wy, sz * wz);
            }
        } else if (dgrad) {
            e = make_int4(0, 1 << 29, 1 << 29, 1 << 29);
        }
        tab[k] = e;
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

CUtensorMap make_panel_map(const float* ptr, int kpad, int rows, int nt) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {cuuint64_t(kpad), cuuint64_t(rows)};
    const cuuint64_t strides[1] = {cuuint64_t(kpad) * sizeof(float)};
    const cuuint32_t box[2] = {cuuint32_t(BK), cuuint32_t(nt)};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw cuda_error("cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
    return m;
}

int pick_nt(int64_t n_real) {
    const int64_t r16 = ceil_div(n_real, 16) * 16;
    return int(r16 <= 128 ? r16 : 128);
}

int pick_stages(int nt) {
    const int stage = 2 * BM * 128 + 2 * nt * 128;
    int s = (220 * 1024) / stage;
    if (s > 6) s = 6;
    return s;
}

size_t smem_bytes(int nt, int stages) {
    return size_t(stages) * size_t(2 * BM * 128 + 2 * nt * 128) + 8 * size_t(2 * stages + 8) + 16 + 1024;
}

template <bool DGRAD, int NTMAX>
void launch_kernel(dim3 grid, size_t smem, cudaStream_t st, const CUtensorMap& mhi, const CUtensorMap& mlo,
                   const float* srcp, const int4* tab, float* outp, const float* bias, int act, const tc_params& p) {
    auto* k = conv_tc_kernel<DGRAD, NTMAX>;
    ZNN_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    k<<<grid, THREADS, smem, st>>>(mhi, mlo, srcp, tab, outp, bias, act, p);
    launch_check(DGRAD ? "conv_dgrad_tc" : "conv_fwd_tc");
}

void launch_tc(cudaStream_t st, bool dgrad, const conv_shape& c, const float* srcp, const float* w,
               const float* bias, int act, float* outp, scratch& ws) {
    const int T = int(c.taps());
    const int f_src = int(dgrad ? c.f_out : c.f_in);
    const int n_real = int(dgrad ? c.f_in : c.f_out);
    const int K = f_src * T;
    const int kpad = int(ceil_div(K, BK) * BK);
    const int nt = pick_nt(n_real);
    const int ntiles = int(ceil_div(n_real, nt));
    const int npad = ntiles * nt;
    const dims3 src = dgrad ? c.m : c.n;
    const dims3 od = dgrad ? c.n : c.m;

    const size_t panel = size_t(npad) * size_t(kpad);
    char* wsp = static_cast<char*>(ws.get(sizeof(float) * panel * 2 + sizeof(int4) * size_t(kpad) + 256));
    float* hi = reinterpret_cast<float*>(wsp);
    float* lo = hi + panel;
    int4* tab = reinterpret_cast<int4*>((reinterpret_cast<uintptr_t>(lo + panel) + 255) & ~uintptr_t(255));

    int64_t blocks = ceil_div(int64_t(panel), 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    split_weights_k<<<unsigned(blocks), 256, 0, st>>>(w, n_real, int(c.f_in), T, K, npad, kpad, dgrad ? 1 : 0, hi,
                                                      lo);
    launch_check("conv_tc_split_weights");
    ktab_k<<<unsigned(ceil_div(kpad, 256)), 256, 0, st>>>(tab, K, kpad, T, int(c.k.y), int(c.k.z), int(c.s.x),
                                                           int(c.s.y), int(c.s.z), src.vol(), int(src.y),
                                                           int(src.z), dgrad ? 1 : 0);
    launch_check("conv_tc_ktab");

    const CUtensorMap mhi = make_panel_map(hi, kpad, npad, nt);
    const CUtensorMap mlo = make_panel_map(lo, kpad, npad, nt);
    tc_params p;
    p.f_src = f_src;
    p.n_real = n_real;
    p.nt = nt;
    p.kblocks = kpad / BK;
    p.stages = pick_stages(nt);
    const int ntmax = nt <= 32 ? 32 : (nt <= 64 ? 64 : 128);
    p.bstride = ntmax;
    p.nbuf = 4;  // 4 x NTMAX <= 512 TMEM columns
    p.vox_out = od.vol();
    p.rows = c.B * p.vox_out;
    p.ox = int(od.x), p.oy = int(od.y), p.oz = int(od.z);
    p.sx = int(src.x), p.sy = int(src.y), p.sz = int(src.z);
    p.src_vol = src.vol();
    const size_t smem = smem_bytes(nt, p.stages);
    const dim3 grid(unsigned(ceil_div(p.rows, BM)), unsigned(ntiles));
    if (dgrad) {
        if (ntmax == 32) launch_kernel<true, 32>(grid, smem, st, mhi, mlo, srcp, tab, outp, nullptr, 3, p);
        else if (ntmax == 64) launch_kernel<true, 64>(grid, smem, st, mhi, mlo, srcp, tab, outp, nullptr, 3, p);
        else launch_kernel<true, 128>(grid, smem, st, mhi, mlo, srcp, tab, outp, nullptr, 3, p);
    } else {
        if (ntmax == 32) launch_kernel<false, 32>(grid, smem, st, mhi, mlo, srcp, tab, outp, bias, act, p);
        else if (ntmax == 64) launch_kernel<false, 64>(grid, smem, st, mhi, mlo, srcp, tab, outp, bias, act, p);
        else launch_kernel<false, 128>(grid, smem, st, mhi, mlo, srcp, tab, outp, bias, act, p);
    }
}

}  // namespace

bool conv_tc_supported(const conv_shape& c, int pass) {
    if (pass == 0) return c.f_out >= 16 && c.n.vol() < (int64_t(1) << 31) && c.f_in * c.taps() < (1 << 30);
    if (pass == 1) return c.f_in >= 16 && c.m.vol() < (int64_t(1) << 31) && c.f_out * c.taps() < (1 << 30);
    return c.f_out >= 16 && c.n.vol() * c.f_in < (int64_t(1) << 31);
}

void conv_fwd_tc(cudaStream_t st, const conv_shape& c, const float* x, const float* w, const float* bias, int act,
                 float* y, scratch& ws) {
    launch_tc(st, false, c, x, w, bias, act, y, ws);
}

void conv_dgrad_tc(cudaStream_t st, const conv_shape& c, const float* g, const float* w, float* dx, scratch& ws) {
    launch_tc(st, true, c, g, w, nullptr, 3, dx, ws);
}

}  // namespace znn_gpu
