// tcgen05 / TMA / mbarrier PTX helpers shared by the tensor-core conv
// kernels (sm_100a only).
#pragma once

#include <cuda.h>

#include <cstdint>

namespace znn_tc {

constexpr int BM = 128;  // tile rows = TMEM lanes
constexpr int BK = 32;   // fp32 K elements per stage (one 128 B swizzle row)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// non-blocking probe of a phase (for warps that poll while doing other work)
__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
        "[%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}
// multicast variant: the same smem offset / mbarrier offset in every CTA of
// ctaMask (cluster ranks) receives the box and its complete_tx
__device__ __forceinline__ void tma_load_2d_mc(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                               uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster "
        "[%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "h"(mask)
        : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile(
        "{\n\t.reg .pred pe;\n\t"
        "elect.sync _|pe, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, pe;\n\t}"
        : "=r"(pred));
    return pred != 0;
}
// ---- CTA-pair (cta_group::2) helpers ----
// shared::cluster address of the same shared variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_cluster(uint32_t bar_cluster, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(bar_cluster),
                 "r"(bytes)
                 : "memory");
}
// TMA into this CTA's shared memory, completion counted on the pair leader's barrier
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                                                 int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
        "[%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tmem_alloc_pair(uint32_t slot_smem, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(slot_smem), "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t tmem, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols));
}
// pair MMA (issued by the leader CTA): M = 256 rows (128 from each CTA's
// TMEM), B halves from both CTAs' shared memory, D in both CTAs' TMEM
__device__ __forceinline__ void mma_tf32_ts_pair_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                                   uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred pe, pa;\n\t"
        "elect.sync _|pe, 0xffffffff;\n\t"
        "setp.ne.b32 pa, %4, 0;\n\t"
        "@pe tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, pa;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit_pair_mc_w(uint32_t bar, uint16_t mask) {
    asm volatile(
        "{\n\t.reg .pred pe;\n\t"
        "elect.sync _|pe, 0xffffffff;\n\t"
        "@pe tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
            bar),
        "h"(mask)
        : "memory");
}

// warpgroup register rebalancing (all 128 threads of the warpgroup execute it)
template <int N>
__device__ __forceinline__ void setmaxnreg_inc() {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void setmaxnreg_dec() {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_alloc(uint32_t slot_smem, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(slot_smem), "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t tmem, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols));
}

// D[tmem] (+)= A[smem] * B[smem]^T, kind::tf32, fp32 accumulate
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// D[tmem] (+)= A[tmem] * B[smem]^T, kind::tf32 (A read from TMEM: lane = row,
// one 32-bit column per K element)
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                            uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}
// Warp-collective issue: every lane of the (converged) warp executes these and
// one elected lane issues. Keeping the issuing warp converged avoids the
// per-instruction ELECT/branch loops the compiler wraps around tcgen05 ops
// executed under a divergent `if (lane == 0)`.
__device__ __forceinline__ void mma_tf32_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                              uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred pe, pa;\n\t"
        "elect.sync _|pe, 0xffffffff;\n\t"
        "setp.ne.b32 pa, %4, 0;\n\t"
        "@pe tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, pa;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit_w(uint32_t bar) {
    asm volatile(
        "{\n\t.reg .pred pe;\n\t"
        "elect.sync _|pe, 0xffffffff;\n\t"
        "@pe tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
        : "memory");
}
__device__ __forceinline__ void mma_commit_mc_w(uint32_t bar, uint16_t mask) {
    asm volatile(
        "{\n\t.reg .pred pe;\n\t"
        "elect.sync _|pe, 0xffffffff;\n\t"
        "@pe tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
            bar),
        "h"(mask)
        : "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, kind::tf32, issued by one elected lane of a converged warp
__device__ __forceinline__ void mma_tf32_w(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred pe, pa;\n\t"
        "elect.sync _|pe, 0xffffffff;\n\t"
        "setp.ne.b32 pa, %4, 0;\n\t"
        "@pe tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, pa;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// one 2D TMA box into shared memory, issued by one elected lane of a converged
// warp; completion counted on `bar` (armed separately with expect_tx)
__device__ __forceinline__ void tma_w(uint32_t bar, uint32_t dst, const CUtensorMap* m, int c0, int c1) {
    asm volatile(
        "{\n\t.reg .pred pe;\n\t"
        "elect.sync _|pe, 0xffffffff;\n\t"
        "@pe cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n\t}" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
// L2 prefetch of a TMA box (no shared memory, no barrier)
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1)
                 : "memory");
}
// converged-warp TMA issue (one elected lane arms the barrier and loads)
__device__ __forceinline__ void tma_pair_w(uint32_t bar, uint32_t bytes, uint32_t dst0, const CUtensorMap* m0,
                                           uint32_t dst1, const CUtensorMap* m1, int c0, int c1) {
    asm volatile(
        "{\n\t.reg .pred pe;\n\t"
        "elect.sync _|pe, 0xffffffff;\n\t"
        "@pe mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t"
        "@pe cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%2], [%3, {%6, %7}], [%0];\n\t"
        "@pe cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%4], [%5, {%6, %7}], [%0];\n\t}" ::"r"(
            bar),
        "r"(bytes), "r"(dst0), "l"(reinterpret_cast<uint64_t>(m0)), "r"(dst1), "l"(reinterpret_cast<uint64_t>(m1)),
        "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tma_pair_mc_w(uint32_t bar, uint32_t bytes, uint32_t dst0, const CUtensorMap* m0,
                                              uint32_t dst1, const CUtensorMap* m1, int c0, int c1, uint16_t mask) {
    asm volatile(
        "{\n\t.reg .pred pe;\n\t"
        "elect.sync _|pe, 0xffffffff;\n\t"
        "@pe mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t"
        "@pe cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster [%2], [%3, {%6, %7}], [%0], %8;\n\t"
        "@pe cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster [%4], [%5, {%6, %7}], [%0], %8;\n\t}" ::"r"(
            bar),
        "r"(bytes), "r"(dst0), "l"(reinterpret_cast<uint64_t>(m0)), "r"(dst1), "l"(reinterpret_cast<uint64_t>(m1)),
        "r"(c0), "r"(c1), "h"(mask)
        : "memory");
}
// arrive on the same mbarrier offset in every CTA of ctaMask when this
// thread's prior MMAs complete
__device__ __forceinline__ void mma_commit_mc(uint32_t bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            bar),
        "h"(mask)
        : "memory");
}
// instruction descriptor: D f32, A/B tf32, both K-major, M x N
__host__ __device__ __forceinline__ uint32_t idesc_tf32(int m, int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}

// K-major, SWIZZLE_128B smem matrix descriptor: rows of 128 B, 8-row atoms
// 1024 B apart (SBO), descriptor version 1 (sm_100), layout 2 = 128B swizzle.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr) {
    uint64_t d = 0;
    d |= uint64_t((addr >> 4) & 0x3FFF);
    d |= uint64_t(1) << 16;
    d |= uint64_t(1024 >> 4) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(2) << 61;
    return d;
}
// byte offset of element (row r, k j) in a 128B-swizzled K-major tile
__device__ __forceinline__ uint32_t sw128_off(uint32_t r, uint32_t j) {
    return r * 128u + ((((j >> 2) ^ (r & 7u)) << 4) | ((j & 3u) << 2));
}

__device__ __forceinline__ float tf32_hi(float v) { return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); }
__device__ __forceinline__ float tf32_rn(float v) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
    return __uint_as_float(r);
}

__device__ __forceinline__ void tmem_ld16(uint32_t addr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
// 8 consecutive 32-bit TMEM columns of this thread's lane (warp-collective)
__device__ __forceinline__ void tmem_st8(uint32_t addr, const float (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(addr),
                 "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
                 "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
                 "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Accumulator drain: tensor-core fp32 accumulation loses precision roughly
// linearly in the number of accumulating MMAs, so the K loop is cut into
// chunks that each start from a fresh TMEM buffer; drain warps add every
// finished chunk into fp32 registers (round-to-nearest) while the MMA warp
// fills the next buffer. NTMAX = compile-time bound on the tile width.
template <int NTMAX>
struct drain_acc {
    float acc[NTMAX];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < NTMAX; ++i) acc[i] = 0.f;
    }
    // add TMEM columns [buf, buf+nt) of this thread's lane into acc
    __device__ __forceinline__ void add(uint32_t lane_addr, int nt) {
#pragma unroll
        for (int c0 = 0; c0 < NTMAX; c0 += 16) {
            if (c0 < nt) {
                float v[16];
                tmem_ld16(lane_addr + uint32_t(c0), v);
                tmem_wait_ld();
#pragma unroll
                for (int q = 0; q < 16; ++q) acc[c0 + q] += v[q];
            }
        }
    }
};

// Drain state for a producer warp that also owns a quarter of the TMEM
// lanes: chunks are drained opportunistically (poll) between K-blocks and
// while waiting for a free smem stage, so a producer can never deadlock
// against an MMA warp that waits for a drained buffer. Warp-uniform control
// flow: the readiness test is broadcast from lane 0 and every lane then does
// its own (immediately successful) acquire wait.
// Every producer warp drains a column range [col0, col0+ncols) of its TMEM
// lane quarter (warp % 4), so two warps share one quarter and each keeps only
// NH accumulators in registers.
template <int NH>
struct chunk_drainer {
    drain_acc<NH> A;
    int next = 0;
    int buf = 0;          // next % nbuf, tracked incrementally (no integer division in the poll loop)
    uint32_t phase = 0;   // (next / nbuf) & 1
    uint32_t accf0, acce0, lane_base;
    int nbuf, bstride, ncols, nchunks;

    __device__ __forceinline__ void init(uint32_t f0, uint32_t e0, uint32_t lb, int nb, int bs, int nc_cols,
                                         int nc) {
        accf0 = f0, acce0 = e0, lane_base = lb, nbuf = nb, bstride = bs, ncols = nc_cols, nchunks = nc;
        next = 0, buf = 0, phase = 0;
        A.zero();
    }
    uint32_t acce_leader = 0;  // != 0: CTA pair, one elected arrive per warp on the leader's barrier
    __device__ __forceinline__ void drain_one() {
        mbar_wait(accf0 + 8u * uint32_t(buf), phase);
        tc_fence_after();
        if (ncols > 0) A.add(lane_base + uint32_t(buf * bstride), ncols);
        tc_fence_before();
        if (acce_leader) {
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mbar_arrive_cluster(acce_leader + 8u * uint32_t(buf));
        } else {
            mbar_arrive(acce0 + 8u * uint32_t(buf));
        }
        ++next;
        if (++buf == nbuf) buf = 0, phase ^= 1u;
    }
    __device__ __forceinline__ void poll() {
        while (next < nchunks) {
            const bool ready = __shfl_sync(0xffffffffu, mbar_test(accf0 + 8u * uint32_t(buf), phase) ? 1 : 0, 0);
            if (!ready) break;
            drain_one();
        }
    }
    __device__ __forceinline__ void finish() {
        while (next < nchunks) drain_one();
    }
    // wait for a free smem stage, draining finished chunks meanwhile
    __device__ __forceinline__ void wait_stage(uint32_t empty, uint32_t parity) {
        while (!__all_sync(0xffffffffu, mbar_test(empty, parity))) poll();
    }
};

}  // namespace znn_tc
