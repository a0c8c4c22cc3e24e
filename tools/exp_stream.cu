// exp_stream.cu -- streaming microbenchmark for the fused-sweep memory pipeline
// (round-2 experiment, not product code).  Question: can tiles whose 12 bits are
// 4 contiguous low physical bits + 8 scattered bits be streamed through shared
// memory by 1D bulk-async copies (cp.async.bulk, UBLKCP) close to the copy
// roofline, with the CTA's threads only touching shared memory?
//
// Variants (psi + lambda, 2^30 complex64 amplitudes each, in place):
//   copy   plain contiguous LDG.128 / STG.128 in-place pass (calibration)
//   ldg    the round-1 skeleton style: each thread LDGs its 16 + 16 amplitudes
//          into registers, one smem exchange (STS, bar, LDS, bar), STG back;
//          L2 prefetch of the next tile; 2 CTAs / SM
//   bulk   warp-specialised: producer warp streams 128 B runs by cp.async.bulk
//          into an NSLOT ring (mbarrier complete_tx), consumer warps LDS ->
//          (trivial compute) -> STS in place, producer bulk-stores the slot back
//          (cp.async.bulk.global.shared::cta.bulk_group)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o exp_stream exp_stream.cu
#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <string>
#include <cstring>
#include <algorithm>

#define CK(x)                                                                                 \
    do {                                                                                      \
        cudaError_t e = (x);                                                                  \
        if (e != cudaSuccess) {                                                               \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
            exit(1);                                                                          \
        }                                                                                     \
    } while (0)

constexpr int NLOC = 30;
struct TileDesc {
    int k;                 // tile bits
    uint8_t pos[16];       // physical position of tile bit t (pos[0..3] = 0..3)
    uint8_t sorted[16];    // ascending
    uint64_t n_tiles;
};

__device__ __forceinline__ uint64_t deposit_tile(const TileDesc &T, uint64_t v) {
    // tile index -> base: insert zeros at the tile positions (ascending)
    for (int i = 0; i < T.k; i++) {
        const int p = T.sorted[i];
        v = ((v >> p) << (p + 1)) | (v & ((1ull << p) - 1));
    }
    return v;
}
__device__ __forceinline__ uint64_t tile_off(const TileDesc &T, uint32_t t) {
    uint64_t o = 0;
    for (int b = 0; b < T.k; b++)
        if ((t >> b) & 1) o |= 1ull << T.pos[b];
    return o;
}

// ---------------------------------------------------------------- copy
__global__ void copy_kernel(float4 *a, float4 *b, uint64_t n4) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x) {
        float4 x = __ldcs(a + i), y = __ldcs(b + i);
        x.x *= 1.0000001f;
        y.x *= 1.0000001f;
        __stcs(a + i, x);
        __stcs(b + i, y);
    }
}

// ---------------------------------------------------------------- ldg skeleton
// 256 threads: lanes = tile bits 0..4, warps = 5..7, registers = 8..11
template <bool XCH, bool PF, int MINB>
__global__ void __launch_bounds__(256, MINB) ldg_kernel(const __grid_constant__ TileDesc T, float2 *psi, float2 *lam, int work) {
    extern __shared__ __align__(16) float2 dsm[];
    float2 *sa = dsm, *sl = dsm + 4096;
    const int tid = threadIdx.x;
    uint64_t toff = 0, roff[16];
    toff = tile_off(T, tid);
    for (int r = 0; r < 16; r++) roff[r] = tile_off(T, (uint32_t)r << 8);
    for (uint64_t tile = blockIdx.x; tile < T.n_tiles; tile += gridDim.x) {
        const uint64_t base = deposit_tile(T, tile);
        if (PF && tile + gridDim.x < T.n_tiles) {
            const uint64_t nb = deposit_tile(T, tile + gridDim.x);
            // one line (16 amplitudes) per thread: lines are tile bits 4..11 (256 lines)
            const uint64_t e = nb + tile_off(T, (uint32_t)tid << 4);
            asm volatile("prefetch.global.L2 [%0];" ::"l"(psi + e));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(lam + e));
        }
        float2 a[16], l[16];
#pragma unroll
        for (int r = 0; r < 16; r++) {
            a[r] = __ldcs(psi + base + toff + roff[r]);
            l[r] = __ldcs(lam + base + toff + roff[r]);
        }
        if (!XCH) {
#pragma unroll
            for (int r = 0; r < 16; r++) {
                __stcs(psi + base + toff + roff[r], a[r]);
                __stcs(lam + base + toff + roff[r], l[r]);
            }
            continue;
        }
        for (int w = 0; w < work / 3; w++) {
#pragma unroll
            for (int r = 0; r < 16; r++) {
                a[r] = __ffma2_rn(a[r], make_float2(1.0f, 1.0f), l[r]);
                l[r] = __ffma2_rn(l[r], make_float2(1.0f, 1.0f), make_float2(-a[r].x, -a[r].y));
            }
        }
        // exchange 1: registers <-> warps (transpose bits 5..7 with 8..10)
#pragma unroll
        for (int r = 0; r < 16; r++) {
            sa[(r << 8) | tid] = a[r];
            sl[(r << 8) | tid] = l[r];
        }
        __syncthreads();
        const int tw = (tid & 31) | (((tid >> 5) & 7) << 8);
#pragma unroll
        for (int r = 0; r < 16; r++) {
            const int j = tw | ((r & 7) << 5) | ((r >> 3) << 11);
            a[r] = sa[j];
            l[r] = sl[j];
        }
        __syncthreads();
        for (int w = 0; w < work / 3; w++) {
#pragma unroll
            for (int r = 0; r < 16; r++) {
                a[r] = __ffma2_rn(a[r], make_float2(1.0f, 1.0f), l[r]);
                l[r] = __ffma2_rn(l[r], make_float2(1.0f, 1.0f), make_float2(-a[r].x, -a[r].y));
            }
        }
        // exchange 2 (back)
#pragma unroll
        for (int r = 0; r < 16; r++) {
            const int j = tw | ((r & 7) << 5) | ((r >> 3) << 11);
            sa[j] = a[r];
            sl[j] = l[r];
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 16; r++) {
            a[r] = sa[(r << 8) | tid];
            l[r] = sl[(r << 8) | tid];
        }
        __syncthreads();
        for (int w = 0; w < work / 3; w++) {
#pragma unroll
            for (int r = 0; r < 16; r++) {
                a[r] = __ffma2_rn(a[r], make_float2(1.0f, 1.0f), l[r]);
                l[r] = __ffma2_rn(l[r], make_float2(1.0f, 1.0f), make_float2(-a[r].x, -a[r].y));
            }
        }
#pragma unroll
        for (int r = 0; r < 16; r++) {
            const uint64_t off = base + toff + roff[r];
            __stcs(psi + off, a[r]);
            __stcs(lam + off, l[r]);
        }
    }
}

// ---------------------------------------------------------------- DSMEM cluster tile (k = 13)
// A 2-CTA cluster holds a 13-bit tile: tile bit 12 = the CTA rank.  Per tile: load the
// CTA's half (ldg, as ldg_kernel), exchange register bit 3 <-> the CTA bit through
// distributed shared memory (half of the data to the peer CTA), cluster barrier, read,
// exchange back, cluster barrier, store.  Same bytes per amplitude as ldg_kernel's two
// local exchanges.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1) dsmem_kernel(const __grid_constant__ TileDesc T,
                                                                                float2 *psi, float2 *lam) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) float2 dsm[];
    float2 *sa = dsm, *sl = dsm + 4096;
    const int tid = threadIdx.x;
    const unsigned rank = cl.block_rank();
    float2 *pa = cl.map_shared_rank(sa, rank ^ 1u), *pl = cl.map_shared_rank(sl, rank ^ 1u);
    uint64_t toff = tile_off(T, tid), roff[16];
    for (int r = 0; r < 16; r++) roff[r] = tile_off(T, (uint32_t)r << 8);
    const uint64_t coff = rank ? (1ull << T.pos[12]) : 0ull;
    const uint64_t n_cl = T.n_tiles;  // tiles of 13 bits
    for (uint64_t tile = blockIdx.x / 2; tile < n_cl; tile += gridDim.x / 2) {
        const uint64_t base = deposit_tile(T, tile) | coff;
        float2 a[16], l[16];
#pragma unroll
        for (int r = 0; r < 16; r++) {
            a[r] = __ldcs(psi + base + toff + roff[r]);
            l[r] = __ldcs(lam + base + toff + roff[r]);
        }
        for (int x = 0; x < 2; x++) {
            // element (rank c, thread t, reg r) -> (rank (r >> 3) & 1, t, (r & 7) | c << 3)
#pragma unroll
            for (int r = 0; r < 16; r++) {
                const int slot = (((r & 7) | (int)(rank << 3)) << 8) | tid;
                if (((r >> 3) & 1) == (int)rank) { sa[slot] = a[r]; sl[slot] = l[r]; }
                else { pa[slot] = a[r]; pl[slot] = l[r]; }
            }
            cl.sync();
#pragma unroll
            for (int r = 0; r < 16; r++) {
                a[r] = sa[(r << 8) | tid];
                l[r] = sl[(r << 8) | tid];
            }
            cl.sync();
        }
#pragma unroll
        for (int r = 0; r < 16; r++) {
            __stcs(psi + base + toff + roff[r], a[r]);
            __stcs(lam + base + toff + roff[r], l[r]);
        }
    }
}

// ---------------------------------------------------------------- bulk ring
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// slot = psi tile (2^k float2) then lambda tile; run j (16 amplitudes) of the tile
// lands at slot offset j * 128 B; consumers: lanes = tile bits 0..4, warps, regs.
template <int K, int NSLOT, int NCW>
__global__ void __launch_bounds__(32 * (NCW + 1), 1) bulk_kernel(const __grid_constant__ TileDesc T, float2 *psi, float2 *lam,
                                                                int work) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int TILE = 1 << K;
    constexpr int RUNS = TILE / 16;
    constexpr int NCT = 32 * NCW;            // consumer threads
    constexpr int NR = TILE / NCT;           // amplitudes per consumer thread per state
    float2 *slots = reinterpret_cast<float2 *>(smem);
    __shared__ __align__(8) uint64_t full[NSLOT], done[NSLOT];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < NSLOT; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&done[s], NCT);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint64_t n_my = T.n_tiles > blockIdx.x ? (T.n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (warp == NCW) {
        // producer warp: per lane the run offsets it moves (RUNS / 32 runs per state)
        constexpr int RPL = RUNS / 32;
        uint64_t roff[RPL];
        for (int i = 0; i < RPL; i++) roff[i] = tile_off(T, (uint32_t)(i * 32 + lane) << 4);
        for (uint64_t j = 0; j < n_my + NSLOT; j++) {
            const int s = (int)(j % NSLOT);
            float2 *sp = slots + (size_t)s * 2 * TILE;
            if (j >= NSLOT) {
                // tile j - NSLOT in slot s is computed: store it back
                const uint64_t jt = j - NSLOT;
                mbar_wait(&done[s], (uint32_t)((jt / NSLOT) & 1));
                const uint64_t base = deposit_tile(T, blockIdx.x + jt * gridDim.x);
                for (int i = 0; i < RPL; i++) {
                    const int run = i * 32 + lane;
                    bulk_s2g(psi + base + roff[i], sp + run * 16, 128);
                    bulk_s2g(lam + base + roff[i], sp + TILE + run * 16, 128);
                }
                bulk_commit();
                bulk_wait_read<0>();
                __syncwarp();
            }
            if (j < n_my) {
                const uint64_t base = deposit_tile(T, blockIdx.x + j * gridDim.x);
                if (lane == 0) mbar_expect_tx(&full[s], 2 * TILE * 8);
                __syncwarp();
                for (int i = 0; i < RPL; i++) {
                    const int run = i * 32 + lane;
                    bulk_g2s(sp + run * 16, psi + base + roff[i], 128, &full[s]);
                    bulk_g2s(sp + TILE + run * 16, lam + base + roff[i], 128, &full[s]);
                }
            }
        }
        return;
    }
    // consumers
    for (uint64_t j = 0; j < n_my; j++) {
        const int s = (int)(j % NSLOT);
        float2 *sp = slots + (size_t)s * 2 * TILE;
        mbar_wait(&full[s], (uint32_t)((j / NSLOT) & 1));
        float2 a[NR], l[NR];
#pragma unroll
        for (int r = 0; r < NR; r++) {
            a[r] = sp[r * NCT + tid];
            l[r] = sp[TILE + r * NCT + tid];
        }
        // stand-in compute: `work` dependent packed FMAs per amplitude pair
        for (int w = 0; w < work; w++) {
#pragma unroll
            for (int r = 0; r < NR; r++) {
                a[r] = __ffma2_rn(a[r], make_float2(1.0f, 1.0f), l[r]);
                l[r] = __ffma2_rn(l[r], make_float2(1.0f, 1.0f), make_float2(-a[r].x, -a[r].y));
            }
        }
#pragma unroll
        for (int r = 0; r < NR; r++) {
            sp[r * NCT + tid] = a[r];
            sp[TILE + r * NCT + tid] = l[r];
        }
        fence_async_smem();
        mbar_arrive(&done[s]);
    }
}

// ---------------------------------------------------------------- tensor TMA ring
// Tensor map (5D, 8-byte elements) of the shard: d0 = the 16 contiguous low
// amplitudes, d1 = an "offset" dimension (stride 128 B: any 16-amplitude-aligned
// base), d2..d4 = three scattered tile bits (size 2).  Box (16, 1, 2, 2, 2) =
// 128 amplitudes = 1 KB; the remaining LB = K - 7 tile bits are enumerated by the
// producer lanes (one box per lane and state).
__device__ __forceinline__ void tma_load5(void *dst, const CUtensorMap *tm, int c1, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
            smem_u32(dst)),
        "l"(tm), "r"(0), "r"(c1), "r"(0), "r"(0), "r"(0), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store5(const CUtensorMap *tm, int c1, const void *src) {
    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(tm),
                 "r"(0), "r"(c1), "r"(0), "r"(0), "r"(0), "r"(smem_u32(src))
                 : "memory");
}
template <int K, int NSLOT, int NCW>
__global__ void __launch_bounds__(32 * (NCW + 1), 1) tma_kernel(const __grid_constant__ TileDesc T, const __grid_constant__ CUtensorMap tmp,
                                                               const __grid_constant__ CUtensorMap tml, int work, int xch) {
    extern __shared__ __align__(1024) unsigned char smem[];
    constexpr int TILE = 1 << K;
    constexpr int LB = K - 7;                // tile bits enumerated by lanes
    constexpr int NCT = 32 * NCW;
    constexpr int NR = TILE / NCT;
    float2 *slots = reinterpret_cast<float2 *>(smem);
    __shared__ __align__(8) uint64_t full[NSLOT], done[NSLOT];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < NSLOT; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&done[s], NCT);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint64_t n_my = T.n_tiles > blockIdx.x ? (T.n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (warp == NCW) {
        const bool act = lane < (1 << LB);
        // offset of this lane's box within the tile (tile bits 7..K-1), in 128 B units
        uint64_t loff = 0;
        for (int b = 0; b < LB; b++)
            if ((lane >> b) & 1) loff |= 1ull << (T.pos[7 + b] - 4);
        for (uint64_t j = 0; j < n_my + NSLOT; j++) {
            const int s = (int)(j % NSLOT);
            float2 *sp = slots + (size_t)s * 2 * TILE;
            if (j >= NSLOT) {
                const uint64_t jt = j - NSLOT;
                mbar_wait(&done[s], (uint32_t)((jt / NSLOT) & 1));
                const uint64_t base = deposit_tile(T, blockIdx.x + jt * gridDim.x);
                if (act) {
                    const int c1 = (int)((base >> 4) + loff);
                    tma_store5(&tmp, c1, sp + lane * 128);
                    tma_store5(&tml, c1, sp + TILE + lane * 128);
                    bulk_commit();
                    bulk_wait_read<0>();
                }
                __syncwarp();
            }
            if (j < n_my) {
                const uint64_t base = deposit_tile(T, blockIdx.x + j * gridDim.x);
                if (lane == 0) mbar_expect_tx(&full[s], 2 * TILE * 8);
                __syncwarp();
                if (act) {
                    const int c1 = (int)((base >> 4) + loff);
                    tma_load5(sp + lane * 128, &tmp, c1, &full[s]);
                    tma_load5(sp + TILE + lane * 128, &tml, c1, &full[s]);
                }
            }
        }
        return;
    }
    for (uint64_t j = 0; j < n_my; j++) {
        const int s = (int)(j % NSLOT);
        float2 *sp = slots + (size_t)s * 2 * TILE;
        mbar_wait(&full[s], (uint32_t)((j / NSLOT) & 1));
        float2 a[NR], l[NR];
#pragma unroll
        for (int r = 0; r < NR; r++) {
            a[r] = sp[r * NCT + tid];
            l[r] = sp[TILE + r * NCT + tid];
        }
        // `work` packed-FMA rounds per amplitude pair in 3 segments, 2 exchanges
        // (STS -> consumer barrier -> LDS -> consumer barrier) in between
        for (int seg = 0; seg < 3; seg++) {
            if (seg > 0 && xch) {
#pragma unroll
                for (int r = 0; r < NR; r++) {
                    sp[(r * NCT + tid) ^ (seg << 5)] = a[r];
                    sp[TILE + ((r * NCT + tid) ^ (seg << 5))] = l[r];
                }
                asm volatile("bar.sync 1, %0;" ::"r"(NCT) : "memory");
#pragma unroll
                for (int r = 0; r < NR; r++) {
                    const int jj = ((r ^ 1) * NCT + tid) ^ (seg << 5);
                    a[r] = sp[jj];
                    l[r] = sp[TILE + jj];
                }
                asm volatile("bar.sync 1, %0;" ::"r"(NCT) : "memory");
            }
            for (int w = 0; w < work / 3; w++) {
#pragma unroll
                for (int r = 0; r < NR; r++) {
                    a[r] = __ffma2_rn(a[r], make_float2(1.0f, 1.0f), l[r]);
                    l[r] = __ffma2_rn(l[r], make_float2(1.0f, 1.0f), make_float2(-a[r].x, -a[r].y));
                }
            }
        }
#pragma unroll
        for (int r = 0; r < NR; r++) {
            sp[r * NCT + tid] = a[r];
            sp[TILE + r * NCT + tid] = l[r];
        }
        fence_async_smem();
        mbar_arrive(&done[s]);
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                             const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeFn get_encode() {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    return (EncodeFn)fn;
}
// tile bits 4..6 at T.pos[4..6] are the box's single-bit dimensions
static bool make_map(CUtensorMap *tm, void *base, const TileDesc &T, int nloc, int l2p) {
    cuuint64_t dims[5] = {16, (cuuint64_t)1 << (nloc - 4), 2, 2, 2};
    cuuint64_t strides[4] = {128, (cuuint64_t)8 << T.pos[4], (cuuint64_t)8 << T.pos[5], (cuuint64_t)8 << T.pos[6]};
    cuuint32_t box[5] = {16, 1, 2, 2, 2};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = get_encode()(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_NONE, (CUtensorMapL2promotion)l2p, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("{\"encode_error\": %d}\n", (int)r); return false; }
    return true;
}

static int g_work = 0;
int main(int argc, char **argv) {
    const char *which = argc > 1 ? argv[1] : "all";
    const uint64_t N = 1ull << NLOC;
    float2 *psi, *lam;
    CK(cudaMalloc(&psi, N * 8));
    CK(cudaMalloc(&lam, N * 8));
    CK(cudaMemset(psi, 0, N * 8));
    CK(cudaMemset(lam, 0, N * 8));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const double bytes = 32.0 * N;
    auto timeit = [&](const char *name, auto launch) {
        for (int i = 0; i < 3; i++) launch();
        CK(cudaDeviceSynchronize());
        const int reps = 10;
        CK(cudaEventRecord(e0));
        for (int i = 0; i < reps; i++) launch();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        ms /= reps;
        printf("{\"variant\": \"%s\", \"ms\": %.4f, \"GBps\": %.1f}\n", name, ms, bytes / (ms * 1e-3) / 1e9);
        fflush(stdout);
    };
    // a stage-like tile: low bits 0..3 + 8 scattered target bits
    TileDesc T;
    memset(&T, 0, sizeof(T));
    const int scat[8] = {5, 9, 12, 15, 18, 21, 25, 28};
    T.k = 12;
    for (int i = 0; i < 4; i++) T.pos[i] = i;
    for (int i = 0; i < 8; i++) T.pos[4 + i] = scat[i];
    for (int i = 0; i < 12; i++) T.sorted[i] = T.pos[i];
    T.n_tiles = N >> 12;
    TileDesc T11 = T;  // k = 11: drop the highest scattered bit
    T11.k = 11;
    T11.n_tiles = N >> 11;
    const std::string w(which);
    if (w == "all" || w == "copy")
        timeit("copy", [&] { copy_kernel<<<sms * 8, 256>>>((float4 *)psi, (float4 *)lam, N / 2); });
    TileDesc Tc = T;  // contiguous tile: bits 0..11
    for (int i = 0; i < 12; i++) Tc.pos[i] = Tc.sorted[i] = i;
    TileDesc T5 = T;  // 5 contiguous low bits (256 B runs) + 7 scattered
    {
        const int p5[12] = {0, 1, 2, 3, 4, 6, 9, 12, 15, 18, 21, 25};
        for (int i = 0; i < 12; i++) T5.pos[i] = T5.sorted[i] = p5[i];
    }
    auto run_ldg = [&](auto kern, const char *name, const TileDesc &TT, int ctas) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
        timeit(name, [&] { kern<<<sms * ctas, 256, 65536>>>(TT, psi, lam, g_work); });
    };
    if (w == "all" || w == "ldg") {
        for (int wk : {0, 24, 48, 96}) {
            g_work = wk;
            char nm[64];
            snprintf(nm, sizeof(nm), "ldg scat xch pf 2cta work=%d", wk);
            run_ldg(ldg_kernel<true, true, 2>, nm, T, 2);
        }
    }
    auto run_bulk = [&](auto kern, const char *name, const TileDesc &TT, int tile, int nslot, int ncw, int ctas,
                        int work) {
        const size_t sm = (size_t)nslot * 2 * tile * 8;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        char nm[128];
        snprintf(nm, sizeof(nm), "%s work=%d", name, work);
        timeit(nm, [&] { kern<<<sms * ctas, 32 * (ncw + 1), sm>>>(TT, psi, lam, work); });
    };
    for (int work : {0, 8, 24}) {
        if (w == "all" || w == "bulk") {
            run_bulk(bulk_kernel<12, 3, 8>, "bulk k12 3slot 8cw 1cta", T, 4096, 3, 8, 1, work);
            run_bulk(bulk_kernel<12, 3, 16>, "bulk k12 3slot 16cw 1cta", T, 4096, 3, 16, 1, work);
            run_bulk(bulk_kernel<11, 3, 8>, "bulk k11 3slot 8cw 2cta", T11, 2048, 3, 8, 2, work);
            run_bulk(bulk_kernel<11, 2, 8>, "bulk k11 2slot 8cw 2cta", T11, 2048, 2, 8, 2, work);
            run_bulk(bulk_kernel<11, 3, 4>, "bulk k11 3slot 4cw 2cta", T11, 2048, 3, 4, 2, work);
        }
    }

    if (w == "all" || w == "tma") {
        CUtensorMap mp, ml;
        if (make_map(&mp, psi, T, NLOC, 0) && make_map(&ml, lam, T, NLOC, 0)) {
            for (int work : {0, 24, 48, 96}) {
                auto go = [&](auto kern, const char *name, int nslot, int ncw) {
                    const size_t sm = (size_t)nslot * 2 * 4096 * 8;
                    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
                    char nm[128];
                    snprintf(nm, sizeof(nm), "%s xch work=%d", name, work);
                    timeit(nm, [&] { kern<<<sms, 32 * (ncw + 1), sm>>>(T, mp, ml, work, 1); });
                };
                go(tma_kernel<12, 2, 8>, "tma k12 2slot 8cw", 2, 8);
                go(tma_kernel<12, 3, 8>, "tma k12 3slot 8cw", 3, 8);
                go(tma_kernel<12, 3, 16>, "tma k12 3slot 16cw", 3, 16);
            }
        }
    }

    if (w == "all" || w == "dsmem") {
        TileDesc T13 = T;  // 13-bit tile: T's 12 bits + physical bit 30 -> use bit 29's neighbour
        T13.k = 13;
        const int p13[13] = {0, 1, 2, 3, 5, 9, 12, 15, 18, 21, 25, 28, 7};
        for (int i = 0; i < 13; i++) T13.pos[i] = p13[i];
        int srt[13];
        for (int i = 0; i < 13; i++) srt[i] = p13[i];
        std::sort(srt, srt + 13);
        for (int i = 0; i < 13; i++) T13.sorted[i] = srt[i];
        T13.n_tiles = N >> 13;
        CK(cudaFuncSetAttribute(dsmem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
        for (int ctas : {2, 4}) {
            char nm[64];
            snprintf(nm, sizeof(nm), "dsmem k13 cluster2 2xch %d CTAs/SM", ctas);
            timeit(nm, [&] { dsmem_kernel<<<sms * ctas, 256, 65536>>>(T13, psi, lam); });
        }
        g_work = 0;
        CK(cudaFuncSetAttribute(ldg_kernel<true, true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
        timeit("ldg k12 2xch (same bytes)", [&] { ldg_kernel<true, true, 2><<<sms * 2, 256, 65536>>>(T, psi, lam, 0); });
    }
    CK(cudaFree(psi));
    CK(cudaFree(lam));
    return 0;
}
