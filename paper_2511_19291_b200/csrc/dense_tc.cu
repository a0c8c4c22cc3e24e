// dense_tc.cu -- a fused dense m-qubit block on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, accumulators in TMEM), SURVEY.md §8(f) rank 4 and the
// north star's "tensor cores only if the fused block really becomes a dense
// 2^k x 2^k contraction worth it".  PAPER.md:91 (§3 "Extensible"): custom
// unitaries on any number of qubits.
//
// The block U (D = 2^m, here m = 6) acts on the m LOWEST physical bits: with the
// state viewed as rows of D contiguous amplitudes, every row transforms as
//   y = U x   <=>   y_row = x_row U^T,
// and in the real (re, im interleaved) representation of complex64 a row is 2D
// floats, so one 128-row tile is the real GEMM  Y[128 x 2D] = X[128 x 2D] B[2D x 2D]
// with B[2c][2j] = Re U_jc, B[2c+1][2j] = -Im U_jc, B[2c][2j+1] = Im U_jc,
// B[2c+1][2j+1] = Re U_jc.  Precision: 3xTF32 (x = x_hi + x_lo with x_hi the
// TF32 truncation; x B ~ x_hi B_hi + x_hi B_lo + x_lo B_hi, fp32 accumulation), or
// 1xTF32 for comparison.
//
// Kernel (one persistent CTA of 128 threads per SM; 192 KB shared memory):
//   B_hi, B_lo (2D x 2D, K-major canonical no-swizzle UMMA layout) loaded once;
//   per tile and K-half: the 128 x D floats of X split into hi / lo and stored in
//   the same layout, fence.proxy.async, one elected thread issues the
//   tcgen05.mma (M = 128, N = 2D = 128, K = 8 per instruction), tcgen05.commit to an
//   mbarrier; epilogue: tcgen05.ld (32 lanes x 32 columns per warp) -> registers
//   -> global, in place.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <vector>

namespace tqd {

namespace dtc {
constexpr int M = 128;        // tile rows (TMEM lanes)
constexpr int N = 128;        // 2D real columns (m = 6)
constexpr int KC = 64;        // K per shared-memory chunk (floats)
constexpr int THREADS = 256;  // 8 warps: loads / epilogue; warp w reads TMEM lanes 32 (w % 4)..

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// canonical K-major, no swizzle (cute UMMA INTERLEAVE): ((8,m),(4 floats,2k)) with the
// 8 rows of a core matrix 16 B apart, core matrices along K at LBO, along M at SBO
__host__ __device__ __forceinline__ uint32_t kmajor_off(int row, int k, int kdim) {
    return (uint32_t)((row >> 3) * (kdim / 4) * 128 + (k >> 2) * 128 + (row & 7) * 16 + (k & 3) * 4);
}
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);  // version 1 (sm_100), SWIZZLE_NONE
}
// instruction descriptor: D f32, A / B tf32, both K-major, N = 128, M = 128
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(IDESC), "r"(acc)
        : "memory");
}
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }
}  // namespace dtc

// bsplit: [B_hi | B_lo], each N x (2D) floats already in the canonical K-major layout
// (kdim = 2D), built on the host.  x: rows of 2D floats (complex64 interleaved).
template <int PREC>
__global__ void __launch_bounds__(dtc::THREADS, 1) dense_block_tc_kernel(float *__restrict__ x, const float *__restrict__ bsplit,
                                                                       uint64_t n_tiles) {
    using namespace dtc;
    extern __shared__ __align__(1024) unsigned char smem[];
    constexpr int K = N;  // 2D
    float *sBh = reinterpret_cast<float *>(smem);
    float *sBl = sBh + N * K;
    float *sAh = sBl + N * K;
    float *sAl = sAh + M * KC;
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    {
        const int4 *src = reinterpret_cast<const int4 *>(bsplit);
        int4 *dst = reinterpret_cast<int4 *>(sBh);
        for (int i = tid; i < 2 * N * K / 4; i += THREADS) dst[i] = src[i];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                     "n"(N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = tmem_base;
    uint32_t phase = 0;
    for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        float *xt = x + tile * (uint64_t)M * K;
        for (int kc = 0; kc < K / KC; kc++) {
            // X chunk -> hi / lo in the canonical layout: warp covers 8 rows x 16 floats per
            // step (512 contiguous shared bytes, 64-byte global segments)
            constexpr int PER = M * KC / 4 / THREADS;  // float4 per thread and chunk
            float4 v[PER];
#pragma unroll
            for (int j = 0; j < PER; j++) {  // all loads in flight first
                const int it = tid + j * THREADS, g = it >> 5, l = it & 31;
                const int row = (g / (KC / 16)) * 8 + (l & 7);
                const int k4 = (g % (KC / 16)) * 4 + (l >> 3);  // float4 index within the chunk
                v[j] = __ldcs(reinterpret_cast<const float4 *>(xt + (uint64_t)row * K + kc * KC + k4 * 4));
            }
#pragma unroll
            for (int j = 0; j < PER; j++) {
                const int it = tid + j * THREADS, g = it >> 5, l = it & 31;
                const int row = (g / (KC / 16)) * 8 + (l & 7);
                const int k4 = (g % (KC / 16)) * 4 + (l >> 3);
                const uint32_t off = kmajor_off(row, k4 * 4, KC);
                const float4 h = make_float4(tf32_hi(v[j].x), tf32_hi(v[j].y), tf32_hi(v[j].z), tf32_hi(v[j].w));
                *reinterpret_cast<float4 *>(reinterpret_cast<char *>(sAh) + off) = h;
                if (PREC == 3)
                    *reinterpret_cast<float4 *>(reinterpret_cast<char *>(sAl) + off) =
                        make_float4(v[j].x - h.x, v[j].y - h.y, v[j].z - h.z, v[j].w - h.w);
            }
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic stores -> tensor-core reads
            __syncthreads();
            if (tid == 0) {
                asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                for (int ks = 0; ks < KC / 8; ks++) {
                    const int kg = kc * KC + ks * 8;  // global k of this MMA step
                    const uint64_t ah = smem_desc(smem_u32(sAh) + ks * 256, 128, (KC / 4) * 128);
                    const uint64_t bh = smem_desc(smem_u32(sBh) + (kg / 4) * 128, 128, (K / 4) * 128);
                    const uint32_t acc = (kc | ks) ? 1u : 0u;
                    mma_tf32(tmem, ah, bh, acc);
                    if (PREC == 3) {
                        const uint64_t al = smem_desc(smem_u32(sAl) + ks * 256, 128, (KC / 4) * 128);
                        const uint64_t bl = smem_desc(smem_u32(sBl) + (kg / 4) * 128, 128, (K / 4) * 128);
                        mma_tf32(tmem, ah, bl, 1u);
                        mma_tf32(tmem, al, bh, 1u);
                    }
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];\n" ::"l"(
                                 (uint64_t)smem_u32(&mbar))
                             : "memory");
            }
            // the MMAs have read the chunk (and, after the last chunk, written D)
            asm volatile(
                "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
                    smem_u32(&mbar)),
                "r"(phase)
                : "memory");
            phase ^= 1;
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        }
        // epilogue: warp w owns TMEM lanes / tile rows 32 (w % 4) .. +31 and columns
        // 64 (w / 4) .. +63, 32 columns per load
        const int row = (warp & 3) * 32 + lane;
        float *yr = xt + (uint64_t)row * K;
#pragma unroll
        for (int c0 = (warp >> 2) * 64; c0 < (warp >> 2) * 64 + 64; c0 += 32) {
            uint32_t v[32];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                  "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                  "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                : "r"(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)c0));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
            for (int j = 0; j < 32; j += 4)
                __stcs(reinterpret_cast<float4 *>(yr + c0 + j), make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]),
                                                                        __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3])));
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncthreads();  // TMEM read out and the tile's rows written before the next tile's MMAs
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    }
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(N));
}

// host: the real representation B of U^T, split into TF32 hi / lo, K-major canonical layout
static void build_bsplit(const double *U, int D, float *out) {
    const int K = 2 * D, Nn = 2 * D;
    float *bh = out, *bl = out + Nn * K;
    auto tf32 = [](float v) {
        uint32_t u;
        memcpy(&u, &v, 4);
        u &= 0xffffe000u;
        float r;
        memcpy(&r, &u, 4);
        return r;
    };
    for (int n = 0; n < Nn; n++)      // B^T row n = output real column
        for (int k = 0; k < K; k++) {  // input real index
            const int j = n >> 1, c = k >> 1;
            const double re = U[2 * (j * D + c)], im = U[2 * (j * D + c) + 1];
            double b;
            if ((k & 1) == 0) b = (n & 1) == 0 ? re : im;
            else b = (n & 1) == 0 ? -im : re;
            const float f = (float)b, h = tf32(f);
            const uint32_t off = dtc::kmajor_off(n, k, K) / 4;
            bh[off] = h;
            bl[off] = f - h;
        }
}

// U: D x D complex, row-major (re, im) doubles; *bsplit: device buffer (allocated here)
cudaError_t dense_tc_upload(const double *U, int m, void **bsplit, cudaStream_t s) {
    if (m != 6) return cudaErrorInvalidValue;
    const int D = 1 << m;
    const size_t bbytes = (size_t)2 * (2 * D) * (2 * D) * sizeof(float);
    if (!*bsplit) {
        cudaError_t e = cudaMalloc(bsplit, bbytes);
        if (e != cudaSuccess) return e;
    }
    std::vector<float> hb((size_t)2 * (2 * D) * (2 * D));
    build_bsplit(U, D, hb.data());
    cudaError_t e = cudaMemcpyAsync(*bsplit, hb.data(), bbytes, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
    return cudaStreamSynchronize(s);  // hb is released on return
}

// in place on x (n_amps complex64, the block on the m = 6 lowest bits); prec 1 or 3 (xTF32)
cudaError_t dense_tc_launch(float *x, uint64_t n_amps, const void *bsplit, int prec, int sms, cudaStream_t s) {
    const uint64_t rows = n_amps / 64;
    if (rows % dtc::M) return cudaErrorInvalidValue;
    const uint64_t n_tiles = rows / dtc::M;
    const size_t smem = (size_t)2 * dtc::N * dtc::N * 4 + (size_t)2 * dtc::M * dtc::KC * 4;
    auto fn = prec == 3 ? dense_block_tc_kernel<3> : dense_block_tc_kernel<1>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int grid = (int)std::min<uint64_t>((uint64_t)sms, n_tiles);
    fn<<<grid, dtc::THREADS, smem, s>>>(x, (const float *)bsplit, n_tiles);
    return cudaGetLastError();
}

}  // namespace tqd
