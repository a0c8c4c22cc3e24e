// kernels.cu -- sm_100a kernels of the forward + adjoint path.
//
//   sweep_kernel<Real, R, BWD>   fused gate sweep over 2^k-amplitude tiles
//                                (forward: Alg. 1/2 contraction
//                                Y = M x_Q X for every gate of the stage;
//                                backward: PAPER.md:220-236 recompute x = U^* y
//                                plus the gradient contraction, on psi and lambda)
//   small_kernel<Real, BWD>      whole shard in one CTA's shared memory
//   lambda_init_kernel           lambda = H psi, E = <psi|H|psi> (Z strings)
//   lambda_add_xy_kernel         lambda += c P psi, E += c <psi|P|psi> (X / Y strings)
//   expval_z_kernel / expval_xy_kernel   <psi|P_t|psi> partial sums
//   gather_kernel                canonical-order readback through pi
//   remap_block_kernel           qubit-remap chunk pack / unpack for the NCCL exchange
//
// Data layout in HBM: the shard is an array of interleaved (re, im) complex
// numbers (float2 for complex64, double2 for complex128), physical index =
// local bits of the qubit map pi.  See DESIGN.md "Data layout".
#include <cuda_runtime.h>

#include <algorithm>
#include <stdint.h>

#include "common.cuh"
#include "tqd_internal.h"

namespace tqd {

// ---------------------------------------------------------------------------
// Small-state kernel: the whole 2^n_loc shard in shared memory, one CTA,
// gate-by-gate (ops address PHYSICAL positions: t0/t1 local positions,
// BitRefs are BK_BASE full-index positions).
__device__ __forceinline__ uint64_t ins0(uint64_t i, int p) {  // insert a 0 bit at position p
    return ((i >> p) << (p + 1)) | (i & ((1ull << p) - 1));
}

template <typename Real, bool BWD>
__global__ void __launch_bounds__(512) small_kernel(const DevOp *__restrict__ ops, int n_ops,
                                                    typename CT<Real>::C *__restrict__ psi,
                                                    typename CT<Real>::C *__restrict__ lam,
                                                    double *__restrict__ grad, int n_loc, uint64_t rank_hi) {
    typedef typename CT<Real>::C C;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double red[32];
    const uint64_t N = 1ull << n_loc;
    // batch of states: CTA b runs state b with its own op list (n_ops each)
    ops += (size_t)blockIdx.x * n_ops;
    psi += (size_t)blockIdx.x * N;
    if (BWD) lam += (size_t)blockIdx.x * N;
    C *A = reinterpret_cast<C *>(smem_raw);
    C *L = A + N;
    for (uint64_t i = threadIdx.x; i < N; i += blockDim.x) {
        A[i] = psi[i];
        if (BWD) L[i] = lam[i];
    }
    __syncthreads();
    auto bit = [&](BitRef b, uint64_t idx) -> int { return (int)(((idx | rank_hi) >> b.idx) & 1ull); };

    for (int oi = 0; oi < n_ops; oi++) {
        const DevOp &op = ops[oi];
        const int kind = op.kind;
        if (BWD && op.ngen) {
            for (int gi = 0; gi < op.ngen; gi++) {
                Real part = 0;
                const int gk = op.gkind[gi];
                if (kind == OP_D1) {
                    for (uint64_t i = threadIdx.x; i < N; i += blockDim.x) {
                        Real v = im_cj(L[i], A[i]);
                        part += bit(op.b0, i) ? -v : v;
                    }
                } else {
                    const int p = op.t0;
                    const C g00 = ldc<C>(op.g[gi], 0), g01 = ldc<C>(op.g[gi], 1), g10 = ldc<C>(op.g[gi], 2),
                            g11 = ldc<C>(op.g[gi], 3);
                    for (uint64_t i = threadIdx.x; i < N / 2; i += blockDim.x) {
                        const uint64_t i0 = ins0(i, p), i1 = i0 | (1ull << p);
                        const C a0 = A[i0], a1 = A[i1], l0 = L[i0], l1 = L[i1];
                        if (gk == GEN_Y) part += re_cj(l1, a0) - re_cj(l0, a1);
                        else if (gk == GEN_X) part += im_cj(l0, a1) + im_cj(l1, a0);
                        else part += 2 * (re_cj(l0, cmul2(g00, a0, g01, a1)) + re_cj(l1, cmul2(g10, a0, g11, a1)));
                    }
                }
                double tot = block_sum<double>((double)part, red);
                if (threadIdx.x == 0) atomicAdd(&grad[op.slot[gi]], tot);
                __syncthreads();
            }
        }
        for (int pass = 0; pass < (BWD ? 2 : 1); pass++) {
            C *X = pass ? L : A;
            switch (kind) {
            case OP_U1: case OP_R1: case OP_P1: {
                const int p = op.t0;
                C m00, m01, m10, m11;
                if (kind == OP_U1) { m00 = ldc<C>(op.m, 0); m01 = ldc<C>(op.m, 1); m10 = ldc<C>(op.m, 2); m11 = ldc<C>(op.m, 3); }
                else if (kind == OP_R1) {
                    m00 = mk<C>((Real)op.m[0], 0); m01 = mk<C>((Real)op.m[1], 0);
                    m10 = mk<C>((Real)op.m[2], 0); m11 = mk<C>((Real)op.m[3], 0);
                } else { m00 = mk<C>(0, 0); m01 = ldc<C>(op.m, 0); m10 = ldc<C>(op.m, 1); m11 = mk<C>(0, 0); }
                for (uint64_t i = threadIdx.x; i < N / 2; i += blockDim.x) {
                    const uint64_t i0 = ins0(i, p), i1 = i0 | (1ull << p);
                    if (op.ctrl.kind != BK_NONE && !bit(op.ctrl, i0)) continue;
                    const C x0 = X[i0], x1 = X[i1];
                    X[i0] = cmul2(m00, x0, m01, x1);
                    X[i1] = cmul2(m10, x0, m11, x1);
                }
                break;
            }
            case OP_D1: {
                const C d0 = ldc<C>(op.m, 0), d1 = ldc<C>(op.m, 1);
                for (uint64_t i = threadIdx.x; i < N; i += blockDim.x) X[i] = cmul(bit(op.b0, i) ? d1 : d0, X[i]);
                break;
            }
            case OP_D2: {
                for (uint64_t i = threadIdx.x; i < N; i += blockDim.x)
                    X[i] = cmul(ldc<C>(op.m, 2 * bit(op.b0, i) + bit(op.b1, i)), X[i]);
                break;
            }
            case OP_U2: {
                const int p0 = op.t0, p1 = op.t1;
                const int lo = p0 < p1 ? p0 : p1, hi = p0 < p1 ? p1 : p0;
                for (uint64_t i = threadIdx.x; i < N / 4; i += blockDim.x) {
                    const uint64_t b = ins0(ins0(i, lo), hi);
                    const uint64_t idx[4] = {b, b | (1ull << p1), b | (1ull << p0), b | (1ull << p0) | (1ull << p1)};
                    C v[4];
                    for (int q = 0; q < 4; q++) v[q] = X[idx[q]];
                    for (int r = 0; r < 4; r++) {
                        C acc = mk<C>(0, 0);
                        for (int q = 0; q < 4; q++) {
                            C pr = cmul(ldc<C>(op.m, 4 * r + q), v[q]);
                            acc.x += pr.x; acc.y += pr.y;
                        }
                        X[idx[r]] = acc;
                    }
                }
                break;
            }
            default: break;
            }
        }
        __syncthreads();
    }
    for (uint64_t i = threadIdx.x; i < N; i += blockDim.x) {
        psi[i] = A[i];
        if (BWD) lam[i] = L[i];
    }
}

// ---------------------------------------------------------------------------
// Whole circuit in ONE launch for small states (PAPER.md:291-309 Listing scale;
// BASELINE.json configs[0]): one CTA per state holds psi and lambda in shared
// memory and runs the forward gates, the adjoint seed lambda = H psi for Z strings
// (E = <psi|H|psi>), and the reverse sweep with its gradients,
// gate by gate with one barrier per gate.  Gradient partials: warp shuffle sums,
// one fp64 atomic per warp and generator.  Ops as small_kernel (physical positions).
template <typename Real>
__device__ __forceinline__ void circ_apply(const DevOp &op, typename CT<Real>::C *A, typename CT<Real>::C *L, uint64_t N,
                                           uint64_t rank_hi, bool two) {
    typedef typename CT<Real>::C C;
    auto bit = [&](BitRef b, uint64_t idx) -> int { return (int)(((idx | rank_hi) >> b.idx) & 1ull); };
    const int kind = op.kind;
    switch (kind) {
    case OP_U1: case OP_R1: case OP_P1: {
        const int p = op.t0;
        C m00, m01, m10, m11;
        if (kind == OP_U1) { m00 = ldc<C>(op.m, 0); m01 = ldc<C>(op.m, 1); m10 = ldc<C>(op.m, 2); m11 = ldc<C>(op.m, 3); }
        else if (kind == OP_R1) {
            m00 = mk<C>((Real)op.m[0], 0); m01 = mk<C>((Real)op.m[1], 0);
            m10 = mk<C>((Real)op.m[2], 0); m11 = mk<C>((Real)op.m[3], 0);
        } else { m00 = mk<C>(0, 0); m01 = ldc<C>(op.m, 0); m10 = ldc<C>(op.m, 1); m11 = mk<C>(0, 0); }
        for (uint64_t i = threadIdx.x; i < N / 2; i += blockDim.x) {
            const uint64_t i0 = ins0(i, p), i1 = i0 | (1ull << p);
            if (op.ctrl.kind != BK_NONE && !bit(op.ctrl, i0)) continue;
            const C x0 = A[i0], x1 = A[i1];
            A[i0] = cmul2(m00, x0, m01, x1);
            A[i1] = cmul2(m10, x0, m11, x1);
            if (two) {
                const C y0 = L[i0], y1 = L[i1];
                L[i0] = cmul2(m00, y0, m01, y1);
                L[i1] = cmul2(m10, y0, m11, y1);
            }
        }
        break;
    }
    case OP_D1: {
        const C d0 = ldc<C>(op.m, 0), d1 = ldc<C>(op.m, 1);
        for (uint64_t i = threadIdx.x; i < N; i += blockDim.x) {
            const C d = bit(op.b0, i) ? d1 : d0;
            A[i] = cmul(d, A[i]);
            if (two) L[i] = cmul(d, L[i]);
        }
        break;
    }
    case OP_D2: {
        for (uint64_t i = threadIdx.x; i < N; i += blockDim.x) {
            const C d = ldc<C>(op.m, 2 * bit(op.b0, i) + bit(op.b1, i));
            A[i] = cmul(d, A[i]);
            if (two) L[i] = cmul(d, L[i]);
        }
        break;
    }
    case OP_U2: {
        const int p0 = op.t0, p1 = op.t1;
        const int lo = p0 < p1 ? p0 : p1, hi = p0 < p1 ? p1 : p0;
        for (uint64_t i = threadIdx.x; i < N / 4; i += blockDim.x) {
            const uint64_t b = ins0(ins0(i, lo), hi);
            const uint64_t idx[4] = {b, b | (1ull << p1), b | (1ull << p0), b | (1ull << p0) | (1ull << p1)};
            for (int pass = 0; pass < (two ? 2 : 1); pass++) {
                C *X = pass ? L : A;
                C v[4];
                for (int q = 0; q < 4; q++) v[q] = X[idx[q]];
                for (int r = 0; r < 4; r++) {
                    C acc = mk<C>(0, 0);
                    for (int q = 0; q < 4; q++) {
                        const C pr = cmul(ldc<C>(op.m, 4 * r + q), v[q]);
                        acc.x += pr.x;
                        acc.y += pr.y;
                    }
                    X[idx[r]] = acc;
                }
            }
        }
        break;
    }
    default: break;
    }
}

template <typename Real>
__global__ void __launch_bounds__(512) circuit_kernel(const DevOp *__restrict__ fops, int n_f,
                                                      const DevOp *__restrict__ bops, int n_b,
                                                      const typename CT<Real>::C *__restrict__ psi,
                                                      const ZTerms *__restrict__ zts, double *__restrict__ eval,
                                                      double *__restrict__ grad, int n_loc, uint64_t rank_hi,
                                                      int ops_smem) {
    typedef typename CT<Real>::C C;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double red[32];
    const uint64_t N = 1ull << n_loc;
    fops += (size_t)blockIdx.x * n_f;
    bops += (size_t)blockIdx.x * n_b;
    psi += (size_t)blockIdx.x * N;
    const ZTerms &zt = zts[blockIdx.x];
    C *A = reinterpret_cast<C *>(smem_raw);
    C *L = A + N;
    const int lane = threadIdx.x & 31;
    for (uint64_t i = threadIdx.x; i < N; i += blockDim.x) A[i] = psi[i];
    if (ops_smem) {
        // the op lists into shared memory (a dependent global load per gate field would
        // cost a round trip per gate): after psi and lambda, 16-byte aligned
        DevOp *sf = reinterpret_cast<DevOp *>(L + N);
        DevOp *sb = sf + n_f;
        const int4 *src = reinterpret_cast<const int4 *>(fops);
        int4 *dst = reinterpret_cast<int4 *>(sf);
        for (int i = threadIdx.x; i < n_f * (int)(sizeof(DevOp) / 16); i += blockDim.x) dst[i] = src[i];
        src = reinterpret_cast<const int4 *>(bops);
        dst = reinterpret_cast<int4 *>(sb);
        for (int i = threadIdx.x; i < n_b * (int)(sizeof(DevOp) / 16); i += blockDim.x) dst[i] = src[i];
        fops = sf;
        bops = sb;
    }
    __syncthreads();
    // forward
    for (int oi = 0; oi < n_f; oi++) {
        circ_apply<Real>(fops[oi], A, L, N, rank_hi, false);
        __syncthreads();
    }
    // lambda = H psi, H = cst - 2 sum_p w_p b_p + sum_t c_t (-1)^{popc(b & z_t)}; E = <psi|H|psi>
    double e = 0.0;
    for (uint64_t i = threadIdx.x; i < N; i += blockDim.x) {
        const uint64_t b = i | rank_hi;
        double h = zt.cst;
        for (int p = 0; p < n_loc; p++)
            if ((b >> p) & 1ull) h -= 2.0 * zt.w[p];
        for (int t = 0; t < zt.T; t++) h += (__popcll(b & zt.z[t]) & 1) ? -zt.c[t] : zt.c[t];
        const C a = A[i];
        L[i] = mk<C>((Real)h * a.x, (Real)h * a.y);
        e += h * ((double)a.x * a.x + (double)a.y * a.y);
    }
    e = block_sum<double>(e, red);
    if (threadIdx.x == 0) atomicAdd(eval, e);
    __syncthreads();
    // reverse sweep: gradients on the post-gate states, then psi, lambda <- U^dag
    auto bit = [&](BitRef bb, uint64_t idx) -> int { return (int)(((idx | rank_hi) >> bb.idx) & 1ull); };
    for (int oi = 0; oi < n_b; oi++) {
        const DevOp &op = bops[oi];
        for (int gi = 0; gi < op.ngen; gi++) {
            Real part = 0;
            const int gk = op.gkind[gi];
            if (op.kind == OP_D1) {
                for (uint64_t i = threadIdx.x; i < N; i += blockDim.x) {
                    const Real v = im_cj(L[i], A[i]);
                    part += bit(op.b0, i) ? -v : v;
                }
            } else {
                const int p = op.t0;
                const C g00 = ldc<C>(op.g[gi], 0), g01 = ldc<C>(op.g[gi], 1), g10 = ldc<C>(op.g[gi], 2),
                        g11 = ldc<C>(op.g[gi], 3);
                for (uint64_t i = threadIdx.x; i < N / 2; i += blockDim.x) {
                    const uint64_t i0 = ins0(i, p), i1 = i0 | (1ull << p);
                    const C a0 = A[i0], a1 = A[i1], l0 = L[i0], l1 = L[i1];
                    if (gk == GEN_Y) part += re_cj(l1, a0) - re_cj(l0, a1);
                    else if (gk == GEN_X) part += im_cj(l0, a1) + im_cj(l1, a0);
                    else part += 2 * (re_cj(l0, cmul2(g00, a0, g01, a1)) + re_cj(l1, cmul2(g10, a0, g11, a1)));
                }
            }
            const double w = warp_sum<double>((double)part);
            if (lane == 0 && w != 0.0) atomicAdd(&grad[op.slot[gi]], w);
        }
        // the un-apply reads and writes only the pairs this thread just read
        circ_apply<Real>(op, A, L, N, rank_hi, true);
        __syncthreads();
    }
}

// Register-resident variant for 8 <= n_loc <= 11 (the cfg-1 latency case): thread t
// of N/8 holds the 8 amplitudes idx = r | lane << 3 | warp << 8 (r = 0..7) of psi (and
// lambda) in registers.  A 1-qubit gate on physical bit p is register-local (p < 3),
// a lane shuffle with lane ^ 2^(p-3) (p < 8) or a shared-memory exchange with the
// partner warp (p >= 8; double-buffered, one barrier); diagonal gates are local.  No
// barrier between gates that do not cross warps.  Gradients use the post-gate pair
// values of the same exchange.  Other ops (4x4 MAT2) fall back to
// a shared-memory pass (circ_apply).
// Compact op of the register-resident circuit kernel, decoded once per launch from
// the DevOp (so the gate loop reads one 16-byte header and its coefficients):
// class by where the target bit lives for RB register bits, 2x2 form, control bit,
// the first generator's kind.  Anything else (U2 / MAT2, several or general
// generators) keeps the DevOp path (CC_GEN).
enum : uint8_t { CC_REG = 0, CC_LANE = 1, CC_WARP = 2, CC_D1 = 3, CC_D2 = 4, CC_GEN = 5 };
enum : uint8_t { CF_CPLX = 0, CF_REAL = 1, CF_SWAP = 2 };
struct alignas(16) COp {
    uint8_t cls, p, cb, b0, b1, form, ngen, gk;  // cb = 0xff: no control
    int32_t slot;
    int32_t pad;
    double m[8];  // 2x2 complex row-major (re, im); real form: m[0..3]; D1: d0, d1; D2: 4 entries
};
template <int RB> __device__ __forceinline__ void decode_cop(const DevOp &d, COp &c) {
    c.cls = CC_GEN;
    c.p = d.t0;
    c.cb = d.ctrl.kind == BK_NONE ? 0xff : d.ctrl.idx;
    c.b0 = d.b0.idx;
    c.b1 = d.b1.idx;
    c.ngen = d.ngen;
    c.gk = d.ngen ? d.gkind[0] : GEN_NONE;
    c.slot = d.ngen ? d.slot[0] : 0;
    c.form = CF_CPLX;
    for (int i = 0; i < 8; i++) c.m[i] = d.m[i];
    const bool simple_gen = d.ngen == 0 || (d.ngen == 1 && (d.gkind[0] == GEN_Y || d.gkind[0] == GEN_X || d.gkind[0] == GEN_Z));
    if (!simple_gen) return;
    if (d.kind == OP_U1 || d.kind == OP_R1 || d.kind == OP_P1) {
        if (d.ngen && d.gkind[0] == GEN_Z) return;
        c.cls = d.t0 < RB ? CC_REG : d.t0 < RB + 5 ? CC_LANE : CC_WARP;
        if (d.kind == OP_R1) c.form = CF_REAL;
        if (d.kind == OP_P1) {
            // [[0, a], [b, 0]]: m = (0, a, b, 0); a = b = 1: a swap
            const double a0 = d.m[0], a1 = d.m[1], b0 = d.m[2], b1 = d.m[3];
            c.m[0] = 0; c.m[1] = 0; c.m[2] = a0; c.m[3] = a1; c.m[4] = b0; c.m[5] = b1; c.m[6] = 0; c.m[7] = 0;
            if (a0 == 1.0 && a1 == 0.0 && b0 == 1.0 && b1 == 0.0) c.form = CF_SWAP;  // X / CNOT target
        }
    } else if (d.kind == OP_D1) {
        if (d.ngen && d.gkind[0] != GEN_Z) return;
        c.cls = CC_D1;
    } else if (d.kind == OP_D2 && d.ngen == 0) {
        c.cls = CC_D2;
    }
}

template <typename C> __device__ __forceinline__ C shfl_c(C v, int m) {
    return mk<C>(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
}
template <typename C> __device__ __forceinline__ C cfma2(C a, C x, C b, C y) { return cmul2(a, x, b, y); }

template <typename Real, int RB>
__global__ void __launch_bounds__(512) circuit_reg_kernel(const DevOp *__restrict__ fops, int n_f,
                                                          const DevOp *__restrict__ bops, int n_b,
                                                          const typename CT<Real>::C *__restrict__ psi,
                                                          const ZTerms *__restrict__ zts, double *__restrict__ eval,
                                                          double *__restrict__ grad, int n_loc) {
    typedef typename CT<Real>::C C;
    constexpr int NRR = 1 << RB;  // amplitudes per thread and state
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double red[32];
    const uint64_t N = 1ull << n_loc;
    fops += (size_t)blockIdx.x * n_f;
    bops += (size_t)blockIdx.x * n_b;
    psi += (size_t)blockIdx.x * N;
    const ZTerms &zt = zts[blockIdx.x];
    // shared: 2 exchange buffers of psi + lambda (4 N), then the op lists
    C *X0 = reinterpret_cast<C *>(smem_raw);
    DevOp *sf = reinterpret_cast<DevOp *>(X0 + 4 * N);
    DevOp *sb = sf + n_f;
    COp *cf = reinterpret_cast<COp *>(sb + n_b);
    COp *cbk = cf + n_f;
    {
        const int4 *src = reinterpret_cast<const int4 *>(fops);
        int4 *dst = reinterpret_cast<int4 *>(sf);
        for (int i = threadIdx.x; i < n_f * (int)(sizeof(DevOp) / 16); i += blockDim.x) dst[i] = src[i];
        src = reinterpret_cast<const int4 *>(bops);
        dst = reinterpret_cast<int4 *>(sb);
        for (int i = threadIdx.x; i < n_b * (int)(sizeof(DevOp) / 16); i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n_f + n_b; i += blockDim.x) decode_cop<RB>(i < n_f ? sf[i] : sb[i - n_f], i < n_f ? cf[i] : cbk[i - n_f]);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t tbase = ((uint32_t)lane << RB) | ((uint32_t)warp << (RB + 5));
    C a[NRR], l[NRR];
#pragma unroll
    for (int r = 0; r < NRR; r++) a[r] = psi[tbase | r];
    __syncthreads();
    int xb = 0;  // exchange buffer parity
    auto cbit = [&](BitRef b, uint32_t idx) -> bool { return b.kind == BK_NONE || ((idx >> b.idx) & 1u); };

    // one 1-qubit op (U1 / R1 / P1, optional control) on psi (and lambda when two);
    // gradient partials of its generators first when grads
    auto one_qubit = [&](const DevOp &op, bool two, bool grads) {
        const int p = op.t0;
        C m[4];
        if (op.kind == OP_U1) { m[0] = ldc<C>(op.m, 0); m[1] = ldc<C>(op.m, 1); m[2] = ldc<C>(op.m, 2); m[3] = ldc<C>(op.m, 3); }
        else if (op.kind == OP_R1) {
            m[0] = mk<C>((Real)op.m[0], 0); m[1] = mk<C>((Real)op.m[1], 0);
            m[2] = mk<C>((Real)op.m[2], 0); m[3] = mk<C>((Real)op.m[3], 0);
        } else { m[0] = mk<C>(0, 0); m[1] = ldc<C>(op.m, 0); m[2] = ldc<C>(op.m, 1); m[3] = mk<C>(0, 0); }
        // partner amplitudes: the pair member with bit p flipped
        C ao[NRR], lo[NRR];
        if (p < RB) {  // compile-time register indices (a runtime index would put a[] in local memory)
#define TQD_RX(F)                                                            \
    _Pragma("unroll") for (int r = 0; r < NRR; r++) {                         \
        ao[r] = a[r ^ (F)];                                                   \
        if (two) lo[r] = l[r ^ (F)];                                          \
    }
            if (RB == 1 || p == 0) { TQD_RX(1) } else { TQD_RX(2 % NRR) }
#undef TQD_RX
        } else if (p < RB + 5) {
            const int mk_ = 1 << (p - RB);
#pragma unroll
            for (int r = 0; r < NRR; r++) { ao[r] = shfl_c(a[r], mk_); if (two) lo[r] = shfl_c(l[r], mk_); }
        } else {
            C *XA = X0 + (size_t)xb * 2 * N, *XL = XA + N;
            xb ^= 1;
#pragma unroll
            for (int r = 0; r < NRR; r++) { XA[tbase | r] = a[r]; if (two) XL[tbase | r] = l[r]; }
            __syncthreads();
            const uint32_t f = 1u << p;
#pragma unroll
            for (int r = 0; r < NRR; r++) { ao[r] = XA[(tbase | r) ^ f]; if (two) lo[r] = XL[(tbase | r) ^ f]; }
        }
        if (grads) {
            for (int gi = 0; gi < op.ngen; gi++) {
                const int gk = op.gkind[gi];
                Real part = 0;
#pragma unroll
                for (int r = 0; r < NRR; r++) {
                    const uint32_t idx = tbase | r;
                    if ((idx >> p) & 1u) continue;  // each pair once, from its bit-0 member
                    const C a0 = a[r], a1 = ao[r], l0 = l[r], l1 = lo[r];
                    if (gk == GEN_Y) part += re_cj(l1, a0) - re_cj(l0, a1);
                    else if (gk == GEN_X) part += im_cj(l0, a1) + im_cj(l1, a0);
                    else {
                        const C g00 = ldc<C>(op.g[gi], 0), g01 = ldc<C>(op.g[gi], 1), g10 = ldc<C>(op.g[gi], 2),
                                g11 = ldc<C>(op.g[gi], 3);
                        part += 2 * (re_cj(l0, cmul2(g00, a0, g01, a1)) + re_cj(l1, cmul2(g10, a0, g11, a1)));
                    }
                }
                const double w = warp_sum<double>((double)part);
                if (lane == 0 && w != 0.0) atomicAdd(&grad[op.slot[gi]], w);
            }
        }
        // y_bit = m[bit][bit] x_mine + m[bit][!bit] x_other
        if (p >= RB) {  // bit p is the same for all of this thread's amplitudes
            const bool hi = (tbase >> p) & 1u;
            const C cm = hi ? m[3] : m[0], co = hi ? m[2] : m[1];
#pragma unroll
            for (int r = 0; r < NRR; r++) {
                if (!cbit(op.ctrl, tbase | r)) continue;
                a[r] = cfma2(cm, a[r], co, ao[r]);
                if (two) l[r] = cfma2(cm, l[r], co, lo[r]);
            }
        } else {
#pragma unroll
            for (int r = 0; r < NRR; r++) {
                if (!cbit(op.ctrl, tbase | r)) continue;
                const bool hi = (r >> p) & 1;
                const C cm = hi ? m[3] : m[0], co = hi ? m[2] : m[1];
                a[r] = cfma2(cm, a[r], co, ao[r]);
                if (two) l[r] = cfma2(cm, l[r], co, lo[r]);
            }
        }
    };
    auto diag = [&](const DevOp &op, bool two) {
#pragma unroll
        for (int r = 0; r < NRR; r++) {
            const uint32_t idx = tbase | r;
            const C d = op.kind == OP_D1 ? ldc<C>(op.m, ((idx >> op.b0.idx) & 1u))
                                         : ldc<C>(op.m, 2 * ((idx >> op.b0.idx) & 1u) + ((idx >> op.b1.idx) & 1u));
            a[r] = cmul(d, a[r]);
            if (two) l[r] = cmul(d, l[r]);
        }
    };
    // anything else: through shared memory with the generic small-state code
    auto generic = [&](const DevOp &op, bool two) {
        C *XA = X0 + (size_t)xb * 2 * N, *XL = XA + N;
        xb ^= 1;
#pragma unroll
        for (int r = 0; r < NRR; r++) { XA[tbase | r] = a[r]; if (two) XL[tbase | r] = l[r]; }
        __syncthreads();
        circ_apply<Real>(op, XA, XL, N, 0, two);
        __syncthreads();
#pragma unroll
        for (int r = 0; r < NRR; r++) { a[r] = XA[tbase | r]; if (two) l[r] = XL[tbase | r]; }
    };
    // ---- fast paths on the compact ops --------------------------------------
    // y_bit = m[bit][bit] x + m[bit][!bit] x_partner, per amplitude r (hi = its bit p)
    auto apply_pair = [&](const COp &c, C &x, const C xo, bool hi) {
        if (c.form == CF_SWAP) {
            x = xo;
        } else if (c.form == CF_REAL) {
            const Real cm = (Real)(hi ? c.m[3] : c.m[0]), co = (Real)(hi ? c.m[2] : c.m[1]);
            x = mk<C>(cm * x.x + co * xo.x, cm * x.y + co * xo.y);
        } else {
            const int im_ = hi ? 3 : 0, io = hi ? 2 : 1;
            const C cm = mk<C>((Real)c.m[2 * im_], (Real)c.m[2 * im_ + 1]);
            const C co = mk<C>((Real)c.m[2 * io], (Real)c.m[2 * io + 1]);
            x = cmul2(cm, x, co, xo);
        }
    };
    auto fast_1q = [&](const COp &c, bool two) {
        const int p = c.p;
        C ao[NRR], lo[NRR];
        if (c.cls == CC_REG) {
            if (RB == 1 || p == 0) {
#pragma unroll
                for (int r = 0; r < NRR; r++) { ao[r] = a[r ^ 1]; if (two) lo[r] = l[r ^ 1]; }
            } else {
#pragma unroll
                for (int r = 0; r < NRR; r++) { ao[r] = a[r ^ (2 % NRR)]; if (two) lo[r] = l[r ^ (2 % NRR)]; }
            }
        } else if (c.cls == CC_LANE) {
            const int mk_ = 1 << (p - RB);
#pragma unroll
            for (int r = 0; r < NRR; r++) { ao[r] = shfl_c(a[r], mk_); if (two) lo[r] = shfl_c(l[r], mk_); }
        } else {
            C *XA = X0 + (size_t)xb * 2 * N, *XL = XA + N;
            xb ^= 1;
#pragma unroll
            for (int r = 0; r < NRR; r++) { XA[tbase | r] = a[r]; if (two) XL[tbase | r] = l[r]; }
            __syncthreads();
            const uint32_t f = 1u << p;
#pragma unroll
            for (int r = 0; r < NRR; r++) { ao[r] = XA[(tbase | r) ^ f]; if (two) lo[r] = XL[(tbase | r) ^ f]; }
        }
        if (two && c.ngen) {  // Y or X generator: 2 Re <lam|G|psi> over the pairs, counted by bit-0 members
            Real part = 0;
#pragma unroll
            for (int r = 0; r < NRR; r++) {
                if (((tbase | r) >> p) & 1u) continue;
                part += c.gk == GEN_Y ? re_cj(lo[r], a[r]) - re_cj(l[r], ao[r]) : im_cj(l[r], ao[r]) + im_cj(lo[r], a[r]);
            }
            const double w = warp_sum<double>((double)part);
            if (lane == 0 && w != 0.0) atomicAdd(&grad[c.slot], w);
        }
#pragma unroll
        for (int r = 0; r < NRR; r++) {
            const uint32_t idx = tbase | r;
            if (c.cb != 0xff && !((idx >> c.cb) & 1u)) continue;
            const bool hi = (idx >> p) & 1u;
            apply_pair(c, a[r], ao[r], hi);
            if (two) apply_pair(c, l[r], lo[r], hi);
        }
    };
    auto fast_diag = [&](const COp &c, bool two) {
        if (two && c.ngen) {  // Z generator on bit b0
            Real part = 0;
#pragma unroll
            for (int r = 0; r < NRR; r++) {
                const Real v = im_cj(l[r], a[r]);
                part += (((tbase | r) >> c.b0) & 1u) ? -v : v;
            }
            const double w = warp_sum<double>((double)part);
            if (lane == 0 && w != 0.0) atomicAdd(&grad[c.slot], w);
        }
#pragma unroll
        for (int r = 0; r < NRR; r++) {
            const uint32_t idx = tbase | r;
            const int j = c.cls == CC_D1 ? (int)((idx >> c.b0) & 1u) : (int)(2 * ((idx >> c.b0) & 1u) + ((idx >> c.b1) & 1u));
            const C d = mk<C>((Real)c.m[2 * j], (Real)c.m[2 * j + 1]);
            a[r] = cmul(d, a[r]);
            if (two) l[r] = cmul(d, l[r]);
        }
    };
    for (int oi = 0; oi < n_f; oi++) {
        const COp &c = cf[oi];
        if (c.cls <= CC_WARP) fast_1q(c, false);
        else if (c.cls <= CC_D2) fast_diag(c, false);
        else {
            const DevOp &op = sf[oi];
            if (op.kind == OP_U1 || op.kind == OP_R1 || op.kind == OP_P1) one_qubit(op, false, false);
            else if (op.kind == OP_D1 || op.kind == OP_D2) diag(op, false);
            else generic(op, false);
        }
    }
    // lambda = H psi, E = <psi|H|psi>
    double e = 0.0;
#pragma unroll
    for (int r = 0; r < NRR; r++) {
        const uint32_t b = tbase | r;
        double h = zt.cst;
        for (int p = 0; p < n_loc; p++)
            if ((b >> p) & 1u) h -= 2.0 * zt.w[p];
        for (int t = 0; t < zt.T; t++) h += (__popcll((uint64_t)b & zt.z[t]) & 1) ? -zt.c[t] : zt.c[t];
        l[r] = mk<C>((Real)h * a[r].x, (Real)h * a[r].y);
        e += h * ((double)a[r].x * a[r].x + (double)a[r].y * a[r].y);
    }
    e = block_sum<double>(e, red);
    if (threadIdx.x == 0) atomicAdd(eval, e);
    // reverse sweep
    for (int oi = 0; oi < n_b; oi++) {
        const COp &c = cbk[oi];
        if (c.cls <= CC_WARP) { fast_1q(c, true); continue; }
        if (c.cls <= CC_D2) { fast_diag(c, true); continue; }
        const DevOp &op = sb[oi];
        if (op.kind == OP_U1 || op.kind == OP_R1 || op.kind == OP_P1) {
            one_qubit(op, true, op.ngen > 0);
        } else if (op.kind == OP_D1 || op.kind == OP_D2) {
            for (int gi = 0; gi < op.ngen; gi++) {  // RZ-type generator on a D1 op
                Real part = 0;
#pragma unroll
                for (int r = 0; r < NRR; r++) {
                    const Real v = im_cj(l[r], a[r]);
                    part += (((tbase | r) >> op.b0.idx) & 1u) ? -v : v;
                }
                const double w = warp_sum<double>((double)part);
                if (lane == 0 && w != 0.0) atomicAdd(&grad[op.slot[gi]], w);
            }
            diag(op, true);
        } else {
            generic(op, true);
        }
    }
}

// Two amplitudes per thread (idx = tid << 1 | r, r = 0, 1): the cfg-1 kernel.  Same
// op semantics as circuit_reg_kernel<Real, 1> but the gate loop is straight code on
// scalar registers (no arrays / lambdas that the compiler shuffles through moves),
// the partner / coefficient choice hoisted per thread.
template <typename C>
__device__ __forceinline__ C c_apply(uint8_t form, const double *m, bool hi, C x, C xo) {
    typedef decltype(C::x) Real;
    if (form == CF_SWAP) return xo;
    if (form == CF_REAL) {
        const Real cm = (Real)(hi ? m[3] : m[0]), co = (Real)(hi ? m[2] : m[1]);
        return mk<C>(cm * x.x + co * xo.x, cm * x.y + co * xo.y);
    }
    const int im_ = hi ? 6 : 0, io = hi ? 4 : 2;
    const C cm = mk<C>((Real)m[im_], (Real)m[im_ + 1]), co = mk<C>((Real)m[io], (Real)m[io + 1]);
    return cmul2(cm, x, co, xo);
}

template <typename Real>
__global__ void __launch_bounds__(512) circuit_r1_kernel(const DevOp *__restrict__ fops, int n_f,
                                                         const DevOp *__restrict__ bops, int n_b,
                                                         const typename CT<Real>::C *__restrict__ psi,
                                                         const ZTerms *__restrict__ zts, double *__restrict__ eval,
                                                         double *__restrict__ grad, int n_loc) {
    typedef typename CT<Real>::C C;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double red[32];
    const uint64_t N = 1ull << n_loc;
    fops += (size_t)blockIdx.x * n_f;
    bops += (size_t)blockIdx.x * n_b;
    psi += (size_t)blockIdx.x * N;
    const ZTerms &zt = zts[blockIdx.x];
    C *X0 = reinterpret_cast<C *>(smem_raw);
    DevOp *sf = reinterpret_cast<DevOp *>(X0 + 4 * N);
    DevOp *sb = sf + n_f;
    COp *cf = reinterpret_cast<COp *>(sb + n_b);
    COp *cbk = cf + n_f;
    {
        const int4 *src = reinterpret_cast<const int4 *>(fops);
        int4 *dst = reinterpret_cast<int4 *>(sf);
        for (int i = threadIdx.x; i < n_f * (int)(sizeof(DevOp) / 16); i += blockDim.x) dst[i] = src[i];
        src = reinterpret_cast<const int4 *>(bops);
        dst = reinterpret_cast<int4 *>(sb);
        for (int i = threadIdx.x; i < n_b * (int)(sizeof(DevOp) / 16); i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n_f + n_b; i += blockDim.x) decode_cop<1>(i < n_f ? sf[i] : sb[i - n_f], i < n_f ? cf[i] : cbk[i - n_f]);
    const int lane = threadIdx.x & 31;
    const uint32_t t0 = (uint32_t)threadIdx.x << 1, t1 = t0 | 1u;
    C a0 = psi[t0], a1 = psi[t1], l0 = mk<C>(0, 0), l1 = mk<C>(0, 0);
    __syncthreads();
    int xb = 0;
    auto grad_add = [&](int slot, Real part) {
        const double w = warp_sum<double>((double)part);
        if (lane == 0 && w != 0.0) atomicAdd(&grad[slot], w);
    };
    auto generic = [&](const DevOp &op, bool two) {
        C *XA = X0 + (size_t)xb * 2 * N, *XL = XA + N;
        xb ^= 1;
        XA[t0] = a0; XA[t1] = a1;
        if (two) { XL[t0] = l0; XL[t1] = l1; }
        __syncthreads();
        circ_apply<Real>(op, XA, XL, N, 0, two);
        __syncthreads();
        a0 = XA[t0]; a1 = XA[t1];
        if (two) { l0 = XL[t0]; l1 = XL[t1]; }
    };
    for (int pass = 0; pass < 2; pass++) {
        const bool two = pass == 1;
        const int nops = two ? n_b : n_f;
        const COp *cc = two ? cbk : cf;
        const DevOp *dd = two ? sb : sf;
        if (two) {  // lambda = H psi, E = <psi|H|psi>
            double e = 0.0;
#pragma unroll
            for (int r = 0; r < 2; r++) {
                const uint32_t b = r ? t1 : t0;
                double h = zt.cst;
                for (int p = 0; p < n_loc; p++)
                    if ((b >> p) & 1u) h -= 2.0 * zt.w[p];
                for (int t = 0; t < zt.T; t++) h += (__popcll((uint64_t)b & zt.z[t]) & 1) ? -zt.c[t] : zt.c[t];
                const C a = r ? a1 : a0;
                const C lv = mk<C>((Real)h * a.x, (Real)h * a.y);
                if (r) l1 = lv; else l0 = lv;
                e += h * ((double)a.x * a.x + (double)a.y * a.y);
            }
            e = block_sum<double>(e, red);
            if (threadIdx.x == 0) atomicAdd(eval, e);
        }
        for (int oi = 0; oi < nops; oi++) {
            const COp &c = cc[oi];
            const uint8_t cls = c.cls;
            if (cls == CC_REG || cls == CC_LANE || cls == CC_WARP) {
                const int p = c.p;
                C ao0, ao1, lo0 = mk<C>(0, 0), lo1 = mk<C>(0, 0);
                if (cls == CC_REG) {  // p == 0: the pair is this thread's (a0, a1)
                    ao0 = a1; ao1 = a0;
                    if (two) { lo0 = l1; lo1 = l0; }
                } else if (cls == CC_LANE) {
                    const int mk_ = 1 << (p - 1);
                    ao0 = shfl_c(a0, mk_); ao1 = shfl_c(a1, mk_);
                    if (two) { lo0 = shfl_c(l0, mk_); lo1 = shfl_c(l1, mk_); }
                } else {
                    C *XA = X0 + (size_t)xb * 2 * N, *XL = XA + N;
                    xb ^= 1;
                    XA[t0] = a0; XA[t1] = a1;
                    if (two) { XL[t0] = l0; XL[t1] = l1; }
                    __syncthreads();
                    const uint32_t f = 1u << p;
                    ao0 = XA[t0 ^ f]; ao1 = XA[t1 ^ f];
                    if (two) { lo0 = XL[t0 ^ f]; lo1 = XL[t1 ^ f]; }
                }
                if (two && c.ngen) {  // Y / X generator, each pair from its bit-0 member
                    Real part = 0;
                    const bool h0 = (t0 >> p) & 1u, h1 = (t1 >> p) & 1u;
                    if (c.gk == GEN_Y) {
                        if (!h0) part += re_cj(lo0, a0) - re_cj(l0, ao0);
                        if (!h1) part += re_cj(lo1, a1) - re_cj(l1, ao1);
                    } else {
                        if (!h0) part += im_cj(l0, ao0) + im_cj(lo0, a0);
                        if (!h1) part += im_cj(l1, ao1) + im_cj(lo1, a1);
                    }
                    grad_add(c.slot, part);
                }
                const bool on0 = c.cb == 0xff || ((t0 >> c.cb) & 1u), on1 = c.cb == 0xff || ((t1 >> c.cb) & 1u);
                // coefficients once per op: for a lane / warp target both amplitudes share the
                // target bit (one row of the 2x2); a register target pairs a0 (bit 0) with a1
                if (c.form == CF_SWAP) {
                    if (on0) { a0 = ao0; if (two) l0 = lo0; }
                    if (on1) { a1 = ao1; if (two) l1 = lo1; }
                } else if (c.form == CF_REAL) {
                    if (cls == CC_REG) {
                        const Real m00 = (Real)c.m[0], m01 = (Real)c.m[1], m10 = (Real)c.m[2], m11 = (Real)c.m[3];
                        if (on0) {  // on0 == on1 (the control is not bit 0)
                            const C x0 = a0, x1 = a1;
                            a0 = mk<C>(m00 * x0.x + m01 * x1.x, m00 * x0.y + m01 * x1.y);
                            a1 = mk<C>(m10 * x0.x + m11 * x1.x, m10 * x0.y + m11 * x1.y);
                            if (two) {
                                const C y0 = l0, y1 = l1;
                                l0 = mk<C>(m00 * y0.x + m01 * y1.x, m00 * y0.y + m01 * y1.y);
                                l1 = mk<C>(m10 * y0.x + m11 * y1.x, m10 * y0.y + m11 * y1.y);
                            }
                        }
                    } else {
                        const bool hi = (t0 >> p) & 1u;
                        const Real cm = (Real)(hi ? c.m[3] : c.m[0]), co = (Real)(hi ? c.m[2] : c.m[1]);
                        if (on0) {
                            a0 = mk<C>(cm * a0.x + co * ao0.x, cm * a0.y + co * ao0.y);
                            if (two) l0 = mk<C>(cm * l0.x + co * lo0.x, cm * l0.y + co * lo0.y);
                        }
                        if (on1) {
                            a1 = mk<C>(cm * a1.x + co * ao1.x, cm * a1.y + co * ao1.y);
                            if (two) l1 = mk<C>(cm * l1.x + co * lo1.x, cm * l1.y + co * lo1.y);
                        }
                    }
                } else {
                    const bool hi0 = (t0 >> p) & 1u, hi1 = (t1 >> p) & 1u;
                    if (on0) { a0 = c_apply(c.form, c.m, hi0, a0, ao0); if (two) l0 = c_apply(c.form, c.m, hi0, l0, lo0); }
                    if (on1) { a1 = c_apply(c.form, c.m, hi1, a1, ao1); if (two) l1 = c_apply(c.form, c.m, hi1, l1, lo1); }
                }
            } else if (cls == CC_D1 || cls == CC_D2) {
                const int j0 = cls == CC_D1 ? (int)((t0 >> c.b0) & 1u) : (int)(2 * ((t0 >> c.b0) & 1u) + ((t0 >> c.b1) & 1u));
                const int j1 = cls == CC_D1 ? (int)((t1 >> c.b0) & 1u) : (int)(2 * ((t1 >> c.b0) & 1u) + ((t1 >> c.b1) & 1u));
                if (two && c.ngen) {  // Z generator on bit b0
                    const Real v0 = im_cj(l0, a0), v1 = im_cj(l1, a1);
                    grad_add(c.slot, (((t0 >> c.b0) & 1u) ? -v0 : v0) + (((t1 >> c.b0) & 1u) ? -v1 : v1));
                }
                const C d0 = mk<C>((Real)c.m[2 * j0], (Real)c.m[2 * j0 + 1]);
                const C d1 = mk<C>((Real)c.m[2 * j1], (Real)c.m[2 * j1 + 1]);
                a0 = cmul(d0, a0); a1 = cmul(d1, a1);
                if (two) { l0 = cmul(d0, l0); l1 = cmul(d1, l1); }
            } else {
                // other ops (U2 / MAT2, general generators): shared memory, small-state code
                const DevOp &op = dd[oi];
                if (two && op.ngen) {
                    C *XA = X0 + (size_t)xb * 2 * N, *XL = XA + N;
                    XA[t0] = a0; XA[t1] = a1; XL[t0] = l0; XL[t1] = l1;
                    __syncthreads();
                    for (int gi = 0; gi < op.ngen; gi++) {
                        Real part = 0;
                        if (op.kind == OP_D1) {
                            for (uint64_t i = threadIdx.x; i < N; i += blockDim.x) {
                                const Real v = im_cj(XL[i], XA[i]);
                                part += ((i >> op.b0.idx) & 1ull) ? -v : v;
                            }
                        } else {
                            const int pp = op.t0;
                            const int gk = op.gkind[gi];
                            const C g00 = ldc<C>(op.g[gi], 0), g01 = ldc<C>(op.g[gi], 1), g10 = ldc<C>(op.g[gi], 2),
                                    g11 = ldc<C>(op.g[gi], 3);
                            for (uint64_t i = threadIdx.x; i < N / 2; i += blockDim.x) {
                                const uint64_t i0 = ins0(i, pp), i1 = i0 | (1ull << pp);
                                const C x0 = XA[i0], x1 = XA[i1], y0 = XL[i0], y1 = XL[i1];
                                if (gk == GEN_Y) part += re_cj(y1, x0) - re_cj(y0, x1);
                                else if (gk == GEN_X) part += im_cj(y0, x1) + im_cj(y1, x0);
                                else part += 2 * (re_cj(y0, cmul2(g00, x0, g01, x1)) + re_cj(y1, cmul2(g10, x0, g11, x1)));
                            }
                        }
                        grad_add(op.slot[gi], part);
                    }
                    __syncthreads();
                }
                generic(op, two);
            }
        }
    }
}

// ---- single-launch layout circuit (tqd_internal.h L3Op; abi.cpp encode_l3) -----
// One CTA per state of 8..10 local qubits, 2^(n_loc-3) threads, 8 amplitudes per
// thread in registers (register slots 0..2 = bits 0..2 of r).  Forward op list,
// lambda = H psi (Z-strings, PAPER.md:226-231 seed) and E, then the reverse list
// with gradients 2 Re <lam|G|psi> on the post-gate states before each un-apply
// (PAPER.md:220-236); per-thread gradient accumulators in shared memory, summed
// once at the end.
template <int V> struct L3C { static constexpr int value = V; };
template <typename F> __device__ __forceinline__ void l3_dispatch(int j, F &&f) {
    if (j == 0) f(L3C<0>{});
    else if (j == 1) f(L3C<1>{});
    else f(L3C<2>{});
}

template <int J, typename Real>
__device__ __forceinline__ void l3_u1(typename CT<Real>::C *x, const L3Op &op, const Real *mr) {
    typedef typename CT<Real>::C C;
    const int ck = op.ck, ci = op.ci;
#pragma unroll
    for (int r = 0; r < 8; r++) {
        if (r & (1 << J)) continue;
        const int s = r | (1 << J);
        const bool on = ck != 1 || ((r >> ci) & 1);
        const C x0 = x[r], x1 = x[s];
        C y0, y1;
        if (op.form == L3F_SWAP) {
            y0 = x1;
            y1 = x0;
        } else if (op.form == L3F_REAL) {
            y0 = mk<C>(mr[0] * x0.x + mr[2] * x1.x, mr[0] * x0.y + mr[2] * x1.y);
            y1 = mk<C>(mr[4] * x0.x + mr[6] * x1.x, mr[4] * x0.y + mr[6] * x1.y);
        } else {
            y0 = cmul2(mk<C>(mr[0], mr[1]), x0, mk<C>(mr[2], mr[3]), x1);
            y1 = cmul2(mk<C>(mr[4], mr[5]), x0, mk<C>(mr[6], mr[7]), x1);
        }
        x[r] = on ? y0 : x0;
        x[s] = on ? y1 : x1;
    }
}

template <typename Real>
__global__ void __launch_bounds__(128) circuit_l3_kernel(const L3Op *__restrict__ ops_g, int n_f, int n_b,
                                                         const uint32_t *__restrict__ xtab,
                                                         const uint16_t *__restrict__ xreg_g, int n_rows,
                                                         const uint16_t *__restrict__ accp, int n_acc,
                                                         const double *__restrict__ gtab_g, int n_gt,
                                                         const typename CT<Real>::C *__restrict__ psi,
                                                         const ZTerms *__restrict__ zts, double *__restrict__ eval,
                                                         double *__restrict__ grad, int n_loc) {
    typedef typename CT<Real>::C C;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double red[32];
    const int T = blockDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t N = 1u << n_loc;
    const int nops = n_f + n_b;
    ops_g += (size_t)blockIdx.x * nops;
    accp += (size_t)blockIdx.x * n_acc;
    gtab_g += (size_t)blockIdx.x * n_gt * 8;
    psi += (size_t)blockIdx.x * N;
    const ZTerms &zt = zts[blockIdx.x];
    // shared memory: [2 buffers x (psi, lambda) x N][ops][xreg rows][generators][accumulators n_acc x T]
    C *buf = reinterpret_cast<C *>(smem_raw);
    L3Op *sops = reinterpret_cast<L3Op *>(buf + 4 * N);
    uint16_t *sxr = reinterpret_cast<uint16_t *>(sops + nops);
    double *sg = reinterpret_cast<double *>(sxr + 16 * n_rows);
    Real *tacc = reinterpret_cast<Real *>(sg + 8 * n_gt);
    {
        const int4 *src = reinterpret_cast<const int4 *>(ops_g);
        int4 *dst = reinterpret_cast<int4 *>(sops);
        for (int i = tid; i < nops * (int)(sizeof(L3Op) / 16); i += T) dst[i] = src[i];
        const int4 *xs = reinterpret_cast<const int4 *>(xreg_g);
        int4 *xd = reinterpret_cast<int4 *>(sxr);
        for (int i = tid; i < n_rows * 2; i += T) xd[i] = xs[i];
        for (int i = tid; i < n_gt * 8; i += T) sg[i] = gtab_g[i];
        for (int i = tid; i < n_acc * T; i += T) tacc[i] = 0;
    }
    C a[8], l[8];
    {
        const uint32_t b0 = __ldg(xtab + tid) & 0xffffu;
        const uint16_t *xr = xreg_g;  // row 0 (global: shared memory not ready yet)
#pragma unroll
        for (int r = 0; r < 8; r++) {
            a[r] = psi[b0 | xr[r]];
            l[r] = mk<C>(0, 0);
        }
    }
    uint32_t xrow = n_rows > 2 ? __ldg(xtab + 2 * T + tid) : 0u;  // the next exchange's row (prefetched)
    __syncthreads();
    int xb = 0;
    auto tbit = [&](int i) -> int { return (tid >> i) & 1; };
    auto exch = [&](const L3Op &op, bool two) {
        const uint32_t row = xrow;
        const int e = op.xi;
        if (e + 1 < n_rows) xrow = __ldg(xtab + (size_t)(e + 1) * T + tid);
        C *B = buf + (size_t)xb * 2 * N;
        xb ^= 1;
        const uint16_t *xr = sxr + 16 * e;
        const uint32_t wb = row & 0xffffu, rb = row >> 16;
#pragma unroll
        for (int r = 0; r < 8; r++) {
            const uint32_t o = wb ^ xr[r];
            B[o] = a[r];
            if (two) B[N + o] = l[r];
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 8; r++) {
            const uint32_t o = rb ^ xr[8 + r];
            a[r] = B[o];
            if (two) l[r] = B[N + o];
        }
    };
    auto run = [&](const L3Op &op, bool two) {
        Real mr[8];
        const int type = op.type;
        if (type == L3_X) {
            exch(op, two);
            return;
        }
        if (type == L3_U1) {
#pragma unroll
            for (int i = 0; i < 8; i++) mr[i] = (Real)op.m[i];
            const bool ton = op.ck != 2 || tbit(op.ci);
            l3_dispatch(op.j, [&](auto JJ) {
                constexpr int J = decltype(JJ)::value;
                if (two) {
                    for (int p = 0; p < op.ngen; p++) {
                        Real part = 0;
                        const int gk = op.gk[p];
#pragma unroll
                        for (int r = 0; r < 8; r++) {
                            if (r & (1 << J)) continue;
                            const int s = r | (1 << J);
                            if (gk == GEN_Y) {
                                part += re_cj(l[s], a[r]) - re_cj(l[r], a[s]);
                            } else if (gk == GEN_X) {
                                part += im_cj(l[r], a[s]) + im_cj(l[s], a[r]);
                            } else {
                                const double *g = sg + 8 * (op.gi + p);
                                const C g00 = mk<C>((Real)g[0], (Real)g[1]), g01 = mk<C>((Real)g[2], (Real)g[3]);
                                const C g10 = mk<C>((Real)g[4], (Real)g[5]), g11 = mk<C>((Real)g[6], (Real)g[7]);
                                part += 2 * (re_cj(l[r], cmul2(g00, a[r], g01, a[s])) + re_cj(l[s], cmul2(g10, a[r], g11, a[s])));
                            }
                        }
                        tacc[op.acc[p] * T + tid] += part;
                    }
                }
                if (ton) {
                    l3_u1<J, Real>(a, op, mr);
                    if (two) l3_u1<J, Real>(l, op, mr);
                }
            });
            return;
        }
        if (type == L3_D1) {
            const C d0 = mk<C>((Real)op.m[0], (Real)op.m[1]), d1 = mk<C>((Real)op.m[2], (Real)op.m[3]);
            if (op.d0k == 1) {
                l3_dispatch(op.d0i, [&](auto JJ) {
                    constexpr int J = decltype(JJ)::value;
                    if (two && op.ngen) {  // GEN_Z on this bit
                        Real part = 0;
#pragma unroll
                        for (int r = 0; r < 8; r++) {
                            const Real v = im_cj(l[r], a[r]);
                            part += ((r >> J) & 1) ? -v : v;
                        }
                        tacc[op.acc[0] * T + tid] += part;
                    }
#pragma unroll
                    for (int r = 0; r < 8; r++) {
                        const C d = ((r >> J) & 1) ? d1 : d0;
                        a[r] = cmul(d, a[r]);
                        if (two) l[r] = cmul(d, l[r]);
                    }
                });
            } else {
                const int b = tbit(op.d0i);
                if (two && op.ngen) {
                    Real part = 0;
#pragma unroll
                    for (int r = 0; r < 8; r++) part += im_cj(l[r], a[r]);
                    tacc[op.acc[0] * T + tid] += b ? -part : part;
                }
                const C d = b ? d1 : d0;
#pragma unroll
                for (int r = 0; r < 8; r++) {
                    a[r] = cmul(d, a[r]);
                    if (two) l[r] = cmul(d, l[r]);
                }
            }
            return;
        }
        if (type == L3_D2) {
            C d[4];
#pragma unroll
            for (int i = 0; i < 4; i++) d[i] = mk<C>((Real)op.m[2 * i], (Real)op.m[2 * i + 1]);
            const int t0 = op.d0k == 2 ? tbit(op.d0i) : 0, t1 = op.d1k == 2 ? tbit(op.d1i) : 0;
#pragma unroll
            for (int r = 0; r < 8; r++) {
                const int v0 = op.d0k == 1 ? ((r >> op.d0i) & 1) : t0;
                const int v1 = op.d1k == 1 ? ((r >> op.d1i) & 1) : t1;
                const int v = 2 * v0 + v1;
                const C dv = v == 0 ? d[0] : v == 1 ? d[1] : v == 2 ? d[2] : d[3];
                a[r] = cmul(dv, a[r]);
                if (two) l[r] = cmul(dv, l[r]);
            }
        }
    };
    for (int oi = 0; oi < n_f; oi++) run(sops[oi], false);
    {
        // lambda = H psi, E = <psi|H|psi> at the forward's final layout (row 1)
        const uint32_t b1 = __ldg(xtab + T + tid) & 0xffffu;
        const uint16_t *xr = sxr + 16;
        double e = 0.0;
#pragma unroll
        for (int r = 0; r < 8; r++) {
            const uint32_t b = b1 | xr[r];
            double h = zt.cst;
            for (int p = 0; p < n_loc; p++)
                if ((b >> p) & 1u) h -= 2.0 * zt.w[p];
            for (int t = 0; t < zt.T; t++) h += (__popcll((uint64_t)b & zt.z[t]) & 1) ? -zt.c[t] : zt.c[t];
            l[r] = mk<C>((Real)h * a[r].x, (Real)h * a[r].y);
            e += h * ((double)a[r].x * a[r].x + (double)a[r].y * a[r].y);
        }
        e = block_sum<double>(e, red);
        if (tid == 0) atomicAdd(eval, e);
    }
    for (int oi = n_f; oi < nops; oi++) run(sops[oi], true);
    __syncthreads();
    const int nw = T >> 5;
    for (int k = warp; k < n_acc; k += nw) {
        double v = 0.0;
        for (int t = lane; t < T; t += 32) v += (double)tacc[k * T + t];
        v = warp_sum<double>(v);
        if (lane == 0 && v != 0.0) atomicAdd(&grad[accp[k]], v);
    }
}

size_t circuit_l3_smem(bool dbl, int n_loc, int nops, int n_rows, int n_gt, int n_acc) {
    const size_t esz = dbl ? 16 : 8;
    return (size_t)4 * ((size_t)1 << n_loc) * esz + (size_t)nops * sizeof(L3Op) + (size_t)32 * n_rows +
           (size_t)64 * n_gt + (size_t)n_acc * ((size_t)1 << (n_loc - 3)) * (dbl ? 8 : 4);
}

cudaError_t launch_circuit_l3(bool dbl, const L3Op *ops, int n_f, int n_b, const uint32_t *xtab, const uint16_t *xreg,
                              int n_rows, const uint16_t *accp, int n_acc, const double *gtab, int n_gt, const void *psi,
                              const ZTerms *zts, double *eval, double *grad, int n_loc, int batch, cudaStream_t s) {
    const size_t smem = circuit_l3_smem(dbl, n_loc, n_f + n_b, n_rows, n_gt, n_acc);
    const int threads = 1 << (n_loc - 3);
#define TQD_L3(T)                                                                                               \
    {                                                                                                           \
        cudaError_t e = cudaFuncSetAttribute(circuit_l3_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                             (int)smem);                                                        \
        if (e != cudaSuccess) return e;                                                                         \
        circuit_l3_kernel<T><<<batch, threads, smem, s>>>(ops, n_f, n_b, xtab, xreg, n_rows, accp, n_acc, gtab, \
                                                          n_gt, (const CT<T>::C *)psi, zts, eval, grad, n_loc);  \
        return cudaGetLastError();                                                                              \
    }
    if (dbl) TQD_L3(double)
    TQD_L3(float)
#undef TQD_L3
}

cudaError_t launch_circuit(bool dbl, const DevOp *fops, int n_f, const DevOp *bops, int n_b, const void *psi,
                           const ZTerms *zts, double *eval, double *grad, int n_loc, uint64_t rank_hi, int batch,
                           cudaStream_t s) {
    const size_t ops_bytes = (size_t)(n_f + n_b) * sizeof(DevOp);
    const size_t reg_smem = (size_t)4 * ((size_t)1 << n_loc) * (dbl ? 16 : 8) + ops_bytes + (size_t)(n_f + n_b) * sizeof(COp);
    if (n_loc >= 8 && n_loc <= 11 && reg_smem <= 200 * 1024) {
        // 2 amplitudes per thread (4 at 11 qubits): up to 512 threads for latency hiding
        const int rb = n_loc <= 10 ? 1 : 2;
        const int threads = 1 << (n_loc - rb);
#define TQD_R(T)                                                                                               \
    {                                                                                                          \
        auto fn = rb == 1 ? circuit_r1_kernel<T> : circuit_reg_kernel<T, 2>;                                   \
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)reg_smem); \
        if (e != cudaSuccess) return e;                                                                        \
        fn<<<batch, threads, reg_smem, s>>>(fops, n_f, bops, n_b, (const CT<T>::C *)psi, zts, eval, grad, n_loc); \
        return cudaGetLastError();                                                                             \
    }
        if (dbl) TQD_R(double)
        TQD_R(float)
#undef TQD_R
    }
    size_t smem = (size_t)2 * ((size_t)1 << n_loc) * (dbl ? 16 : 8);
    const int ops_smem = smem + ops_bytes <= 200 * 1024;
    if (ops_smem) smem += ops_bytes;
    const int threads = 512;
#define TQD_C(T)                                                                                               \
    {                                                                                                          \
        auto fn = circuit_kernel<T>;                                                                           \
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
        if (e != cudaSuccess) return e;                                                                        \
        fn<<<batch, threads, smem, s>>>(fops, n_f, bops, n_b, (const CT<T>::C *)psi, zts, eval, grad, n_loc, rank_hi, ops_smem); \
        return cudaGetLastError();                                                                             \
    }
    if (dbl) TQD_C(double)
    TQD_C(float)
#undef TQD_C
}

static int grid_for(uint64_t n, int threads);
// ---------------------------------------------------------------------------
// Product-state prefix (exact rewrite; abi.cpp prefix_build): every qubit's leading
// 1-qubit gates act on |0> before the qubit meets a multi-qubit gate, so after them
// the state is the product psi_P(b) = prod_q s_q(b_q).  With the local physical bits
// cut into groups of PF_BITS (low first), psi_P(b) = prod_g tab_g[b's bits of group g]
// (tables built on the host in fp64).  prefix_init writes psi_P (replaces |0..0>
// and the prefix gates' sweeps); prefix_contract computes, for the adjoint state at
// the prefix boundary, M_g[i] = sum_{b: group g of b = i} conj(lam(b)) prod_{h != g}
// tab_h[b's bits of group h] -- the environments from which the host finishes the
// prefix gates' gradients 2 Re <lam|d psi_P / d theta>.
constexpr int PF_BITS = 10;
constexpr int PF_MAXG = 4;
template <typename Real>
__global__ void __launch_bounds__(256) prefix_init_kernel(typename CT<Real>::C *__restrict__ psi, uint64_t n, int ng,
                                                          const typename CT<Real>::C *__restrict__ tab, Real cre,
                                                          Real cim) {
    typedef typename CT<Real>::C C;
    const C cr = mk<C>(cre, cim);  // this rank's factor of the global (sharded) qubits
    for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < n; b += (uint64_t)gridDim.x * blockDim.x) {
        C v = cmul(cr, tab[b & ((1u << PF_BITS) - 1)]);
        for (int g = 1; g < ng; g++) v = cmul(v, tab[(g << PF_BITS) + ((b >> (PF_BITS * g)) & ((1u << PF_BITS) - 1))]);
        psi[b] = v;
    }
}

// one CTA (256 threads) per contiguous range of 1024-amplitude chunks (group 0 = the
// chunk offset, groups >= 1 uniform per chunk); M_0 in per-thread fp64 registers, the
// chunk sums S_c = sum conj(lam) tab_0 -> M_g[g-index] += S_c * prod_{h >= 1, h != g}
// tab_h in shared memory; global fp64 atomics at the end
template <typename Real>
__global__ void __launch_bounds__(256) prefix_contract_kernel(const typename CT<Real>::C *__restrict__ lam, uint64_t n,
                                                              int ng, const typename CT<Real>::C *__restrict__ tab,
                                                              double *__restrict__ M) {
    typedef typename CT<Real>::C C;
    constexpr int CH = 1 << PF_BITS, PER = CH / 256;
    extern __shared__ __align__(16) double sm[];  // (ng - 1) x CH complex fp64
    __shared__ double red[2][32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < (ng - 1) * CH * 2; i += 256) sm[i] = 0.0;
    double m0r[PER], m0i[PER];
    C t0[PER];
#pragma unroll
    for (int j = 0; j < PER; j++) {
        m0r[j] = m0i[j] = 0.0;
        t0[j] = tab[tid + 256 * j];
    }
    __syncthreads();
    const uint64_t nch = n >> PF_BITS;
    const uint64_t per = (nch + gridDim.x - 1) / gridDim.x;
    const uint64_t c0 = (uint64_t)blockIdx.x * per, c1 = c0 + per < nch ? c0 + per : nch;
    for (uint64_t c = c0; c < c1; c++) {
        // the chunk's factors of groups >= 1 (uniform): all of them and all-but-one
        C f[PF_MAXG];
        C P = mk<C>(1, 0);
        for (int g = 1; g < ng; g++) {
            f[g] = tab[(g << PF_BITS) + ((c >> (PF_BITS * (g - 1))) & (CH - 1))];
            P = cmul(P, f[g]);
        }
        double sr = 0.0, si = 0.0;
#pragma unroll
        for (int j = 0; j < PER; j++) {
            const C l = lam[(c << PF_BITS) + tid + 256 * j];
            const C x = mk<C>(l.x, -l.y);  // conj(lambda)
            const C y = cmul(x, P);
            m0r[j] += (double)y.x;
            m0i[j] += (double)y.y;
            const C z = cmul(x, t0[j]);
            sr += (double)z.x;
            si += (double)z.y;
        }
        sr = warp_sum(sr);
        si = warp_sum(si);
        if (lane == 0) { red[0][warp] = sr; red[1][warp] = si; }
        __syncthreads();
        if (tid < ng - 1) {  // thread g-1 adds S_c * prod_{h >= 1, h != g} f_h into M_g
            double Sr = 0.0, Si = 0.0;
            for (int w = 0; w < 8; w++) { Sr += red[0][w]; Si += red[1][w]; }
            const int g = tid + 1;
            double er = 1.0, ei = 0.0;
            for (int h = 1; h < ng; h++) {
                if (h == g) continue;
                const double nr = er * (double)f[h].x - ei * (double)f[h].y, ni = er * (double)f[h].y + ei * (double)f[h].x;
                er = nr; ei = ni;
            }
            const int idx = (int)((c >> (PF_BITS * (g - 1))) & (CH - 1));
            sm[((g - 1) * CH + idx) * 2] += Sr * er - Si * ei;
            sm[((g - 1) * CH + idx) * 2 + 1] += Sr * ei + Si * er;
        }
        __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < PER; j++) {
        if (m0r[j] != 0.0) atomicAdd(&M[(tid + 256 * j) * 2], m0r[j]);
        if (m0i[j] != 0.0) atomicAdd(&M[(tid + 256 * j) * 2 + 1], m0i[j]);
    }
    for (int i = tid; i < (ng - 1) * CH * 2; i += 256)
        if (sm[i] != 0.0) atomicAdd(&M[CH * 2 + i], sm[i]);
}

cudaError_t launch_prefix_init(bool dbl, void *psi, uint64_t n, int ng, const void *tab, double cre, double cim,
                               cudaStream_t s) {
    const int th = 256;
    if (dbl) prefix_init_kernel<double><<<grid_for(n, th), th, 0, s>>>((double2 *)psi, n, ng, (const double2 *)tab, cre, cim);
    else prefix_init_kernel<float><<<grid_for(n, th), th, 0, s>>>((float2 *)psi, n, ng, (const float2 *)tab, (float)cre, (float)cim);
    return cudaGetLastError();
}
cudaError_t launch_prefix_contract(bool dbl, const void *lam, uint64_t n, int ng, const void *tab, double *M, int sms,
                                   cudaStream_t s) {
    const uint64_t nch = n >> PF_BITS;
    const int grid = (int)std::min<uint64_t>(nch, (uint64_t)sms * 4);
    const size_t smem = (size_t)(ng - 1) * (1u << PF_BITS) * 2 * sizeof(double);
    cudaError_t e = dbl ? cudaFuncSetAttribute(prefix_contract_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                        : cudaFuncSetAttribute(prefix_contract_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (dbl) prefix_contract_kernel<double><<<grid, 256, smem, s>>>((const double2 *)lam, n, ng, (const double2 *)tab, M);
    else prefix_contract_kernel<float><<<grid, 256, smem, s>>>((const float2 *)lam, n, ng, (const float2 *)tab, M);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Z-string observables in physical masks.

// lambda = H psi with H = sum_t c_t Z_t (diagonal): h(b) = sum_t c_t (-1)^{popc(b & z_t)};
// E partial = sum_b h(b) |psi_b|^2   (the seed dy of the reverse pass)
//
// Single-bit terms: h = cst - 2 sum_p w_p b_p (byte tables over b).  Multi-bit
// terms (e.g. the strings of an absorbed CNOT ladder): the parity of b & z_t is
// the XOR of three parity MASKS over the terms (bit t = parity of z_t with part
// of b): the thread's low 8 index bits (per kernel), the amplitude's slot u in
// a 4096-amplitude chunk (per kernel, smem) and the chunk base incl. rank bits
// (per chunk), so each amplitude costs one XOR and ceil(T/8) byte-table lookups
// of sum_{t in S} c_t, independent of the strings' lengths.
constexpr int LI_U = 16;  // amplitudes per thread per 4096-amplitude chunk
template <typename Real>
__global__ void __launch_bounds__(256) lambda_init_kernel(const typename CT<Real>::C *__restrict__ psi,
                                                          typename CT<Real>::C *__restrict__ lam, uint64_t n,
                                                          uint64_t rank_hi, const __grid_constant__ ZTerms terms,
                                                          double *__restrict__ eout) {
    typedef typename CT<Real>::C C;
    __shared__ double red[32];
    // byte tables: tab[j][v] = sum_{i<8} w[8j + i] bit_i(v);  tabt[j][v] = sum_{i<8} c[8j + i] bit_i(v)
    __shared__ Real tab[8][256], tabt[8][256];
    __shared__ uint64_t zs[64], pu[LI_U];
    __shared__ Real linu[LI_U];
    const int T = terms.T;
    int nb = 0;
    for (int p = 0; p < 64; p++)
        if (terms.w[p] != 0.0) nb = p / 8 + 1;
    const int ntb = (T + 7) / 8;
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) {
        const int j = i >> 8, v = i & 255;
        double s = 0, st = 0;
        for (int q = 0; q < 8; q++)
            if ((v >> q) & 1) {
                s += terms.w[8 * j + q];
                if (8 * j + q < T) st += terms.c[8 * j + q];
            }
        tab[j][v] = (Real)s;
        tabt[j][v] = (Real)st;
    }
    if (threadIdx.x < 64) zs[threadIdx.x] = threadIdx.x < T ? terms.z[threadIdx.x] : 0ull;
    double ctot = terms.cst;
    for (int t = 0; t < T; t++) ctot += terms.c[t];
    __syncthreads();
    auto pmask = [&](uint64_t b) {  // bit t = parity(b & z_t)
        uint64_t m = 0;
        for (int t = 0; t < T; t++) m |= (uint64_t)(__popcll(b & zs[t]) & 1) << t;
        return m;
    };
    auto lin = [&](uint64_t b) {
        Real s = 0;
        for (int j = 0; j < nb; j++) s += tab[j][(b >> (8 * j)) & 255];
        return s;
    };
    if (threadIdx.x < LI_U) {
        pu[threadIdx.x] = pmask((uint64_t)threadIdx.x << 8);
        linu[threadIdx.x] = lin((uint64_t)threadIdx.x << 8);
    }
    const uint64_t pj = pmask((uint64_t)threadIdx.x);
    const Real linj = lin((uint64_t)threadIdx.x);
    __syncthreads();
    const Real K = (Real)ctot;
    double acc = 0;
    const uint64_t chunks = (n + 4095) >> 12;
    for (uint64_t ch = blockIdx.x; ch < chunks; ch += gridDim.x) {
        const uint64_t base = ch << 12;
        const uint64_t pb = T ? pmask(base | rank_hi) : 0;
        const Real linb = lin(base | rank_hi);
        // all 16 loads first (memory-level parallelism), then h and the stores
        C xs[LI_U];
#pragma unroll
        for (int u = 0; u < LI_U; u++) {
            const uint64_t i = base + ((uint64_t)u << 8) + threadIdx.x;
            xs[u] = i < n ? psi[i] : mk<C>(0, 0);
        }
        Real cacc = 0;
#pragma unroll
        for (int u = 0; u < LI_U; u++) {
            const uint64_t i = base + ((uint64_t)u << 8) + threadIdx.x;
            const uint64_t S = pj ^ pu[u] ^ pb;
            Real sv = linj + linu[u] + linb;
            for (int j = 0; j < ntb; j++) sv += tabt[j][(S >> (8 * j)) & 255];
            const Real h = K - 2 * sv;
            const C x = xs[u];
            if (i < n) lam[i] = mk<C>(h * x.x, h * x.y);
            cacc += h * (x.x * x.x + x.y * x.y);
        }
        acc += (double)cacc;
    }
    double tot = block_sum<double>(acc, red);
    if (threadIdx.x == 0) atomicAdd(eout, tot);
}

// X / Y strings in the adjoint seed (PAPER.md:226-231 with H = sum_t c_t P_t):
// lambda_j += sum_t c_t (P_t psi)_j for terms sharing one x mask, where
// (P psi)_j = i^{q} (-1)^{popc((b_j ^ x) & z)} psi_{j ^ x}   (q = #Y mod 4; the same
// convention as expval_xy_kernel), psi_{j ^ x} read from `peer` (this shard, or
// the partner rank's when x has rank bits).  E partial += Re(conj(psi_j) * that).
template <typename Real>
__global__ void __launch_bounds__(256) lambda_add_xy_kernel(const typename CT<Real>::C *__restrict__ psi,
                                                            const typename CT<Real>::C *__restrict__ peer,
                                                            typename CT<Real>::C *__restrict__ lam, uint64_t n,
                                                            uint64_t rank_hi, uint64_t xloc, uint64_t xfull,
                                                            const uint64_t *__restrict__ zmask, const int *__restrict__ ny,
                                                            const double *__restrict__ coef, int T,
                                                            double *__restrict__ eout) {
    typedef typename CT<Real>::C C;
    __shared__ double red[32];
    double acc = 0;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t bsrc = (j | rank_hi) ^ xfull;
        const C y = peer[j ^ xloc];
        Real ar = 0, ai = 0;  // sum_t c_t s_t, complex (s_t = i^q (-1)^parity)
        for (int t = 0; t < T; t++) {
            Real c = (Real)coef[t];
            if (__popcll(bsrc & zmask[t]) & 1) c = -c;
            switch (ny[t] & 3) {
            case 0: ar += c; break;
            case 1: ai += c; break;
            case 2: ar -= c; break;
            default: ai -= c; break;
            }
        }
        const C v = mk<C>(ar * y.x - ai * y.y, ar * y.y + ai * y.x);
        const C l = lam[j];
        lam[j] = mk<C>(l.x + v.x, l.y + v.y);
        const C x = psi[j];
        acc += (double)(x.x * v.x + x.y * v.y);
    }
    double tot = block_sum<double>(acc, red);
    if (threadIdx.x == 0) atomicAdd(eout, tot);
}

// ---------------------------------------------------------------------------
// Shot noise, approximate (Gaussian) sampler.  Counter-based
// normals indexed by the CANONICAL outcome (so results do not depend on the qubit
// map pi or the sharding): splitmix64 + Box-Muller, fp64 (R21, R22).
__device__ __forceinline__ uint64_t splitmix64_d(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
__device__ __forceinline__ double uniform_d(uint64_t seed, uint64_t k) {
    return (double)(splitmix64_d(seed ^ (k * 0xD1B54A32D192ED03ull)) >> 11) * 0x1.0p-53;
}
__device__ __forceinline__ double normal_d(uint64_t seed, uint64_t i) {
    const double u1 = uniform_d(seed, 2 * i), u2 = uniform_d(seed, 2 * i + 1);
    return sqrt(-2.0 * log(1.0 - u1)) * cospi(2.0 * u2);
}
__device__ __forceinline__ uint64_t canon_of(uint64_t P, const GatherMap &gm) {
    uint64_t c = 0;
    for (int b = 0; b < gm.n; b++) c |= ((P >> gm.phys_of_canon_bit[b]) & 1ull) << b;
    return c;
}

// Global sums of the sample's per-qubit estimates for up to 16 qubits (physical
// positions qpos): out[q] += sum p s_q, out[16 + q] += sum u z s_q, out[32] += sum u z,
// out[33..34] = psi at the last canonical outcome K (written by its owner only).
struct GaussQ {
    int nq;
    uint8_t qpos[16];
};
template <typename Real>
__global__ void __launch_bounds__(256) gauss_sums_kernel(const typename CT<Real>::C *__restrict__ psi, uint64_t n,
                                                         uint64_t rank_hi, GatherMap gm, uint64_t seed, GaussQ gq,
                                                         double *__restrict__ out) {
    typedef typename CT<Real>::C C;
    __shared__ double red[32];
    double m[16], A[16], B = 0;
#pragma unroll
    for (int q = 0; q < 16; q++) m[q] = A[q] = 0;
    const uint64_t K = (gm.n >= 64) ? ~0ull : ((1ull << gm.n) - 1);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t P = i | rank_hi;
        const C x = psi[i];
        const double p = (double)x.x * x.x + (double)x.y * x.y;
        const uint64_t c = canon_of(P, gm);
        const double uz = c == K ? 0.0 : sqrt(p) * normal_d(seed, c);
        if (c == K) { out[33] = (double)x.x; out[34] = (double)x.y; }
        B += uz;
#pragma unroll
        for (int q = 0; q < 16; q++) {
            if (q < gq.nq) {
                const bool neg = (P >> gq.qpos[q]) & 1ull;
                m[q] += neg ? -p : p;
                A[q] += neg ? -uz : uz;
            }
        }
    }
    for (int q = 0; q < gq.nq; q++) {
        double t = block_sum<double>(m[q], red);
        if (threadIdx.x == 0) atomicAdd(&out[q], t);
        t = block_sum<double>(A[q], red);
        if (threadIdx.x == 0) atomicAdd(&out[16 + q], t);
    }
    const double tb = block_sum<double>(B, red);
    if (threadIdx.x == 0) atomicAdd(&out[32], tb);
}

// Adjoint seed of L = sum_q c_q Zhat_q (the derivative of the closed form in DESIGN.md
// §8c w.r.t. psi*):  lambda_j = alpha S(j) psi_j + k2 z_j (S(j) + Fc) e_j + [j = K] kc e_K,
// S(j) = sum_q c_q s_q(j) = cst - 2 sum_p w_p bit_p(j), e_j = psi_j / |psi_j|.
template <typename Real>
__global__ void __launch_bounds__(256) lambda_gauss_kernel(const typename CT<Real>::C *__restrict__ psi,
                                                           typename CT<Real>::C *__restrict__ lam, uint64_t n,
                                                           uint64_t rank_hi, GatherMap gm, uint64_t seed, ZTerms terms,
                                                           double alpha, double fc, double k2, double kc) {
    typedef typename CT<Real>::C C;
    const uint64_t K = (gm.n >= 64) ? ~0ull : ((1ull << gm.n) - 1);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t P = i | rank_hi;
        double s = terms.cst;
        for (int b = 0; b < 64; b++)
            if (terms.w[b] != 0.0 && ((P >> b) & 1ull)) s -= 2.0 * terms.w[b];
        const C x = psi[i];
        const double xr = x.x, xi = x.y, u = sqrt(xr * xr + xi * xi);
        const uint64_t c = canon_of(P, gm);
        double lr = alpha * s * xr, li = alpha * s * xi;
        if (u > 0) {
            double f = 0.0;
            if (c != K) f += k2 * normal_d(seed, c) * (s + fc);
            else f += kc;
            lr += f * xr / u;
            li += f * xi / u;
        }
        lam[i] = mk<C>((Real)lr, (Real)li);
    }
}

// ---------------------------------------------------------------------------
// Shot noise, exact: per-chunk probability masses, then every
// chunk that received shots resolves them by a block prefix sum over its
// probabilities and a search per shot (inverse CDF in the shard's physical order).
constexpr int SAMPLE_CHUNK = 4096;

template <typename Real>
__global__ void __launch_bounds__(256) chunk_mass_kernel(const typename CT<Real>::C *__restrict__ psi, uint64_t n_chunks,
                                                         int csz, double *__restrict__ out) {
    typedef typename CT<Real>::C C;
    __shared__ double red[32];
    for (uint64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
        double s = 0;
        for (int i = threadIdx.x; i < csz; i += blockDim.x) {
            const C x = psi[c * csz + i];
            s += (double)x.x * x.x + (double)x.y * x.y;
        }
        s = block_sum<double>(s, red);
        if (threadIdx.x == 0) out[c] = s;
        __syncthreads();
    }
}

// one CTA per chunk with shots: shots [off[j], off[j+1]) with residual uniforms
// r (mass units inside the chunk, sorted); writes the canonical outcome of each
template <typename Real>
__global__ void __launch_bounds__(256) chunk_sample_kernel(const typename CT<Real>::C *__restrict__ psi,
                                                           const uint64_t *__restrict__ chunk_id,
                                                           const uint32_t *__restrict__ off, const double *__restrict__ r,
                                                           const uint64_t *__restrict__ shot_idx, uint64_t rank_hi,
                                                           GatherMap gm, int csz, double *__restrict__ out) {
    typedef typename CT<Real>::C C;
    __shared__ double cdf[SAMPLE_CHUNK];  // csz <= SAMPLE_CHUNK
    __shared__ double wsum[32];
    const uint64_t c = chunk_id[blockIdx.x];
    // inclusive prefix of the chunk's probabilities (16 per thread, warp / block scan)
    const int per = max(1, csz / (int)blockDim.x);  // <= 16 (blockDim = max(32, min(256, csz)))
    double loc[16];
    double acc = 0;
    for (int j = 0; j < per; j++) {
        const int e = threadIdx.x * per + j;
        if (e < csz) {
            const C x = psi[c * csz + e];
            acc += (double)x.x * x.x + (double)x.y * x.y;
        }
        loc[j] = acc;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double incl = acc;
    for (int o = 1; o < 32; o <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        double v = lane < nw ? wsum[lane] : 0.0;
        for (int o = 1; o < 32; o <<= 1) {
            const double t = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += t;
        }
        if (lane < nw) wsum[lane] = v;
    }
    __syncthreads();
    const double before = (incl - acc) + (warp ? wsum[warp - 1] : 0.0);
    for (int j = 0; j < per; j++)
        if (threadIdx.x * per + j < csz) cdf[threadIdx.x * per + j] = before + loc[j];
    __syncthreads();
    for (uint32_t s = off[blockIdx.x] + threadIdx.x; s < off[blockIdx.x + 1]; s += blockDim.x) {
        const double u = r[s];
        int lo = 0, hi = csz - 1;  // first index with cdf > u (clamped to the chunk)
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (cdf[mid] > u) hi = mid;
            else lo = mid + 1;
        }
        while (lo > 0 && cdf[lo] == cdf[lo - 1]) lo--;  // rounding at the chunk end: never a p = 0 outcome
        const uint64_t P = (c * csz + lo) | rank_hi;
        out[shot_idx[s]] = (double)canon_of(P, gm);
    }
}

// out[t] += sum_b |psi_b|^2 (-1)^{popc(b & z_t)}, up to 16 terms per launch.
// A CTA iteration covers one 4096-amplitude chunk: thread j holds amplitudes
// base + 256 u + j (u = 0..15, coalesced per u).  The sign factorises over the
// three disjoint index parts, (-1)^{popc(j & z)} (per thread) x (-1)^{popc(base & z)}
// (per chunk) x (-1)^{popc(u & z>>8)}, so the u sums of all terms are one 16-point
// Walsh-Hadamard transform of the thread's |psi|^2 values: ~10 instructions per
// amplitude for 16 terms instead of a popcount per term (these Z strings can be
// long, e.g. after absorbing a CNOT ladder).
template <typename Real>
__global__ void __launch_bounds__(256) expval_z_kernel(const typename CT<Real>::C *__restrict__ psi, uint64_t n,
                                                       uint64_t rank_hi, const uint64_t *__restrict__ zmask, int T,
                                                       double *__restrict__ out) {
    typedef typename CT<Real>::C C;
    __shared__ double red[32];
    __shared__ Real wsh[16][256];
    uint64_t z[16];
#pragma unroll
    for (int t = 0; t < 16; t++) z[t] = t < T ? zmask[t] : 0;
    uint32_t pj = 0;  // bit t: parity of (thread bits & z_t)
#pragma unroll
    for (int t = 0; t < 16; t++) pj |= (uint32_t)(__popcll((uint64_t)threadIdx.x & z[t]) & 1) << t;
    double dacc[16];
#pragma unroll
    for (int t = 0; t < 16; t++) dacc[t] = 0;
    const uint64_t chunks = (n + 4095) >> 12;
    for (uint64_t ch = blockIdx.x; ch < chunks; ch += gridDim.x) {
        const uint64_t base = ch << 12;
        Real w[16];
#pragma unroll
        for (int u = 0; u < 16; u++) {
            const uint64_t i = base + ((uint64_t)u << 8) + threadIdx.x;
            Real p = 0;
            if (i < n) {
                const C x = psi[i];
                p = x.x * x.x + x.y * x.y;
            }
            w[u] = p;
        }
#pragma unroll
        for (int b = 0; b < 4; b++)
#pragma unroll
            for (int u = 0; u < 16; u++)
                if (!(u & (1 << b))) {
                    const Real a0 = w[u], a1 = w[u | (1 << b)];
                    w[u] = a0 + a1;
                    w[u | (1 << b)] = a0 - a1;
                }
#pragma unroll
        for (int u = 0; u < 16; u++) wsh[u][threadIdx.x] = w[u];
        uint32_t pb = 0;  // bit t: parity of (chunk base incl. rank bits & z_t)
#pragma unroll
        for (int t = 0; t < 16; t++) pb |= (uint32_t)(__popcll((base | rank_hi) & z[t]) & 1) << t;
        const uint32_t sg = pj ^ pb;
#pragma unroll
        for (int t = 0; t < 16; t++) {
            if (t >= T) break;
            const Real v = wsh[(z[t] >> 8) & 15][threadIdx.x];
            dacc[t] += (double)(((sg >> t) & 1u) ? -v : v);
        }
    }
    for (int t = 0; t < T; t++) {
        double tot = block_sum<double>(dacc[t], red);
        if (threadIdx.x == 0) atomicAdd(&out[t], tot);
    }
}

// out[t] += sum_b Re( i^{ny_t} (-1)^{popc(b & z_t)} conj(psi_{b^x}) psi_b ): one x mask, <= 16 terms
template <typename Real>
__global__ void __launch_bounds__(256) expval_xy_kernel(const typename CT<Real>::C *__restrict__ psi,
                                                        const typename CT<Real>::C *__restrict__ peer, uint64_t n,
                                                        uint64_t rank_hi, uint64_t xloc, const uint64_t *__restrict__ zmask,
                                                        const int *__restrict__ ny, int T, double *__restrict__ out) {
    typedef typename CT<Real>::C C;
    __shared__ double red[32];
    double acc[16];
#pragma unroll
    for (int t = 0; t < 16; t++) acc[t] = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t b = i | rank_hi;
        const C x = psi[i], y = peer[i ^ xloc];  // peer: this shard, or the partner rank's (X on rank bits)
        const Real re = y.x * x.x + y.y * x.y;  // conj(y) x
        const Real im = y.x * x.y - y.y * x.x;
#pragma unroll
        for (int t = 0; t < 16; t++) {
            if (t < T) {
                const int q = ny[t] & 3;  // i^q
                Real v = q == 0 ? re : q == 1 ? -im : q == 2 ? -re : im;
                acc[t] += (double)((__popcll(b & zmask[t]) & 1) ? -v : v);
            }
        }
    }
    for (int t = 0; t < T; t++) {
        double tot = block_sum<double>(acc[t], red);
        if (threadIdx.x == 0) atomicAdd(&out[t], tot);
    }
}

// canonical index -> physical index through pi; amplitudes owned by other ranks -> 0
template <typename Real>
__global__ void gather_kernel(const typename CT<Real>::C *__restrict__ psi, typename CT<Real>::C *__restrict__ out,
                              uint64_t first, uint64_t count, GatherMap gm) {
    typedef typename CT<Real>::C C;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t c = first + i;
        uint64_t p = 0;
        for (int b = 0; b < gm.n; b++)
            if ((c >> b) & 1) p |= 1ull << gm.phys_of_canon_bit[b];
        const uint64_t r = p >> gm.n_loc;
        out[i] = (r == gm.rank) ? psi[p & ((1ull << gm.n_loc) - 1)] : mk<C>(0, 0);
    }
}

template <typename Real>
__global__ void set_one_kernel(typename CT<Real>::C *psi) {
    psi[0] = mk<typename CT<Real>::C>(1, 0);
}

// Remap exchange through bounded staging ("interchanging qubit
// positions" + redistribution; SURVEY.md §8(e) chunked exchange).  The exchange
// swaps global positions gpos[i] with local positions lpos[i]: with the partner
// rank whose gpos-bits equal b, this rank swaps its block b (the amplitudes whose
// lpos-bits equal b), chunk by chunk.  Element e of a block = the local index
// with the lpos-bits = b (bdep) and the remaining local bits (ascending, the mask
// `rest`) = e.  pack: stage[i] = shard[idx(e0 + i)]; unpack: the reverse.
__device__ __forceinline__ uint64_t pdep64(uint64_t v, uint64_t mask) {
    uint64_t r = 0;
    for (uint64_t bb = 1; mask; bb <<= 1) {
        const uint64_t low = mask & (~mask + 1);
        if (v & bb) r |= low;
        mask &= mask - 1;
    }
    return r;
}
template <typename Real>
__global__ void __launch_bounds__(256) remap_block_kernel(typename CT<Real>::C *__restrict__ shard,
                                                          typename CT<Real>::C *__restrict__ stage, uint64_t e0,
                                                          uint64_t cnt, uint64_t bdep, uint64_t rest, int unpack) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (uint64_t)gridDim.x * blockDim.x;
    if (t >= cnt) return;
    // deposit once, then step by a masked add (carries pass through the non-rest bits)
    uint64_t idx = pdep64(e0 + t, rest);
    const uint64_t sdep = pdep64(stride, rest);
    for (uint64_t i = t; i < cnt; i += stride) {
        const uint64_t p = idx | bdep;
        if (unpack) shard[p] = stage[i];
        else stage[i] = shard[p];
        idx = ((idx | ~rest) + sdep) & rest;
    }
}

// test hook (TQD_DEBUG_REMAP_DELAY_US): hold this rank's stream for a while so a
// peer runs ahead (exchange race tests); sleeps, waits on nothing
__global__ void debug_delay_kernel(uint32_t us) {
    for (uint32_t i = 0; i < us; i++) __nanosleep(1000);
}

// ---------------------------------------------------------------------------
// Launchers (host side, called from engine.cpp)
#define TQD_DECL(NAME)                                                                                          \
    cudaError_t launch_sweep_##NAME(const DevStage *, const void *, const int32_t *, void *, void *, double *,       \
                                    uint64_t, const ScatterInfo &, int, int, int, int, int, int, int, cudaStream_t); \
    int sweep_occupancy_##NAME(int k, int W, int n_ops, int n_slots, int nseg, int n_cvals);
TQD_DECL(f32_fwd)
TQD_DECL(f32_bwd)
TQD_DECL(f64_fwd)
TQD_DECL(f64_bwd)
#undef TQD_DECL

cudaError_t launch_sweep(bool dbl, bool bwd, const DevStage *d_stage, const void *d_kops, const int32_t *d_slots,
                         void *psi, void *lam, double *grad, uint64_t rank_hi, const ScatterInfo &sc, int k, int W,
                         int n_ops, int n_slots, int nseg, int n_cvals, int grid, cudaStream_t s) {
    if (dbl)
        return bwd ? launch_sweep_f64_bwd(d_stage, d_kops, d_slots, psi, lam, grad, rank_hi, sc, k, W, n_ops, n_slots, nseg, n_cvals, grid, s)
                   : launch_sweep_f64_fwd(d_stage, d_kops, d_slots, psi, lam, grad, rank_hi, sc, k, W, n_ops, n_slots, nseg, n_cvals, grid, s);
    return bwd ? launch_sweep_f32_bwd(d_stage, d_kops, d_slots, psi, lam, grad, rank_hi, sc, k, W, n_ops, n_slots, nseg, n_cvals, grid, s)
               : launch_sweep_f32_fwd(d_stage, d_kops, d_slots, psi, lam, grad, rank_hi, sc, k, W, n_ops, n_slots, nseg, n_cvals, grid, s);
}

int sweep_max_ctas_per_sm(bool dbl, bool bwd, int k, int W, int n_ops, int n_slots, int nseg, int n_cvals) {
    if (dbl)
        return bwd ? sweep_occupancy_f64_bwd(k, W, n_ops, n_slots, nseg, n_cvals)
                   : sweep_occupancy_f64_fwd(k, W, n_ops, n_slots, nseg, n_cvals);
    return bwd ? sweep_occupancy_f32_bwd(k, W, n_ops, n_slots, nseg, n_cvals)
               : sweep_occupancy_f32_fwd(k, W, n_ops, n_slots, nseg, n_cvals);
}

cudaError_t launch_small(bool dbl, bool bwd, const DevOp *d_ops, int n_ops, void *psi, void *lam, double *grad,
                         int n_loc, uint64_t rank_hi, int batch, cudaStream_t s) {
    const size_t esz = dbl ? 16 : 8;
    const size_t smem = (size_t)(bwd ? 2 : 1) * ((size_t)1 << n_loc) * esz;
    const int threads = 512;
#define TQD_S(T, BB)                                                                                   \
    {                                                                                                   \
        auto fn = small_kernel<T, BB>;                                                                  \
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); \
        if (e != cudaSuccess) return e;                                                                 \
        fn<<<batch, threads, smem, s>>>(d_ops, n_ops, (CT<T>::C *)psi, (CT<T>::C *)lam, grad, n_loc, rank_hi); \
        return cudaGetLastError();                                                                      \
    }
    if (dbl) { if (bwd) TQD_S(double, true) else TQD_S(double, false) }
    else { if (bwd) TQD_S(float, true) else TQD_S(float, false) }
#undef TQD_S
}

static int grid_for(uint64_t n, int threads) {
    uint64_t g = (n + threads - 1) / threads;
    if (g > 148 * 8) g = 148 * 8;
    if (g < 1) g = 1;
    return (int)g;
}

cudaError_t launch_lambda_init(bool dbl, const void *psi, void *lam, uint64_t n, uint64_t rank_hi, const ZTerms &t,
                               double *eout, cudaStream_t s) {
    const int th = 256;
    const int g = grid_for((n + 15) / 16, th);  // one 4096-amplitude chunk per CTA iteration
    if (dbl) lambda_init_kernel<double><<<g, th, 0, s>>>((const double2 *)psi, (double2 *)lam, n, rank_hi, t, eout);
    else lambda_init_kernel<float><<<g, th, 0, s>>>((const float2 *)psi, (float2 *)lam, n, rank_hi, t, eout);
    return cudaGetLastError();
}

cudaError_t launch_expval_z(bool dbl, const void *psi, uint64_t n, uint64_t rank_hi, const uint64_t *d_z, int T,
                            double *out, cudaStream_t s) {
    const int th = 256;
    const int g = grid_for((n + 15) / 16, th);  // one 4096-amplitude chunk per CTA iteration
    if (dbl) expval_z_kernel<double><<<g, th, 0, s>>>((const double2 *)psi, n, rank_hi, d_z, T, out);
    else expval_z_kernel<float><<<g, th, 0, s>>>((const float2 *)psi, n, rank_hi, d_z, T, out);
    return cudaGetLastError();
}

cudaError_t launch_expval_xy(bool dbl, const void *psi, const void *peer, uint64_t n, uint64_t rank_hi, uint64_t xloc,
                             const uint64_t *d_z, const int *d_ny, int T, double *out, cudaStream_t s) {
    const int th = 256;
    if (dbl)
        expval_xy_kernel<double><<<grid_for(n, th), th, 0, s>>>((const double2 *)psi, (const double2 *)peer, n, rank_hi,
                                                                xloc, d_z, d_ny, T, out);
    else
        expval_xy_kernel<float><<<grid_for(n, th), th, 0, s>>>((const float2 *)psi, (const float2 *)peer, n, rank_hi, xloc,
                                                               d_z, d_ny, T, out);
    return cudaGetLastError();
}

cudaError_t launch_lambda_add_xy(bool dbl, const void *psi, const void *peer, void *lam, uint64_t n, uint64_t rank_hi,
                                 uint64_t xloc, uint64_t xfull, const uint64_t *d_z, const int *d_ny, const double *d_c,
                                 int T, double *eout, cudaStream_t s) {
    const int th = 256;
    if (dbl)
        lambda_add_xy_kernel<double><<<grid_for(n, th), th, 0, s>>>((const double2 *)psi, (const double2 *)peer,
                                                                    (double2 *)lam, n, rank_hi, xloc, xfull, d_z, d_ny,
                                                                    d_c, T, eout);
    else
        lambda_add_xy_kernel<float><<<grid_for(n, th), th, 0, s>>>((const float2 *)psi, (const float2 *)peer,
                                                                   (float2 *)lam, n, rank_hi, xloc, xfull, d_z, d_ny,
                                                                   d_c, T, eout);
    return cudaGetLastError();
}

cudaError_t launch_gauss_sums(bool dbl, const void *psi, uint64_t n, uint64_t rank_hi, const GatherMap &gm, uint64_t seed,
                              const int *qpos, int nq, double *out, cudaStream_t s) {
    GaussQ gq;
    gq.nq = nq;
    for (int q = 0; q < 16; q++) gq.qpos[q] = (uint8_t)(q < nq ? qpos[q] : 0);
    const int th = 256;
    if (dbl) gauss_sums_kernel<double><<<grid_for(n, th), th, 0, s>>>((const double2 *)psi, n, rank_hi, gm, seed, gq, out);
    else gauss_sums_kernel<float><<<grid_for(n, th), th, 0, s>>>((const float2 *)psi, n, rank_hi, gm, seed, gq, out);
    return cudaGetLastError();
}

cudaError_t launch_lambda_gauss(bool dbl, const void *psi, void *lam, uint64_t n, uint64_t rank_hi, const GatherMap &gm,
                                uint64_t seed, const ZTerms &t, double alpha, double fc, double k2, double kc,
                                cudaStream_t s) {
    const int th = 256;
    if (dbl)
        lambda_gauss_kernel<double><<<grid_for(n, th), th, 0, s>>>((const double2 *)psi, (double2 *)lam, n, rank_hi, gm,
                                                                   seed, t, alpha, fc, k2, kc);
    else
        lambda_gauss_kernel<float><<<grid_for(n, th), th, 0, s>>>((const float2 *)psi, (float2 *)lam, n, rank_hi, gm,
                                                                  seed, t, alpha, fc, k2, kc);
    return cudaGetLastError();
}

cudaError_t launch_chunk_mass(bool dbl, const void *psi, uint64_t n_chunks, int csz, double *out, cudaStream_t s) {
    const int th = std::max(32, std::min(256, csz));
    const int grid = (int)std::min<uint64_t>(n_chunks, 148 * 8);
    if (dbl) chunk_mass_kernel<double><<<grid, th, 0, s>>>((const double2 *)psi, n_chunks, csz, out);
    else chunk_mass_kernel<float><<<grid, th, 0, s>>>((const float2 *)psi, n_chunks, csz, out);
    return cudaGetLastError();
}

cudaError_t launch_chunk_sample(bool dbl, const void *psi, int n_active, const uint64_t *chunk_id, const uint32_t *off,
                                const double *r, const uint64_t *shot_idx, uint64_t rank_hi, const GatherMap &gm,
                                int csz, double *out, cudaStream_t s) {
    if (n_active == 0) return cudaSuccess;
    const int th = std::max(32, std::min(256, csz));
    if (dbl)
        chunk_sample_kernel<double><<<n_active, th, 0, s>>>((const double2 *)psi, chunk_id, off, r, shot_idx, rank_hi, gm,
                                                           csz, out);
    else
        chunk_sample_kernel<float><<<n_active, th, 0, s>>>((const float2 *)psi, chunk_id, off, r, shot_idx, rank_hi, gm,
                                                          csz, out);
    return cudaGetLastError();
}

int sample_chunk_amps() { return SAMPLE_CHUNK; }

cudaError_t launch_gather(bool dbl, const void *psi, void *out, uint64_t first, uint64_t count, const GatherMap &gm,
                          cudaStream_t s) {
    const int th = 256;
    if (dbl) gather_kernel<double><<<grid_for(count, th), th, 0, s>>>((const double2 *)psi, (double2 *)out, first, count, gm);
    else gather_kernel<float><<<grid_for(count, th), th, 0, s>>>((const float2 *)psi, (float2 *)out, first, count, gm);
    return cudaGetLastError();
}

cudaError_t launch_set_one(bool dbl, void *psi, cudaStream_t s) {
    if (dbl) set_one_kernel<double><<<1, 1, 0, s>>>((double2 *)psi);
    else set_one_kernel<float><<<1, 1, 0, s>>>((float2 *)psi);
    return cudaGetLastError();
}

cudaError_t launch_remap_block(bool dbl, void *shard, void *stage, uint64_t e0, uint64_t cnt, uint64_t bdep, uint64_t rest,
                              bool unpack, cudaStream_t s) {
    if (cnt == 0) return cudaSuccess;
    const int th = 256;
    if (dbl) remap_block_kernel<double><<<grid_for(cnt, th), th, 0, s>>>((double2 *)shard, (double2 *)stage, e0, cnt, bdep, rest, unpack);
    else remap_block_kernel<float><<<grid_for(cnt, th), th, 0, s>>>((float2 *)shard, (float2 *)stage, e0, cnt, bdep, rest, unpack);
    return cudaGetLastError();
}
cudaError_t launch_debug_delay(uint32_t us, cudaStream_t s) {
    debug_delay_kernel<<<1, 1, 0, s>>>(us);
    return cudaGetLastError();
}

}  // namespace tqd
