// sweep.cuh -- the fused gate-sweep kernel (forward and adjoint), sm_100a.
//
// Forward (BWD = false): for every 2^k-amplitude tile of the shard, load it
// into registers (coalesced: lanes = physical bits 0..4), run the stage's gates
// (Y = M x_Q X per gate, Alg. 2's lazy order record = the
// layouts / qubit map pi), change register layout through shared memory where
// the next gates need other target bits, store (optionally onto permuted tile
// positions).  One HBM read + one HBM write per amplitude per stage.
//
// Adjoint (BWD = true): the same tile walk over psi and lambda together, gates
// in reverse: first the gradient partial 2 Re <lam|G_p|psi> on the post-gate
// states, then psi <- U^dag psi (x = U^* y) and
// lambda <- U^dag lambda (dx = U^T dy).
//
// Instantiated once per (precision, direction) in sweep_*.cu so nvcc compiles
// the four variants in parallel.
#pragma once
#include "common.cuh"
#include "tqd_internal.h"

namespace tqd {

constexpr int SWEEP_R = 4;  // register bits: 16 amplitudes (x2 states in the adjoint) per thread

template <int V> struct IC { static constexpr int value = V; };

template <int R, typename F> __device__ __forceinline__ void dispatch1(int t, F &&f) {
    switch (t) {
    case 0: f(IC<0>{}); break;
    case 1: if constexpr (R > 1) f(IC<1>{}); break;
    case 2: if constexpr (R > 2) f(IC<2>{}); break;
    case 3: if constexpr (R > 3) f(IC<3>{}); break;
    case 4: if constexpr (R > 4) f(IC<4>{}); break;
    default: break;
    }
}

// ---- register-level gates.  a[] = 2^R amplitudes; register index ri has bit i
// = value of tile-local bit lay.reg[i].  TB is compile time.  CTRL: pair (ri, rj)
// is updated only if (ri & cm) == cm and `on` (register / thread control).

template <int R, int TB, bool CTRL, typename C>
__device__ __forceinline__ void reg_u1(C *a, C m00, C m01, C m10, C m11, int cm, bool on) {
#pragma unroll
    for (int ri = 0; ri < (1 << R); ri++) {
        if (ri & (1 << TB)) continue;
        const int rj = ri | (1 << TB);
        const C x0 = a[ri], x1 = a[rj];
        const C y0 = cmul2(m00, x0, m01, x1), y1 = cmul2(m10, x0, m11, x1);
        if (CTRL) {
            const bool p = on && ((ri & cm) == cm);
            a[ri] = p ? y0 : x0;
            a[rj] = p ? y1 : x1;
        } else {
            a[ri] = y0;
            a[rj] = y1;
        }
    }
}

template <int R, int TB, bool CTRL, typename C, typename Real>
__device__ __forceinline__ void reg_r1(C *a, Real m00, Real m01, Real m10, Real m11, int cm, bool on) {
#pragma unroll
    for (int ri = 0; ri < (1 << R); ri++) {
        if (ri & (1 << TB)) continue;
        const int rj = ri | (1 << TB);
        const C x0 = a[ri], x1 = a[rj];
        const C y0 = mk<C>(m00 * x0.x + m01 * x1.x, m00 * x0.y + m01 * x1.y);
        const C y1 = mk<C>(m10 * x0.x + m11 * x1.x, m10 * x0.y + m11 * x1.y);
        if (CTRL) {
            const bool p = on && ((ri & cm) == cm);
            a[ri] = p ? y0 : x0;
            a[rj] = p ? y1 : x1;
        } else {
            a[ri] = y0;
            a[rj] = y1;
        }
    }
}

template <int R, int TB, bool CTRL, bool PLAIN, typename C>
__device__ __forceinline__ void reg_p1(C *a, C pa, C pb, int cm, bool on) {
#pragma unroll
    for (int ri = 0; ri < (1 << R); ri++) {
        if (ri & (1 << TB)) continue;
        const int rj = ri | (1 << TB);
        const C x0 = a[ri], x1 = a[rj];
        const C y0 = PLAIN ? x1 : cmul(pa, x1);
        const C y1 = PLAIN ? x0 : cmul(pb, x0);
        if (CTRL) {
            const bool p = on && ((ri & cm) == cm);
            a[ri] = p ? y0 : x0;
            a[rj] = p ? y1 : x1;
        } else {
            a[ri] = y0;
            a[rj] = y1;
        }
    }
}

template <int R, int TB, typename C>
__device__ __forceinline__ void reg_d1(C *a, C d0, C d1) {
#pragma unroll
    for (int ri = 0; ri < (1 << R); ri++) a[ri] = cmul((ri & (1 << TB)) ? d1 : d0, a[ri]);
}

template <int R, typename C>
__device__ __forceinline__ void reg_scale(C *a, C d) {
#pragma unroll
    for (int ri = 0; ri < (1 << R); ri++) a[ri] = cmul(d, a[ri]);
}

// diagonal 2q: phase index 2*v0 + v1; v = register bit (mask m != 0) or thread value rv
template <int R, typename C>
__device__ __forceinline__ void reg_d2(C *a, const C *d, int m0, int rv0, int m1, int rv1) {
#pragma unroll
    for (int ri = 0; ri < (1 << R); ri++) {
        const int v0 = m0 ? ((ri & m0) != 0) : rv0;
        const int v1 = m1 ? ((ri & m1) != 0) : rv1;
        const C e0 = v1 ? d[1] : d[0];
        const C e1 = v1 ? d[3] : d[2];
        a[ri] = cmul(v0 ? e1 : e0, a[ri]);
    }
}

template <int R, int T0, int T1, typename C>
__device__ __forceinline__ void reg_u2(C *a, const C *M) {
#pragma unroll
    for (int ri = 0; ri < (1 << R); ri++) {
        if (ri & ((1 << T0) | (1 << T1))) continue;
        const int idx[4] = {ri, ri | (1 << T1), ri | (1 << T0), ri | (1 << T0) | (1 << T1)};
        C v[4];
#pragma unroll
        for (int q = 0; q < 4; q++) v[q] = a[idx[q]];
#pragma unroll
        for (int r = 0; r < 4; r++) {
            C acc = cmul(M[4 * r], v[0]);
#pragma unroll
            for (int q = 1; q < 4; q++) {
                const C p = cmul(M[4 * r + q], v[q]);
                acc.x += p.x;
                acc.y += p.y;
            }
            a[idx[r]] = acc;
        }
    }
}

// ---- gradient partials: 2 Re <lam|G|psi> over this thread's amplitudes ----
template <int R, int TB, typename C, typename Real>
__device__ __forceinline__ Real grad_pair(const C *a, const C *l, int gk, const double *g) {
    Real acc = 0;
    if (gk == GEN_Y) {  // G = -(i/2) Y = [[0, -1/2], [1/2, 0]]
#pragma unroll
        for (int ri = 0; ri < (1 << R); ri++) {
            if (ri & (1 << TB)) continue;
            const int rj = ri | (1 << TB);
            acc += re_cj(l[rj], a[ri]) - re_cj(l[ri], a[rj]);
        }
    } else if (gk == GEN_X) {  // G = -(i/2) X
#pragma unroll
        for (int ri = 0; ri < (1 << R); ri++) {
            if (ri & (1 << TB)) continue;
            const int rj = ri | (1 << TB);
            acc += im_cj(l[ri], a[rj]) + im_cj(l[rj], a[ri]);
        }
    } else {  // general anti-Hermitian generator
        const C g00 = ldc<C>(g, 0), g01 = ldc<C>(g, 1), g10 = ldc<C>(g, 2), g11 = ldc<C>(g, 3);
#pragma unroll
        for (int ri = 0; ri < (1 << R); ri++) {
            if (ri & (1 << TB)) continue;
            const int rj = ri | (1 << TB);
            const C v0 = cmul2(g00, a[ri], g01, a[rj]);
            const C v1 = cmul2(g10, a[ri], g11, a[rj]);
            acc += 2 * (re_cj(l[ri], v0) + re_cj(l[rj], v1));
        }
    }
    return acc;
}

// RZ generator G = -(i/2) Z on a register bit: sum_b z_b Im(conj(lam_b) psi_b)
template <int R, int TB, typename C, typename Real>
__device__ __forceinline__ Real grad_z_reg(const C *a, const C *l) {
    Real acc = 0;
#pragma unroll
    for (int ri = 0; ri < (1 << R); ri++) {
        const Real v = im_cj(l[ri], a[ri]);
        acc += (ri & (1 << TB)) ? -v : v;
    }
    return acc;
}

template <int R, typename C, typename Real>
__device__ __forceinline__ Real grad_z_const(const C *a, const C *l, int bit) {
    Real acc = 0;
#pragma unroll
    for (int ri = 0; ri < (1 << R); ri++) acc += im_cj(l[ri], a[ri]);
    return bit ? -acc : acc;
}

// ---- one op on the register file ----
template <typename Real, int R, bool BWD>
__device__ __forceinline__ void run_op(const DevOp &op, typename CT<Real>::C *a, typename CT<Real>::C *l,
                                       uint32_t tix, uint64_t basefull, double *sacc) {
    typedef typename CT<Real>::C C;
    auto bitval = [&](BitRef b) -> int {
        return b.kind == BK_TIX ? (int)((tix >> b.idx) & 1u) : (int)((basefull >> b.idx) & 1ull);
    };
    const int kind = op.kind;

    if (BWD && op.ngen) {
        for (int gi = 0; gi < op.ngen; gi++) {
            Real part = 0;
            const int gk = op.gkind[gi];
            if (kind == OP_D1) {
                if (op.b0.kind == BK_REG)
                    dispatch1<R>(op.b0.idx, [&](auto tb) { part = grad_z_reg<R, decltype(tb)::value, C, Real>(a, l); });
                else
                    part = grad_z_const<R, C, Real>(a, l, bitval(op.b0));
            } else {
                dispatch1<R>(op.t0, [&](auto tb) { part = grad_pair<R, decltype(tb)::value, C, Real>(a, l, gk, op.g[gi]); });
            }
            part = warp_sum(part);
            if ((threadIdx.x & 31) == 0) atomicAdd(&sacc[op.slot[gi]], (double)part);
        }
    }

    bool on = true;
    int cm = 0;
    if (op.ctrl.kind == BK_REG) cm = 1 << op.ctrl.idx;
    else if (op.ctrl.kind != BK_NONE) on = bitval(op.ctrl) != 0;
    const bool ctrl = (cm != 0) || (op.ctrl.kind != BK_NONE);

    switch (kind) {
    case OP_U1: {
        const C m00 = ldc<C>(op.m, 0), m01 = ldc<C>(op.m, 1), m10 = ldc<C>(op.m, 2), m11 = ldc<C>(op.m, 3);
        dispatch1<R>(op.t0, [&](auto tb) {
            constexpr int TB = decltype(tb)::value;
            if (ctrl) {
                reg_u1<R, TB, true>(a, m00, m01, m10, m11, cm, on);
                if (BWD) reg_u1<R, TB, true>(l, m00, m01, m10, m11, cm, on);
            } else {
                reg_u1<R, TB, false>(a, m00, m01, m10, m11, 0, true);
                if (BWD) reg_u1<R, TB, false>(l, m00, m01, m10, m11, 0, true);
            }
        });
        break;
    }
    case OP_R1: {
        const Real m00 = (Real)op.m[0], m01 = (Real)op.m[1], m10 = (Real)op.m[2], m11 = (Real)op.m[3];
        dispatch1<R>(op.t0, [&](auto tb) {
            constexpr int TB = decltype(tb)::value;
            if (ctrl) {
                reg_r1<R, TB, true, C, Real>(a, m00, m01, m10, m11, cm, on);
                if (BWD) reg_r1<R, TB, true, C, Real>(l, m00, m01, m10, m11, cm, on);
            } else {
                reg_r1<R, TB, false, C, Real>(a, m00, m01, m10, m11, 0, true);
                if (BWD) reg_r1<R, TB, false, C, Real>(l, m00, m01, m10, m11, 0, true);
            }
        });
        break;
    }
    case OP_P1: {
        const C pa = ldc<C>(op.m, 0), pb = ldc<C>(op.m, 1);
        const bool plain = op.t1 != 0;
        dispatch1<R>(op.t0, [&](auto tb) {
            constexpr int TB = decltype(tb)::value;
            if (plain) {
                if (ctrl) {
                    reg_p1<R, TB, true, true>(a, pa, pb, cm, on);
                    if (BWD) reg_p1<R, TB, true, true>(l, pa, pb, cm, on);
                } else {
                    reg_p1<R, TB, false, true>(a, pa, pb, 0, true);
                    if (BWD) reg_p1<R, TB, false, true>(l, pa, pb, 0, true);
                }
            } else {
                if (ctrl) {
                    reg_p1<R, TB, true, false>(a, pa, pb, cm, on);
                    if (BWD) reg_p1<R, TB, true, false>(l, pa, pb, cm, on);
                } else {
                    reg_p1<R, TB, false, false>(a, pa, pb, 0, true);
                    if (BWD) reg_p1<R, TB, false, false>(l, pa, pb, 0, true);
                }
            }
        });
        break;
    }
    case OP_D1: {
        const C d0 = ldc<C>(op.m, 0), d1 = ldc<C>(op.m, 1);
        if (op.b0.kind == BK_REG) {
            dispatch1<R>(op.b0.idx, [&](auto tb) {
                reg_d1<R, decltype(tb)::value>(a, d0, d1);
                if (BWD) reg_d1<R, decltype(tb)::value>(l, d0, d1);
            });
        } else {
            const C d = bitval(op.b0) ? d1 : d0;
            reg_scale<R>(a, d);
            if (BWD) reg_scale<R>(l, d);
        }
        break;
    }
    case OP_D2: {
        C d[4];
#pragma unroll
        for (int q = 0; q < 4; q++) d[q] = ldc<C>(op.m, q);
        const int m0 = op.b0.kind == BK_REG ? (1 << op.b0.idx) : 0;
        const int m1 = op.b1.kind == BK_REG ? (1 << op.b1.idx) : 0;
        const int v0 = m0 ? 0 : bitval(op.b0);
        const int v1 = m1 ? 0 : bitval(op.b1);
        reg_d2<R>(a, d, m0, v0, m1, v1);
        if (BWD) reg_d2<R>(l, d, m0, v0, m1, v1);
        break;
    }
    case OP_U2: {
        C M[16];
#pragma unroll
        for (int q = 0; q < 16; q++) M[q] = ldc<C>(op.m, q);
        dispatch1<R>(op.t0, [&](auto c0) {
            dispatch1<R>(op.t1, [&](auto c1) {
                constexpr int T0 = decltype(c0)::value, T1 = decltype(c1)::value;
                if constexpr (T0 != T1) {
                    reg_u2<R, T0, T1>(a, M);
                    if (BWD) reg_u2<R, T0, T1>(l, M);
                }
            });
        });
        break;
    }
    default: break;
    }
}

// ---- the fused sweep kernel: one CTA = 32 * 2^W threads, persistent over tiles
template <typename Real, int R, bool BWD>
__global__ void __launch_bounds__(256) sweep_kernel(const DevStage *__restrict__ stg, const DevOp *__restrict__ ops,
                                                    const int32_t *__restrict__ slot_param,
                                                    typename CT<Real>::C *__restrict__ psi,
                                                    typename CT<Real>::C *__restrict__ lam,
                                                    double *__restrict__ grad, uint64_t rank_hi) {
    typedef typename CT<Real>::C C;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ DevStage S;
    __shared__ double sacc[BWD ? MAX_STAGE_SLOTS : 1];

    {
        const uint32_t *src = reinterpret_cast<const uint32_t *>(stg);
        uint32_t *dst = reinterpret_cast<uint32_t *>(&S);
        for (int i = threadIdx.x; i < (int)(sizeof(DevStage) / 4); i += blockDim.x) dst[i] = src[i];
        if (BWD)
            for (int i = threadIdx.x; i < MAX_STAGE_SLOTS; i += blockDim.x) sacc[i] = 0.0;
    }
    __syncthreads();

    const int k = S.k;
    const int W = S.W;
    const int nseg = S.nseg;
    C *sm_a = reinterpret_cast<C *>(smem_raw);
    C *sm_l = sm_a + ((size_t)1 << k);
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const DevOp *sops = ops + S.op_base;

    auto thr_phys_off = [&](const DevLayout &L, const uint8_t *phys) -> uint64_t {
        uint64_t off = 0;
#pragma unroll
        for (int i = 0; i < LANE_BITS; i++)
            if ((lane >> i) & 1) off |= 1ull << phys[L.lane[i]];
        for (int w = 0; w < W; w++)
            if ((warp >> w) & 1) off |= 1ull << phys[L.warp[w]];
        return off;
    };
    auto thr_tix = [&](const DevLayout &L) -> uint32_t {
        uint32_t t = 0;
#pragma unroll
        for (int i = 0; i < LANE_BITS; i++) t |= (uint32_t)((lane >> i) & 1) << L.lane[i];
        for (int w = 0; w < W; w++) t |= (uint32_t)((warp >> w) & 1) << L.warp[w];
        return t;
    };
    auto thr_sm = [&](const DevLayout &L) -> uint32_t {
        uint32_t t = 0;
#pragma unroll
        for (int i = 0; i < LANE_BITS; i++)
            if ((lane >> i) & 1) t ^= S.swz[L.lane[i]];
        for (int w = 0; w < W; w++)
            if ((warp >> w) & 1) t ^= S.swz[L.warp[w]];
        return t;
    };

    for (int64_t tile = blockIdx.x; tile < S.n_tiles; tile += gridDim.x) {
        // deposit the tile index into the non-tile physical positions
        uint64_t base = (uint64_t)tile;
        for (int i = 0; i < k; i++) {
            const int p = S.tile_sorted[i];
            base = ((base >> p) << (p + 1)) | (base & ((1ull << p) - 1));
        }
        const uint64_t basefull = base | rank_hi;

        C a[1 << R];
        C l[BWD ? (1 << R) : 1];
        {
            const DevLayout &L = S.lay[0];
            const uint64_t off = base | thr_phys_off(L, S.ld_phys);
            uint64_t roff[R];
#pragma unroll
            for (int i = 0; i < R; i++) roff[i] = 1ull << S.ld_phys[L.reg[i]];
#pragma unroll
            for (int ri = 0; ri < (1 << R); ri++) {
                uint64_t o = off;
#pragma unroll
                for (int i = 0; i < R; i++)
                    if (ri & (1 << i)) o |= roff[i];
                a[ri] = psi[o];
                if (BWD) l[ri] = lam[o];
            }
        }

        for (int s = 0; s < nseg; s++) {
            if (s > 0) {  // layout change through shared memory
                const DevLayout &Lw = S.lay[s - 1];
                const DevLayout &Lr = S.lay[s];
                const uint32_t tw = thr_sm(Lw), tr = thr_sm(Lr);
                uint32_t cw[R], cr[R];
#pragma unroll
                for (int i = 0; i < R; i++) { cw[i] = S.swz[Lw.reg[i]]; cr[i] = S.swz[Lr.reg[i]]; }
#pragma unroll
                for (int ri = 0; ri < (1 << R); ri++) {
                    uint32_t o = tw;
#pragma unroll
                    for (int i = 0; i < R; i++)
                        if (ri & (1 << i)) o ^= cw[i];
                    sm_a[o] = a[ri];
                    if (BWD) sm_l[o] = l[ri];
                }
                __syncthreads();
#pragma unroll
                for (int ri = 0; ri < (1 << R); ri++) {
                    uint32_t o = tr;
#pragma unroll
                    for (int i = 0; i < R; i++)
                        if (ri & (1 << i)) o ^= cr[i];
                    a[ri] = sm_a[o];
                    if (BWD) l[ri] = sm_l[o];
                }
                __syncthreads();
            }
            const uint32_t tix = thr_tix(S.lay[s]);
            const int e = S.seg_begin[s + 1];
            for (int oi = S.seg_begin[s]; oi < e; oi++) run_op<Real, R, BWD>(sops[oi], a, l, tix, basefull, sacc);
        }

        {
            const DevLayout &L = S.lay[nseg - 1];
            const uint64_t off = base | thr_phys_off(L, S.st_phys);
            uint64_t roff[R];
#pragma unroll
            for (int i = 0; i < R; i++) roff[i] = 1ull << S.st_phys[L.reg[i]];
#pragma unroll
            for (int ri = 0; ri < (1 << R); ri++) {
                uint64_t o = off;
#pragma unroll
                for (int i = 0; i < R; i++)
                    if (ri & (1 << i)) o |= roff[i];
                psi[o] = a[ri];
                if (BWD) lam[o] = l[ri];
            }
        }
    }

    if (BWD) {
        __syncthreads();
        for (int i = threadIdx.x; i < S.n_slots; i += blockDim.x) {
            const double v = sacc[i];
            if (v != 0.0) atomicAdd(&grad[slot_param[S.slot_base + i]], v);
        }
    }
}

template <typename Real, bool BWD>
static size_t sweep_smem_bytes(int k) {
    return (size_t)(BWD ? 2 : 1) * ((size_t)1 << k) * sizeof(typename CT<Real>::C);
}

template <typename Real, bool BWD>
cudaError_t launch_sweep_impl(const DevStage *d_stage, const DevOp *d_ops, const int32_t *d_slots, void *psi, void *lam,
                              double *grad, uint64_t rank_hi, int k, int W, int grid, cudaStream_t s) {
    typedef typename CT<Real>::C C;
    auto fn = sweep_kernel<Real, SWEEP_R, BWD>;
    const size_t smem = sweep_smem_bytes<Real, BWD>(k);
    static size_t attr = 0;
    if (smem > attr) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr = smem;
    }
    fn<<<grid, 32 << W, smem, s>>>(d_stage, d_ops, d_slots, (C *)psi, (C *)lam, grad, rank_hi);
    return cudaGetLastError();
}

template <typename Real, bool BWD>
int sweep_occupancy_impl(int k, int W) {
    auto fn = sweep_kernel<Real, SWEEP_R, BWD>;
    const size_t smem = sweep_smem_bytes<Real, BWD>(k);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, 32 << W, smem) != cudaSuccess) {
        cudaGetLastError();
        return 1;
    }
    return nb;
}

}  // namespace tqd

#define TQD_INSTANTIATE_SWEEP(REAL, BWD, NAME)                                                                    \
    namespace tqd {                                                                                             \
    cudaError_t launch_sweep_##NAME(const DevStage *d_stage, const DevOp *d_ops, const int32_t *d_slots, void *psi, \
                                    void *lam, double *grad, uint64_t rank_hi, int k, int W, int grid,             \
                                    cudaStream_t s) {                                                             \
        return launch_sweep_impl<REAL, BWD>(d_stage, d_ops, d_slots, psi, lam, grad, rank_hi, k, W, grid, s);     \
    }                                                                                                           \
    int sweep_occupancy_##NAME(int k, int W) { return sweep_occupancy_impl<REAL, BWD>(k, W); }                  \
    }
