// sweep.cuh -- the fused gate-sweep kernel (forward and adjoint), sm_100a.
//
// Forward (BWD = false): for every 2^k-amplitude tile of the shard, load it
// into registers (coalesced: lanes = physical bits 0..4), run the stage's gates
// (Y = M x_Q X per gate; Alg. 2's lazy order record = the
// register layouts + qubit map pi), change register layout through shared
// memory where the next gates need other target bits, store (optionally onto
// permuted tile positions).  One HBM read + one HBM write per amplitude per
// stage, whatever the number of gates in it.
//
// Adjoint (BWD = true): the same tile walk over psi and lambda together, gates
// in reverse: first the gradient partials 2 Re <lam|G_p|psi> on the post-gate
// states, then psi <- U^dag psi (x = U^* y) and
// lambda <- U^dag lambda (dx = U^T dy).
//
// Register file: each thread holds 2^R amplitudes (x2 in the adjoint) in TWO
// buffers A and B; ops alternate A->B, B->A.  Every op therefore writes fresh
// registers, so the runtime op dispatch needs no register shuffling at the
// loop back-edge (the v1 kernel spent 28% of its instructions on MOVs there,
// profiles/r01_v1_*_ncu.json).
//
// Instantiated once per (precision, direction) in sweep_*.cu.
#pragma once
#include <atomic>

#include "common.cuh"
#include "tqd_internal.h"

namespace tqd {

constexpr int SWEEP_R = TQD_SWEEP_R;  // register bits: 2^R amplitudes (x2 states in the adjoint) per thread
#ifndef TQD_LB_THREADS
#define TQD_LB_THREADS (32 << (12 - 5 - SWEEP_R))  // threads per CTA at k = 12
#endif
#ifndef TQD_LB_MINB_F32_BWD
#define TQD_LB_MINB_F32_BWD 2
#endif
#ifndef TQD_LB_MINB_F32_FWD
#define TQD_LB_MINB_F32_FWD (SWEEP_R == 3 ? 2 : 3)
#endif
constexpr int SWEEP_THREADS = TQD_LB_THREADS;
constexpr int NR = 1 << SWEEP_R;
constexpr int MAX_WARPS = 1 << WMAX;

template <int V> struct IC { static constexpr int value = V; };
__host__ __device__ constexpr int ctz4(int m) { return (m & 1) ? 0 : (m & 2) ? 1 : (m & 4) ? 2 : 3; }

template <typename F> __device__ __forceinline__ void dispatch4(int t, F &&f) {
    switch (t) {
    case 0: f(IC<0>{}); break;
    case 1: f(IC<1>{}); break;
    case 2: f(IC<2>{}); break;
    default: f(IC<3>{}); break;
    }
}

template <typename F> __device__ __forceinline__ void dispatch16(int t, F &&f) {
    switch (t) {
    case 0: f(IC<0>{}); break;   case 1: f(IC<1>{}); break;   case 2: f(IC<2>{}); break;
    case 3: f(IC<3>{}); break;   case 4: f(IC<4>{}); break;   case 5: f(IC<5>{}); break;
    case 6: f(IC<6>{}); break;   case 7: f(IC<7>{}); break;   case 8: f(IC<8>{}); break;
    case 9: f(IC<9>{}); break;   case 10: f(IC<10>{}); break; case 11: f(IC<11>{}); break;
    case 12: f(IC<12>{}); break; case 13: f(IC<13>{}); break; case 14: f(IC<14>{}); break;
    default: f(IC<15>{}); break;
    }
}

// ---- complex helpers on packed coefficients --------------------------------
// complex coefficient stored as (re, 0, im, im) at e[0..3]:
//   cmul_e(e, x) = e * x,  cfma_e(e, x, acc) = acc + e * x
// float: a packed FMUL2/FFMA2 with the real part broadcast + one FFMA2 with the
// halves of x swapped and the (im, im) pair half-negated; double: scalar.
__device__ __forceinline__ float2 cmul_e(const float *e, float2 x) {
    const float4 v = *reinterpret_cast<const float4 *>(e);
    return __ffma2_rn(make_float2(-v.z, v.w), make_float2(x.y, x.x), __fmul2_rn(make_float2(v.x, v.x), x));
}
__device__ __forceinline__ float2 cfma_e(const float *e, float2 x, float2 acc) {
    const float4 v = *reinterpret_cast<const float4 *>(e);
    return __ffma2_rn(make_float2(-v.z, v.w), make_float2(x.y, x.x), __ffma2_rn(make_float2(v.x, v.x), x, acc));
}
__device__ __forceinline__ double2 cmul_e(const double *e, double2 x) {
    return make_double2(e[0] * x.x - e[2] * x.y, e[0] * x.y + e[2] * x.x);
}
__device__ __forceinline__ double2 cfma_e(const double *e, double2 x, double2 acc) {
    return make_double2(acc.x + e[0] * x.x - e[2] * x.y, acc.y + e[0] * x.y + e[2] * x.x);
}

// ---- layer ops: one 2x2 per active register bit, in place -------------------
template <int MASK, typename C, typename Real>
__device__ __forceinline__ void layer_gen(C *t, const Real *m) {
#pragma unroll
    for (int b = 0; b < SWEEP_R; b++) {
        if (!((MASK >> b) & 1)) continue;
        const Real *mb = m + 16 * b;  // entries 00, 01, 10, 11
#pragma unroll
        for (int r = 0; r < NR; r++) {
            if (r & (1 << b)) continue;
            const int s = r | (1 << b);
            const C x0 = t[r], x1 = t[s];
            t[r] = cfma_e(mb + 4, x1, cmul_e(mb, x0));
            t[s] = cfma_e(mb + 12, x1, cmul_e(mb + 8, x0));
        }
    }
}

// y = a*x + b*y for a complex pair with real coefficients: one packed f32x2
// FMUL + FFMA per amplitude on sm_100a (fma.rn.f32x2), scalar in double
__device__ __forceinline__ float2 raxpy(float a, float2 x, float b, float2 y) {
    return __ffma2_rn(make_float2(b, b), y, __fmul2_rn(make_float2(a, a), x));
}
__device__ __forceinline__ double2 raxpy(double a, double2 x, double b, double2 y) {
    return make_double2(a * x.x + b * y.x, a * x.y + b * y.y);
}

template <int MASK, typename C, typename Real>
__device__ __forceinline__ void layer_real(C *t, const Real *m) {
#pragma unroll
    for (int b = 0; b < SWEEP_R; b++) {
        if (!((MASK >> b) & 1)) continue;
        const Real *mb = m + 8 * b;
        const Real m00 = mb[0], m01 = mb[1], m10 = mb[2], m11 = mb[3];
#pragma unroll
        for (int r = 0; r < NR; r++) {
            if (r & (1 << b)) continue;
            const int s = r | (1 << b);
            const C x0 = t[r], x1 = t[s];
            t[r] = raxpy(m00, x0, m01, x1);
            t[s] = raxpy(m10, x0, m11, x1);
        }
    }
}

// diagonal layer: m holds the 16 phase products ph[r] = prod_b d_b[bit_b(r)]
// (built on the host): one complex multiply per amplitude for up to 4 gates
template <typename C, typename Real>
__device__ __forceinline__ void layer_diag(C *t, const Real *m) {
#pragma unroll
    for (int r = 0; r < NR; r++) t[r] = cmul_e(m + 4 * r, t[r]);
}

// controlled general 2x2 (rare: controlled MAT2), in place; runtime control
template <int T, typename C, typename Real>
__device__ __forceinline__ void op_cu(C *a, const Real *m, int cm, bool on) {
    if constexpr (T >= SWEEP_R) return;
#pragma unroll
    for (int r = 0; r < NR; r++) {
        if (r & (1 << T)) continue;
        const int s = r | (1 << T);
        const C x0 = a[r], x1 = a[s];
        const C y0 = cfma_e(m + 4, x1, cmul_e(m, x0)), y1 = cfma_e(m + 12, x1, cmul_e(m + 8, x0));
        const Real p = (on && ((r & cm) == cm)) ? (Real)1 : (Real)0;  // arithmetic blend: no register moves
        a[r] = mk<C>(x0.x + p * (y0.x - x0.x), x0.y + p * (y0.y - x0.y));
        a[s] = mk<C>(x1.x + p * (y1.x - x1.x), x1.y + p * (y1.y - x1.y));
    }
}

template <int T0, int T1, typename C, typename Real>
__device__ __forceinline__ void op_u2(C *a, const Real *m) {
    if constexpr (T0 >= SWEEP_R || T1 >= SWEEP_R) return;
#pragma unroll
    for (int r = 0; r < NR; r++) {
        if (r & ((1 << T0) | (1 << T1))) continue;
        const int idx[4] = {r, r | (1 << T1), r | (1 << T0), r | (1 << T0) | (1 << T1)};
        C v[4];
#pragma unroll
        for (int q = 0; q < 4; q++) v[q] = a[idx[q]];
#pragma unroll
        for (int i = 0; i < 4; i++) {
            C acc = cmul_e(m + 16 * i, v[0]);
#pragma unroll
            for (int q = 1; q < 4; q++) acc = cfma_e(m + 16 * i + 4 * q, v[q], acc);
            a[idx[i]] = acc;
        }
    }
}

// diagonal 2q on arbitrary bits: v = register bit (mask) or per-thread value
template <typename C, typename Real>
__device__ __forceinline__ void op_d2(C *a, const Real *m, int m0, int rv0, int m1, int rv1) {
#pragma unroll
    for (int r = 0; r < NR; r++) {
        const int v0 = m0 ? ((r & m0) != 0) : rv0;
        const int v1 = m1 ? ((r & m1) != 0) : rv1;
        a[r] = cmul_e(m + 4 * (2 * v0 + v1), a[r]);
    }
}

// ---- gradient partials on (psi, lambda): 2 Re <lam|G|psi> --------------------
// element-wise x*y + z on the (re, im) pair (packed f32x2 FMA for float)
__device__ __forceinline__ float2 cfma_elem(float2 x, float2 y, float2 z) { return __ffma2_rn(x, y, z); }
__device__ __forceinline__ double2 cfma_elem(double2 x, double2 y, double2 z) {
    return make_double2(fma(x.x, y.x, z.x), fma(x.y, y.y, z.y));
}
template <int T, typename C, typename Real>
__device__ __forceinline__ Real grad_bit(const C *a, const C *l, int gk, const Real *g) {
    Real acc = 0;
    if constexpr (T >= SWEEP_R) return acc;
    if (gk == GEN_Y) {  // G = -(i/2) Y = [[0, -1/2], [1/2, 0]]: Re(conj l1 a0) - Re(conj l0 a1)
        C pos = mk<C>(0, 0), neg = mk<C>(0, 0);
#pragma unroll
        for (int r = 0; r < NR; r++) {
            if (r & (1 << T)) continue;
            const int s = r | (1 << T);
            pos = cfma_elem(l[s], a[r], pos);
            neg = cfma_elem(l[r], a[s], neg);
        }
        acc = (pos.x + pos.y) - (neg.x + neg.y);
    } else if (gk == GEN_X) {  // G = -(i/2) X
#pragma unroll
        for (int r = 0; r < NR; r++) {
            if (r & (1 << T)) continue;
            const int s = r | (1 << T);
            acc += im_cj(l[r], a[s]) + im_cj(l[s], a[r]);
        }
    } else if (gk == GEN_Z) {  // G = -(i/2) Z: sum_b z_b Im(conj(lam_b) psi_b)
#pragma unroll
        for (int r = 0; r < NR; r++) {
            const Real v = im_cj(l[r], a[r]);
            acc += (r & (1 << T)) ? -v : v;
        }
    } else {  // general anti-Hermitian generator
        const C g00 = mk<C>(g[0], g[1]), g01 = mk<C>(g[2], g[3]), g10 = mk<C>(g[4], g[5]), g11 = mk<C>(g[6], g[7]);
#pragma unroll
        for (int r = 0; r < NR; r++) {
            if (r & (1 << T)) continue;
            const int s = r | (1 << T);
            const C v0 = cmul2(g00, a[r], g01, a[s]);
            const C v1 = cmul2(g10, a[r], g11, a[s]);
            acc += 2 * (re_cj(l[r], v0) + re_cj(l[s], v1));
        }
    }
    return acc;
}

template <typename C, typename Real>
__device__ __forceinline__ Real grad_z_const(const C *a, const C *l, int bit) {
    Real acc = 0;
#pragma unroll
    for (int r = 0; r < NR; r++) acc += im_cj(l[r], a[r]);
    return bit ? -acc : acc;
}

// ---- layer fast paths (adjoint): gradients of every RY / RZ of a layer ----------
// packed helpers: (x.x + y.x, x.y + y.y) and (x.x - y.x, x.y - y.y)
__device__ __forceinline__ float2 padd(float2 x, float2 y) { return __fadd2_rn(x, y); }
__device__ __forceinline__ float2 psub(float2 x, float2 y) { return __fadd2_rn(x, make_float2(-y.x, -y.y)); }
__device__ __forceinline__ double2 padd(double2 x, double2 y) { return make_double2(x.x + y.x, x.y + y.y); }
__device__ __forceinline__ double2 psub(double2 x, double2 y) { return make_double2(x.x - y.x, x.y - y.y); }
template <typename C> __device__ __forceinline__ C pneg(C x) { return mk<C>(-x.x, -x.y); }
template <typename C> __device__ __forceinline__ C pswap(C x) { return mk<C>(x.y, x.x); }
__device__ __forceinline__ float2 pmul(float2 x, float2 y) { return __fmul2_rn(x, y); }
__device__ __forceinline__ double2 pmul(double2 x, double2 y) { return make_double2(x.x * y.x, x.y * y.y); }

// RY generator G = -(i/2) Y on register bit T:
//   2 Re <lam|G|psi> = sum_pairs Re(conj l1 a0) - Re(conj l0 a1)
// two packed accumulators (independent FFMA2 chains), one final add
#ifndef TQD_GRAD_CHAINS
#define TQD_GRAD_CHAINS 1  // FFMA2 accumulator chains per RY gradient (1: fewer live registers; 1 / 2 / 4 measured
                           // 10.53 / 10.66 / 10.70 ms per adjoint sweep at 30 q)
#endif
template <int T, typename C, typename Real>
__device__ __forceinline__ Real grad_y(const C *a, const C *l) {
    if constexpr (T >= SWEEP_R) return (Real)0;
    constexpr int NC = TQD_GRAD_CHAINS;
    C acc[NC];
#pragma unroll
    for (int c = 0; c < NC; c++) acc[c] = mk<C>(0, 0);
    int i = 0;
#pragma unroll
    for (int r = 0; r < NR; r++) {
        if (r & (1 << T)) continue;
        const int s = r | (1 << T);
        acc[i % NC] = cfma_elem(l[s], a[r], acc[i % NC]);
        acc[(i + 1) % NC] = cfma_elem(pneg(l[r]), a[s], acc[(i + 1) % NC]);
        i += 2;
    }
#pragma unroll
    for (int c = 1; c < NC; c++) acc[0] = padd(acc[0], acc[c]);
    return acc[0].x + acc[0].y;
}

template <int MASK, typename C, typename Real>
__device__ __forceinline__ void grad_y_layer(const C *a, const C *l, uint32_t gm, const uint16_t *soff, Real *tt) {
    if constexpr ((MASK & 1) != 0) if (gm & 1) tt[soff[0]] += grad_y<0, C, Real>(a, l);
    if constexpr ((MASK & 2) != 0) if (gm & 2) tt[soff[1]] += grad_y<1, C, Real>(a, l);
    if constexpr ((MASK & 4) != 0) if (gm & 4) tt[soff[2]] += grad_y<2, C, Real>(a, l);
    if constexpr ((MASK & 8) != 0 && SWEEP_R > 3) if (gm & 8) tt[soff[3]] += grad_y<3, C, Real>(a, l);
}

// RZ generators G = -(i/2) Z on the register bits of a diagonal layer:
//   g_b = sum_r (-1)^{bit_b(r)} w_r,  w_r = Im(conj(lam_r) psi_r) = p_r.x - p_r.y
// with p_r = lam_r * swap(psi_r) (packed); single-bit Walsh sums by a packed
// butterfly (differences at each level, sums carried up)
template <typename C, typename Real>
__device__ __forceinline__ void grad_z_layer(const C *a, const C *l, uint32_t gm, const uint16_t *soff, Real *tt) {
    C cur[NR];
#pragma unroll
    for (int r = 0; r < NR; r++) cur[r] = pmul(l[r], pswap(a[r]));
#pragma unroll
    for (int b = 0; b < SWEEP_R; b++) {
        // level b: pairs differ in original bit b; differences summed, sums carried up
        const int half = NR >> (b + 1);
        C d = psub(cur[0], cur[1]);
        cur[0] = padd(cur[0], cur[1]);
#pragma unroll
        for (int j = 1; j < half; j++) {
            d = padd(d, psub(cur[2 * j], cur[2 * j + 1]));
            cur[j] = padd(cur[2 * j], cur[2 * j + 1]);
        }
        if ((gm >> b) & 1) tt[soff[b]] += d.x - d.y;
    }
}

// ---- diagonal block (K_DBLK, tqd_internal.h DTerm): one phase per amplitude for
// a whole run of diagonal gates.  Per thread: fixed-point turn sums of the terms
// whose lane / warp / base bits are set (th: constant, al[b]: per register bit),
// phases by sincospi, then exp(i Phi(r)) = table[r] * w(r) with
// w(r) = e^{i th} prod_{b in r} e^{i al[b]}.
// e^{i 2 pi u / 2^32} (float) / e^{i 2 pi u / 2^64} (double) from a 256-entry
// table of e^{i 2 pi k / 256} (shared memory, built per CTA) times a short Taylor
// series of the remaining angle delta < 2 pi / 256 (errors < 2e-8 / 1e-20)
__device__ __forceinline__ float2 cis_turn(uint32_t u, const float2 *tab) {
    const float2 t = tab[u >> 24];
    const float d = (float)(u & 0xffffffu) * 1.4629180792671596e-09f;  // 2 pi / 2^32
    const float d2 = d * d;
    const float c = 1.0f - 0.5f * d2, sn = d * (1.0f - d2 * (1.0f / 6.0f));
    return make_float2(t.x * c - t.y * sn, t.x * sn + t.y * c);
}
__device__ __forceinline__ double2 cis_turn(uint64_t u, const double2 *tab) {
    const double2 t = tab[u >> 56];
    const double d = (double)(u & 0xffffffffffffffull) * 3.4061215800865545e-19;  // 2 pi / 2^64
    const double d2 = d * d;
    const double c = 1.0 - d2 * (0.5 - d2 * (1.0 / 24 - d2 * (1.0 / 720 - d2 * (1.0 / 40320))));
    const double sn = d * (1.0 - d2 * (1.0 / 6 - d2 * (1.0 / 120 - d2 * (1.0 / 5040 - d2 * (1.0 / 362880)))));
    return make_double2(t.x * c - t.y * sn, t.x * sn + t.y * c);
}
__device__ __forceinline__ void cis_table_entry(int k, float2 *tab) {
    float s, c;
    sincospif((float)k / 128.0f, &s, &c);
    tab[k] = make_float2(c, s);
}
__device__ __forceinline__ void cis_table_entry(int k, double2 *tab) {
    double s, c;
    sincospi((double)k / 128.0, &s, &c);
    tab[k] = make_double2(c, s);
}
// complex product on registers (packed FMUL2 + FFMA2 for float)
__device__ __forceinline__ float2 cmulp(float2 x, float2 y) {
    return __ffma2_rn(make_float2(-x.y, x.y), make_float2(y.y, y.x), __fmul2_rn(make_float2(x.x, x.x), y));
}
__device__ __forceinline__ double2 cmulp(double2 x, double2 y) { return cmul(x, y); }

template <typename Real> struct DAcc {
    typedef decltype(DTerm<Real>::ang) U;
};

// sum of a kop's terms [i0, i1) with the given target (0xff = th, else register bit)
template <typename Real>
__device__ __forceinline__ typename DAcc<Real>::U dblk_sum(const DTerm<Real> *tm, int i0, int i1, uint32_t target,
                                                           uint32_t tix, uint64_t basefull) {
    typedef typename DAcc<Real>::U U;
    U acc = 0;
    for (int i = i0; i < i1; i++) {
        const DTerm<Real> t = tm[i];
        const uint32_t va = t.a.kind == BK_TIX ? ((tix >> t.a.idx) & 1u)
                            : t.a.kind == BK_BASE ? (uint32_t)((basefull >> t.a.idx) & 1ull) : 1u;
        const uint32_t vb = t.b.kind == BK_TIX ? ((tix >> t.b.idx) & 1u)
                            : t.b.kind == BK_BASE ? (uint32_t)((basefull >> t.b.idx) & 1ull) : 1u;
        const bool hit = t.a.kind == BK_REG ? (t.a.idx == target && vb) : (target == 0xffu && va && vb);
        acc += hit ? t.ang : (U)0;
    }
    return acc;
}

// The applying kop of a diagonal-block run (tqd_internal.h DTerm): th / al[b] =
// precomputed C rows (per thread) + U values (per tile) + the M terms of the run's
// kops; then exp(i Phi(r)) = table[r] e^{i th} prod_{b in r} e^{i al_b}.
template <typename Real, bool BWD>
__device__ __forceinline__ void run_dblk(const uint4 h, const KOp<Real> &op, typename CT<Real>::C *a,
                                         typename CT<Real>::C *l, uint32_t tix, uint64_t basefull,
                                         const DevStage &S, const typename DAcc<Real>::U *uacc,
                                         const typename CT<Real>::C *ctb) {
    typedef typename CT<Real>::C C;
    typedef typename DAcc<Real>::U U;
    // this thread's C rows: dynamic shared memory after the sweep kernel's other
    // regions (sweep_smem_bytes order); recomputed here so that the op loop carries
    // no extra pointer (S, uacc and ctb are static shared arrays)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const U *ctab;
    {
        const size_t T = blockDim.x;
        const size_t off = (size_t)(BWD ? 2 : 1) * ((size_t)1 << S.k) * sizeof(C) + (size_t)S.n_ops * sizeof(KOp<Real>) +
                           (BWD ? (size_t)S.n_slots * T * sizeof(Real) : 0) + (size_t)(3 * S.nseg - 2) * T * sizeof(uint32_t) +
                           2 * T * sizeof(uint64_t);
        ctab = reinterpret_cast<const U *>(smem_raw + off) + threadIdx.x;
    }
    const int first = (int)((h.x >> 24) & 0xffu);  // data kops before this one
    const uint32_t xm = h.y & 0xffu;
    const uint32_t coff = (h.y >> 8) & 0xffu, uoff = (h.y >> 16) & 0xffu;
    U th = 0, al[SWEEP_R];
#pragma unroll
    for (int b = 0; b < SWEEP_R; b++) al[b] = 0;
    if (coff != 0xffu) {
        int j = (int)coff;
        th += ctab[(j++) * blockDim.x];
#pragma unroll
        for (int b = 0; b < SWEEP_R; b++)
            if ((xm >> b) & 1u) al[b] += ctab[(j++) * blockDim.x];
    }
    if (uoff != 0xffu) {
        int j = (int)uoff;
        th += uacc[j++];
#pragma unroll
        for (int b = 0; b < SWEEP_R; b++)
            if ((xm >> b) & 1u) al[b] += uacc[j++];
    }
    for (int q = first; q >= 0; q--) {  // M terms (lane / warp x base) of every kop of the run
        const KOp<Real> &kq = (&op)[-q];
        const uint32_t hz = reinterpret_cast<const uint4 *>(&kq)->z;
        const int i0 = (int)((hz & 0xffu) + ((hz >> 8) & 0xffu)), i1 = i0 + (int)((hz >> 16) & 0xffu);
        if (i1 == i0) continue;
        const DTerm<Real> *tm = reinterpret_cast<const DTerm<Real> *>(kq.g);
        // one pass over the terms: a term feeds th (no register bit) or al[its register
        // bit] (terms moved here when the C / U budgets ran out)
        for (int i = i0; i < i1; i++) {
            const DTerm<Real> t = tm[i];
            const uint32_t va = t.a.kind == BK_TIX ? ((tix >> t.a.idx) & 1u)
                                : t.a.kind == BK_BASE ? (uint32_t)((basefull >> t.a.idx) & 1ull) : 1u;
            const uint32_t vb = t.b.kind == BK_TIX ? ((tix >> t.b.idx) & 1u)
                                : t.b.kind == BK_BASE ? (uint32_t)((basefull >> t.b.idx) & 1ull) : 1u;
            const typename DAcc<Real>::U v = vb ? t.ang : (typename DAcc<Real>::U)0;
            if (t.a.kind != BK_REG) {
                th += va ? v : (typename DAcc<Real>::U)0;
            } else {
#pragma unroll
                for (int b = 0; b < SWEEP_R; b++) al[b] += (t.a.idx == b) ? v : (typename DAcc<Real>::U)0;
            }
        }
    }
    // in place, no per-amplitude phase array: table[r] e^{i th} first, then
    // e^{i al_b} on the amplitudes with register bit b set
    const C w0 = cis_turn(th, ctb);
    if ((h.x >> 16) & 2u) {  // identity table
        if (th != 0) {  // (a run flushed for one register bit has no th terms: th == 0 exactly)
#pragma unroll
            for (int r = 0; r < NR; r++) {
                a[r] = cmulp(w0, a[r]);
                if (BWD) l[r] = cmulp(w0, l[r]);
            }
        }
    } else {
#pragma unroll
        for (int r = 0; r < NR; r++) {
            const C ph = cmul_e(op.m + 4 * r, w0);
            a[r] = cmulp(ph, a[r]);
            if (BWD) l[r] = cmulp(ph, l[r]);
        }
    }
#pragma unroll
    for (int b = 0; b < SWEEP_R; b++) {
        if (!((xm >> b) & 1u)) continue;
        const C u = cis_turn(al[b], ctb);
#pragma unroll
        for (int r = 0; r < NR; r++) {
            if (!(r & (1 << b))) continue;
            a[r] = cmulp(u, a[r]);
            if (BWD) l[r] = cmulp(u, l[r]);
        }
    }
}

// ---- one op, in place on psi (and lambda in the adjoint) ----------------------
// h = the op's 16-byte dispatch header (already in registers: prefetched while
// the previous op ran), op = the full op in shared memory (coefficients).
template <typename Real, bool BWD, bool DB>
__device__ __forceinline__ void run_kop(const uint4 h, const KOp<Real> &op, typename CT<Real>::C *a,
                                        typename CT<Real>::C *l, uint32_t tix, uint64_t basefull, Real *tt,
                                        const DevStage &S, const typename DAcc<Real>::U *uacc,
                                        const typename CT<Real>::C *ctb) {
    typedef typename CT<Real>::C C;
    auto bitval = [&](uint32_t kind, uint32_t idx) -> int {
        return kind == BK_TIX ? (int)((tix >> idx) & 1u) : (int)((basefull >> idx) & 1ull);
    };
    const int code = h.x & 0xff;
    const uint32_t gm = (h.y >> 8) & 0xff;  // layer fast path (grad_y_layer / grad_z_layer in the switch)
    if (BWD) {
        const int ngen = (h.x >> 8) & 0xff;
        if (ngen && !gm) {
            // general path: gradients on the post-gate states (R7): g_p += 2 Re <lam|G_p|psi>
            const uint32_t gbits = h.y & 0xff;
            const uint32_t gkinds = h.w & 0xffff;
            for (int gi = 0; gi < ngen; gi++) {
                Real part = 0;
                if (code == KC_PHASE) {
                    part = grad_z_const<C, Real>(a, l, bitval((h.z) & 0xff, (h.z >> 8) & 0xff));
                } else {
                    const int gk = (gkinds >> (4 * gi)) & 15;
                    const Real *g = op.g[gi];
                    dispatch4((gbits >> (2 * gi)) & 3,
                              [&](auto tb) { part = grad_bit<decltype(tb)::value, C, Real>(a, l, gk, g); });
                }
                tt[op.soff[gi]] += part;
            }
        }
    }
    const uint32_t creg = (h.x >> 16) & 0xff;
    const uint32_t ck = (h.y >> 16) & 0xff, ci = h.y >> 24;
    const bool on = ck == BK_NONE ? true : bitval(ck, ci) != 0;
    const int cm = creg != 0xff ? (1 << creg) : 0;
    switch (code) {
    case 1: if (BWD && gm) grad_y_layer<1, C, Real>(a, l, gm, op.soff, tt); layer_real<1, C, Real>(a, op.m); if (BWD) layer_real<1, C, Real>(l, op.m); break;
    case 2: if (BWD && gm) grad_y_layer<2, C, Real>(a, l, gm, op.soff, tt); layer_real<2, C, Real>(a, op.m); if (BWD) layer_real<2, C, Real>(l, op.m); break;
    case 3: if (BWD && gm) grad_y_layer<3, C, Real>(a, l, gm, op.soff, tt); layer_real<3, C, Real>(a, op.m); if (BWD) layer_real<3, C, Real>(l, op.m); break;
    case 4: if (BWD && gm) grad_y_layer<4, C, Real>(a, l, gm, op.soff, tt); layer_real<4, C, Real>(a, op.m); if (BWD) layer_real<4, C, Real>(l, op.m); break;
    case 5: if (BWD && gm) grad_y_layer<5, C, Real>(a, l, gm, op.soff, tt); layer_real<5, C, Real>(a, op.m); if (BWD) layer_real<5, C, Real>(l, op.m); break;
    case 6: if (BWD && gm) grad_y_layer<6, C, Real>(a, l, gm, op.soff, tt); layer_real<6, C, Real>(a, op.m); if (BWD) layer_real<6, C, Real>(l, op.m); break;
    case 7: if (BWD && gm) grad_y_layer<7, C, Real>(a, l, gm, op.soff, tt); layer_real<7, C, Real>(a, op.m); if (BWD) layer_real<7, C, Real>(l, op.m); break;
    case 8: if (BWD && gm) grad_y_layer<8, C, Real>(a, l, gm, op.soff, tt); layer_real<8, C, Real>(a, op.m); if (BWD) layer_real<8, C, Real>(l, op.m); break;
    case 9: if (BWD && gm) grad_y_layer<9, C, Real>(a, l, gm, op.soff, tt); layer_real<9, C, Real>(a, op.m); if (BWD) layer_real<9, C, Real>(l, op.m); break;
    case 10: if (BWD && gm) grad_y_layer<10, C, Real>(a, l, gm, op.soff, tt); layer_real<10, C, Real>(a, op.m); if (BWD) layer_real<10, C, Real>(l, op.m); break;
    case 11: if (BWD && gm) grad_y_layer<11, C, Real>(a, l, gm, op.soff, tt); layer_real<11, C, Real>(a, op.m); if (BWD) layer_real<11, C, Real>(l, op.m); break;
    case 12: if (BWD && gm) grad_y_layer<12, C, Real>(a, l, gm, op.soff, tt); layer_real<12, C, Real>(a, op.m); if (BWD) layer_real<12, C, Real>(l, op.m); break;
    case 13: if (BWD && gm) grad_y_layer<13, C, Real>(a, l, gm, op.soff, tt); layer_real<13, C, Real>(a, op.m); if (BWD) layer_real<13, C, Real>(l, op.m); break;
    case 14: if (BWD && gm) grad_y_layer<14, C, Real>(a, l, gm, op.soff, tt); layer_real<14, C, Real>(a, op.m); if (BWD) layer_real<14, C, Real>(l, op.m); break;
    case 15: if (BWD && gm) grad_y_layer<15, C, Real>(a, l, gm, op.soff, tt); layer_real<15, C, Real>(a, op.m); if (BWD) layer_real<15, C, Real>(l, op.m); break;
    case 16: layer_gen<1, C, Real>(a, op.m); if (BWD) layer_gen<1, C, Real>(l, op.m); break;
    case 17: layer_gen<2, C, Real>(a, op.m); if (BWD) layer_gen<2, C, Real>(l, op.m); break;
    case 18: layer_gen<3, C, Real>(a, op.m); if (BWD) layer_gen<3, C, Real>(l, op.m); break;
    case 19: layer_gen<4, C, Real>(a, op.m); if (BWD) layer_gen<4, C, Real>(l, op.m); break;
    case 20: layer_gen<5, C, Real>(a, op.m); if (BWD) layer_gen<5, C, Real>(l, op.m); break;
    case 21: layer_gen<6, C, Real>(a, op.m); if (BWD) layer_gen<6, C, Real>(l, op.m); break;
    case 22: layer_gen<7, C, Real>(a, op.m); if (BWD) layer_gen<7, C, Real>(l, op.m); break;
    case 23: layer_gen<8, C, Real>(a, op.m); if (BWD) layer_gen<8, C, Real>(l, op.m); break;
    case 24: layer_gen<9, C, Real>(a, op.m); if (BWD) layer_gen<9, C, Real>(l, op.m); break;
    case 25: layer_gen<10, C, Real>(a, op.m); if (BWD) layer_gen<10, C, Real>(l, op.m); break;
    case 26: layer_gen<11, C, Real>(a, op.m); if (BWD) layer_gen<11, C, Real>(l, op.m); break;
    case 27: layer_gen<12, C, Real>(a, op.m); if (BWD) layer_gen<12, C, Real>(l, op.m); break;
    case 28: layer_gen<13, C, Real>(a, op.m); if (BWD) layer_gen<13, C, Real>(l, op.m); break;
    case 29: layer_gen<14, C, Real>(a, op.m); if (BWD) layer_gen<14, C, Real>(l, op.m); break;
    case 30: layer_gen<15, C, Real>(a, op.m); if (BWD) layer_gen<15, C, Real>(l, op.m); break;
    case KC_DIAG: if (BWD && gm) grad_z_layer<C, Real>(a, l, gm, op.soff, tt); layer_diag<C, Real>(a, op.m); if (BWD) layer_diag<C, Real>(l, op.m); break;
    case 32: op_cu<0, C, Real>(a, op.m, cm, on); if (BWD) op_cu<0, C, Real>(l, op.m, cm, on); break;
    case 33: op_cu<1, C, Real>(a, op.m, cm, on); if (BWD) op_cu<1, C, Real>(l, op.m, cm, on); break;
    case 34: op_cu<2, C, Real>(a, op.m, cm, on); if (BWD) op_cu<2, C, Real>(l, op.m, cm, on); break;
    case 35: op_cu<3, C, Real>(a, op.m, cm, on); if (BWD) op_cu<3, C, Real>(l, op.m, cm, on); break;
    case 38: op_u2<0, 1, C, Real>(a, op.m); if (BWD) op_u2<0, 1, C, Real>(l, op.m); break;
    case 39: op_u2<0, 2, C, Real>(a, op.m); if (BWD) op_u2<0, 2, C, Real>(l, op.m); break;
    case 40: op_u2<0, 3, C, Real>(a, op.m); if (BWD) op_u2<0, 3, C, Real>(l, op.m); break;
    case 41: op_u2<1, 0, C, Real>(a, op.m); if (BWD) op_u2<1, 0, C, Real>(l, op.m); break;
    case 42: op_u2<1, 2, C, Real>(a, op.m); if (BWD) op_u2<1, 2, C, Real>(l, op.m); break;
    case 43: op_u2<1, 3, C, Real>(a, op.m); if (BWD) op_u2<1, 3, C, Real>(l, op.m); break;
    case 44: op_u2<2, 0, C, Real>(a, op.m); if (BWD) op_u2<2, 0, C, Real>(l, op.m); break;
    case 45: op_u2<2, 1, C, Real>(a, op.m); if (BWD) op_u2<2, 1, C, Real>(l, op.m); break;
    case 46: op_u2<2, 3, C, Real>(a, op.m); if (BWD) op_u2<2, 3, C, Real>(l, op.m); break;
    case 47: op_u2<3, 0, C, Real>(a, op.m); if (BWD) op_u2<3, 0, C, Real>(l, op.m); break;
    case 48: op_u2<3, 1, C, Real>(a, op.m); if (BWD) op_u2<3, 1, C, Real>(l, op.m); break;
    case 49: op_u2<3, 2, C, Real>(a, op.m); if (BWD) op_u2<3, 2, C, Real>(l, op.m); break;
    case KC_PHASE: {
        const Real *d = op.m + 4 * bitval(h.z & 0xff, (h.z >> 8) & 0xff);
#pragma unroll
        for (int r = 0; r < NR; r++) a[r] = cmul_e(d, a[r]);
        if (BWD) {
#pragma unroll
            for (int r = 0; r < NR; r++) l[r] = cmul_e(d, l[r]);
        }
        break;
    }
    case KC_DBLK:
        if constexpr (DB) run_dblk<Real, BWD>(h, op, a, l, tix, basefull, S, uacc, ctb);
        break;
    case KC_D2: {
        const uint32_t k0 = h.z & 0xff, i0 = (h.z >> 8) & 0xff, k1 = (h.z >> 16) & 0xff, i1 = h.z >> 24;
        const int m0 = k0 == BK_REG ? (1 << i0) : 0;
        const int m1 = k1 == BK_REG ? (1 << i1) : 0;
        const int v0 = m0 ? 0 : bitval(k0, i0);
        const int v1 = m1 ? 0 : bitval(k1, i1);
        op_d2<C, Real>(a, op.m, m0, v0, m1, v1);
        if (BWD) op_d2<C, Real>(l, op.m, m0, v0, m1, v1);
        break;
    }
    default: break;
    }
}

// asynchronous global -> shared 16-byte copies (the next tile's staging, TQD_SWEEP_STAGE:
// an experiment, off: measured slower, profiles/r02_experiments.md)
#ifndef TQD_SWEEP_STAGE
#define TQD_SWEEP_STAGE 0
#endif
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// evict-first global accesses of the streamed shards (cache-streaming hints)
__device__ __forceinline__ float2 ldcs_c(const float2 *p) { return __ldcs(p); }
__device__ __forceinline__ double2 ldcs_c(const double2 *p) { return __ldcs(p); }
__device__ __forceinline__ void stcs_c(float2 *p, float2 v) { __stcs(p, v); }
__device__ __forceinline__ void stcs_c(double2 *p, double2 v) { __stcs(p, v); }

// ---- the fused sweep kernel: one CTA = 32 * 2^W threads, persistent over tiles.
// DB: the stage has diagonal-block runs (a separate instantiation keeps their
// shared arrays, precomputation and code out of the stages that have none)
template <typename Real, bool BWD, bool DB>
__global__ void __launch_bounds__(SWEEP_THREADS, sizeof(Real) == 4 ? (BWD ? TQD_LB_MINB_F32_BWD : TQD_LB_MINB_F32_FWD) : 1) sweep_kernel(const DevStage *__restrict__ stg, const KOp<Real> *__restrict__ ops,
                                                    const int32_t *__restrict__ slot_param,
                                                    typename CT<Real>::C *__restrict__ psi,
                                                    typename CT<Real>::C *__restrict__ lam,
                                                    double *__restrict__ grad, uint64_t rank_hi,
                                                    const __grid_constant__ ScatterInfo sc) {
    typedef typename CT<Real>::C C;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ DevStage S;
    __shared__ uint64_t s_ldc[SWEEP_R], s_stc[SWEEP_R];  // element offsets of the register bits (load / store)
    __shared__ uint32_t s_wc[MAXSEG][SWEEP_R], s_rc[MAXSEG][SWEEP_R];  // byte address vectors of the register bits

    {
        const uint32_t *src = reinterpret_cast<const uint32_t *>(stg);
        uint32_t *dst = reinterpret_cast<uint32_t *>(&S);
        for (int i = threadIdx.x; i < (int)(sizeof(DevStage) / 4); i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    const int k = S.k;
    const int W = S.W;
    const int nseg = S.nseg;
    // batch of states: CTA blockIdx.x serves state blockIdx.x % B (grid is a multiple of
    // B); each state has its own copy of the op stream and gradient-slot table
    const int B = S.batch > 0 ? S.batch : 1;
    const int bidx = (int)(blockIdx.x % (unsigned)B);
    const int gsz = (int)(gridDim.x / (unsigned)B);  // CTAs per state
    const int gid = (int)(blockIdx.x / (unsigned)B);
    const uint64_t bst = (uint64_t)S.n_tiles << k;     // amplitudes per state shard
    psi += bidx * bst;
    if (BWD) lam += bidx * bst;
    // shared memory: [exchange psi (2^k)] [exchange lambda (2^k, adjoint)] [kernel ops]
    C *sm_a = reinterpret_cast<C *>(smem_raw);
    C *sm_l = sm_a + ((size_t)1 << k);
    KOp<Real> *s_ops = reinterpret_cast<KOp<Real> *>(smem_raw + (size_t)(BWD ? 2 : 1) * ((size_t)1 << k) * sizeof(C));
    // adjoint: per-thread gradient accumulators [slot][thread] (no per-tile reductions)
    Real *tacc = reinterpret_cast<Real *>(s_ops + S.n_ops);
    // per-thread constants, computed once per kernel: tix[seg], write / read base of each exchange
    uint32_t *s_tix = reinterpret_cast<uint32_t *>(tacc + (BWD ? S.n_slots * blockDim.x : 0));
    uint32_t *s_tw = s_tix + nseg * blockDim.x;
    uint32_t *s_tr = s_tw + (nseg - 1) * blockDim.x;
    // per-thread L2-prefetch offsets (element offsets within a tile, up to 2 per thread)
    uint64_t *s_pf = reinterpret_cast<uint64_t *>(s_tr + (nseg - 1) * blockDim.x);  // 8 B aligned (threads * 4 B is)
    // diagonal blocks: per-thread C rows [row][thread], per-tile U values [2][DBLK_UCAP]
    typedef typename DAcc<Real>::U DU;
    DU *s_ctab = reinterpret_cast<DU *>(s_pf + 2 * blockDim.x);
    __shared__ DU s_uacc[DB ? DBLK_UCAP : 1];  // this tile's U values
    __shared__ uint8_t s_uk[DB ? DBLK_UCAP : 1], s_ut[DB ? DBLK_UCAP : 1];  // U value -> kop index, target (0xff = th)
    __shared__ C s_cis[DB ? 256 : 1];                                       // e^{i 2 pi k / 256} for cis_turn
    {
        const int4 *src = reinterpret_cast<const int4 *>(ops + S.op_base + (size_t)bidx * S.n_ops);
        int4 *dst = reinterpret_cast<int4 *>(s_ops);
        const int n16 = (int)(S.n_ops * sizeof(KOp<Real>) / 16);
        for (int i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = src[i];
        if (threadIdx.x < SWEEP_R) {
            const int i = threadIdx.x;
            s_ldc[i] = 1ull << S.ld_phys[S.lay[0].reg[i]];
            s_stc[i] = 1ull << S.st_phys[S.lay[nseg - 1].reg[i]];
        }
        for (int i = threadIdx.x; i < (nseg - 1) * SWEEP_R; i += blockDim.x) {
            const int x = i / SWEEP_R, b = i % SWEEP_R;
            s_wc[x][b] = S.wcol[x][S.lay[x].reg[b]] * (uint32_t)sizeof(C);
            s_rc[x][b] = S.rcol[x][S.lay[x + 1].reg[b]] * (uint32_t)sizeof(C);
        }
        if (BWD)
            for (int i = threadIdx.x; i < S.n_slots * (int)blockDim.x; i += blockDim.x) tacc[i] = 0;
    }
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;

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
    auto thr_cols = [&](const uint32_t *cols, const DevLayout &L) -> uint32_t {
        uint32_t t = 0;
#pragma unroll
        for (int i = 0; i < LANE_BITS; i++)
            if ((lane >> i) & 1) t ^= cols[L.lane[i]];
        for (int w = 0; w < W; w++)
            if ((warp >> w) & 1) t ^= cols[L.warp[w]];
        return t;
    };
    // diagonal blocks: C sums once per kernel (lane / warp bits are fixed per thread
    // and segment) into this thread's rows, the per-tile U work list (value -> applying
    // kop, target) once per kernel
    if constexpr (DB)
        for (int kk = threadIdx.x; kk < 256; kk += blockDim.x) cis_table_entry(kk, s_cis);
    if (DB && (S.n_cvals || S.n_uvals)) {
        for (int j = 0; j < S.n_cvals; j++) s_ctab[j * blockDim.x + threadIdx.x] = 0;
        for (int s = 0; s < nseg; s++) {
            const uint32_t tx = thr_tix(S.lay[s]);
            for (int oi = S.seg_begin[s]; oi < S.seg_begin[s + 1]; oi++) {
                const uint4 h = *reinterpret_cast<const uint4 *>(&s_ops[oi]);
                const uint32_t code = h.x & 0xffu;
                if (code != KC_DBLK && code != KC_DDATA) continue;
                const int nC = (int)(h.z & 0xffu);
                const uint32_t xm = h.y & 0xffu, coff = (h.y >> 8) & 0xffu, uoff = (h.y >> 16) & 0xffu;
                const DTerm<Real> *tm = reinterpret_cast<const DTerm<Real> *>(s_ops[oi].g);
                if (nC && coff != 0xffu) {
                    int j = (int)coff;
                    s_ctab[(j++) * blockDim.x + threadIdx.x] += dblk_sum<Real>(tm, 0, nC, 0xffu, tx, 0);
                    for (int b = 0; b < SWEEP_R; b++)
                        if ((xm >> b) & 1u) s_ctab[(j++) * blockDim.x + threadIdx.x] += dblk_sum<Real>(tm, 0, nC, (uint32_t)b, tx, 0);
                }
                if (code == KC_DBLK && uoff != 0xffu && threadIdx.x == 0) {
                    int j = (int)uoff;
                    s_uk[j] = (uint8_t)oi;
                    s_ut[j++] = 0xffu;
                    for (int b = 0; b < SWEEP_R; b++)
                        if ((xm >> b) & 1u) { s_uk[j] = (uint8_t)oi; s_ut[j++] = (uint8_t)b; }
                }
            }
        }
    }
    const uint64_t ld_thr = thr_phys_off(S.lay[0], S.ld_phys);
    const uint64_t st_thr = thr_phys_off(S.lay[nseg - 1], S.st_phys);
    {
        const int T = blockDim.x, tid = threadIdx.x;
        for (int s = 0; s < nseg; s++) s_tix[s * T + tid] = thr_tix(S.lay[s]);
        for (int x = 0; x + 1 < nseg; x++) {
            s_tw[x * T + tid] = (thr_cols(S.wcol[x], S.lay[x]) ^ S.wcst[x]) * (uint32_t)sizeof(C);
            s_tr[x * T + tid] = (thr_cols(S.rcol[x], S.lay[x + 1]) ^ S.rcst[x]) * (uint32_t)sizeof(C);
        }
    }
    // L2 prefetch of the NEXT tile (issued while this one computes): the tile's
    // load set is 2^(5-C) x 16 lines of 128 B per warp (C = the pinned low bits that
    // fill a line); lane j of the warp covers line i*32 + j with one prefetch per i
    int n_pf = 0;
    {
        const DevLayout &L = S.lay[0];
        int C = 0;
        while (C < LANE_BITS && S.ld_phys[L.lane[C]] == C) C++;
        const int lbits = LANE_BITS - C;                // lane bits outside the line
        const int nlines = 16 << lbits;                 // lines per warp load set
        n_pf = nlines >= 64 ? 2 : 1;
        uint64_t wpart = 0;
        for (int w = 0; w < W; w++)
            if ((warp >> w) & 1) wpart |= 1ull << S.ld_phys[L.warp[w]];
        for (int i = 0; i < n_pf; i++) {
            const int idx = (i * 32 + lane) % nlines;
            uint64_t off = wpart;
            for (int t = 0; t < lbits; t++)
                if ((idx >> t) & 1) off |= 1ull << S.ld_phys[L.lane[C + t]];
            const int r = (idx >> lbits) & (NR - 1);
            for (int b = 0; b < SWEEP_R; b++)
                if ((r >> b) & 1) off |= 1ull << S.ld_phys[L.reg[b]];
            s_pf[i * blockDim.x + threadIdx.x] = off;
        }
    }
    __syncthreads();

    // tile index -> physical base: deposit into the non-tile positions once, then
    // step by a masked add (carries propagate only through non-tile positions)
    auto deposit = [&](uint64_t v) {
        for (int i = 0; i < k; i++) {
            const int p = S.tile_sorted[i];
            v = ((v >> p) << (p + 1)) | (v & ((1ull << p) - 1));
        }
        return v;
    };
    const uint64_t tmask = deposit(~0ull) & (S.n_tiles > 1 ? ~0ull : 0ull);
    const uint64_t step = deposit((uint64_t)gsz);
    uint64_t base = deposit((uint64_t)gid);
#if TQD_SWEEP_STAGE
    // Staged tile loads: the next tile's psi (and lambda) are copied into the exchange
    // buffers by cp.async while this tile's last segment computes and stores (the
    // buffers are idle after the last exchange); the tile starts with shared-memory
    // reads instead of exposed global-load latency.  Staging layout: tile-local index
    // order (16-byte chunk ch = tile bits [cb, k) of its first amplitude); the thread
    // index covers the low chunk bits (consecutive threads: consecutive 16 bytes of a
    // 128-byte run), passes j the high ones.
    constexpr int cb = sizeof(C) == 8 ? 1 : 0;  // tile bits inside one 16-byte chunk
    const bool stage_ok = cb == 0 || S.ld_phys[0] == 0;
    const int lgT = __ffs((int)blockDim.x) - 1;
    const int tb = min(k - cb, lgT), jb = k - cb - tb;
    const bool st_act = (threadIdx.x >> tb) == 0u;
    uint64_t stg_thr = 0;
    for (int i = 0; i < tb; i++)
        if ((threadIdx.x >> i) & 1u) stg_thr |= 1ull << S.ld_phys[cb + i];
    auto stage_issue = [&](uint64_t nb) {
        if (st_act) {
            for (int j = 0; j < (1 << jb); j++) {
                uint64_t off = nb | stg_thr;
                for (int i = 0; i < jb; i++)
                    if ((j >> i) & 1) off |= 1ull << S.ld_phys[cb + tb + i];
                const uint32_t ch = threadIdx.x | ((uint32_t)j << tb);
                cp_async16(reinterpret_cast<char *>(sm_a) + (size_t)ch * 16, psi + off);
                if (BWD) cp_async16(reinterpret_cast<char *>(sm_l) + (size_t)ch * 16, lam + off);
            }
        }
        cp_async_commit();
    };
    if (stage_ok && gid < S.n_tiles) stage_issue(base);
#endif
    for (int64_t tile = gid; tile < S.n_tiles; tile += gsz, base = ((base | ~tmask) + step) & tmask) {
        const uint64_t basefull = base | rank_hi;
        const bool has_next = tile + gsz < S.n_tiles;
        const uint64_t next_base = ((base | ~tmask) + step) & tmask;

        C a[NR];
        C l[BWD ? NR : 1];
#if TQD_SWEEP_STAGE
        if (stage_ok) {
            cp_async_wait_all();
            __syncthreads();
            // layout 0 from the staged tile (tile-local index order)
            uint32_t o[NR], c[SWEEP_R];
#pragma unroll
            for (int i = 0; i < SWEEP_R; i++) c[i] = (1u << S.lay[0].reg[i]) * (uint32_t)sizeof(C);
            o[0] = s_tix[threadIdx.x] * (uint32_t)sizeof(C);
#pragma unroll
            for (int r = 1; r < NR; r++) o[r] = o[r & (r - 1)] ^ c[ctz4(r)];
#pragma unroll
            for (int r = 0; r < NR; r++) {
                a[r] = *reinterpret_cast<const C *>(reinterpret_cast<const char *>(sm_a) + o[r]);
                if (BWD) l[r] = *reinterpret_cast<const C *>(reinterpret_cast<const char *>(sm_l) + o[r]);
            }
            __syncthreads();  // every warp holds its amplitudes: the buffers are free
            if (nseg == 1 && has_next) stage_issue(next_base);
        } else
#endif
        {
            // Gray-code walk over the register offsets: one 64-bit add per address
            const uint64_t b0 = base | ld_thr;
            uint64_t o[NR], c[SWEEP_R];
#pragma unroll
            for (int i = 0; i < SWEEP_R; i++) c[i] = s_ldc[i];
            o[0] = b0;
#pragma unroll
            for (int r = 1; r < NR; r++) o[r] = o[r & (r - 1)] + c[ctz4(r)];
#pragma unroll
            for (int r = 0; r < NR; r++) {
                // streaming: read once per sweep, do not keep in L2 (the next tiles'
                // prefetched lines must survive there)
                a[r] = ldcs_c(psi + o[r]);
                if (BWD) l[r] = ldcs_c(lam + o[r]);
            }
        }
        // diagonal blocks: this tile's U sums (base bits only), between two barriers
        if (DB && S.n_uvals) {
            __syncthreads();  // every thread is done with the previous tile's values
            // one warp per value, one lane per term of each kop of the run (nU <= 16),
            // exact wrapping integer sums by shuffle
            const int nw = (int)(blockDim.x >> 5);
            for (int v = warp; v < S.n_uvals; v += nw) {
                const int oi = s_uk[v];
                const uint32_t tgt = s_ut[v];
                const int first = (int)((reinterpret_cast<const uint4 *>(&s_ops[oi])->x >> 24) & 0xffu);
                DU sum = 0;
                for (int q = oi - first; q <= oi; q++) {
                    const uint32_t hz = reinterpret_cast<const uint4 *>(&s_ops[q])->z;
                    const int nC = (int)(hz & 0xffu), nU = (int)((hz >> 8) & 0xffu);
                    if (lane < nU)
                        sum += dblk_sum<Real>(reinterpret_cast<const DTerm<Real> *>(s_ops[q].g), nC + lane, nC + lane + 1,
                                              tgt, 0, basefull);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
                if (lane == 0) s_uacc[v] = sum;
            }
            __syncthreads();
        }
        if (has_next) {
            const uint64_t nb = next_base;
            for (int i = 0; i < n_pf; i++) {
                const uint64_t e = nb + s_pf[i * blockDim.x + threadIdx.x];
                asm volatile("prefetch.global.L2 [%0];" ::"l"(psi + e));
                if (BWD) asm volatile("prefetch.global.L2 [%0];" ::"l"(lam + e));
            }
        }

        for (int s = 0; s < nseg; s++) {
            if (s > 0) {
                // layout change through shared memory; the permutation gates of the
                // previous segment (CNOT / X: GF(2)-affine index maps) ride along
                const int x = s - 1;
                uint32_t aff = 0;
                for (int i = 0; i < S.naff[x]; i++)
                    if ((basefull >> S.aff_pos[x][i]) & 1ull) aff ^= S.aff_vec[x][i];
                aff *= (uint32_t)sizeof(C);
                const uint32_t tw = s_tw[x * blockDim.x + threadIdx.x] ^ (S.aff_read[x] ? 0u : aff);
                const uint32_t tr = s_tr[x * blockDim.x + threadIdx.x] ^ (S.aff_read[x] ? aff : 0u);
                {
                    // Gray-code walk: one XOR per register address
                    uint32_t c[SWEEP_R], o[NR];
#pragma unroll
                    for (int b = 0; b < SWEEP_R; b++) c[b] = s_wc[x][b];
                    o[0] = tw;
#pragma unroll
                    for (int r = 1; r < NR; r++) o[r] = o[r & (r - 1)] ^ c[ctz4(r)];
#pragma unroll
                    for (int r = 0; r < NR; r++) {
                        *reinterpret_cast<C *>(reinterpret_cast<char *>(sm_a) + o[r]) = a[r];
                        if (BWD) *reinterpret_cast<C *>(reinterpret_cast<char *>(sm_l) + o[r]) = l[r];
                    }
                }
                {
                    // write -> read: only the warps sharing the kept warp-index bits exchange data
                    const uint32_t um = S.xsync[x] & 0x0fu, full = (1u << W) - 1u;
                    if (um == full) {
                        __syncwarp();
                    } else if (um == 0) {
                        __syncthreads();
                    } else {
                        const uint32_t nthr = 32u << (W - __popc(um));
                        asm volatile("bar.sync %0, %1;" ::"r"(1u + ((uint32_t)warp & um)), "r"(nthr) : "memory");
                    }
                }
                {
                    uint32_t c[SWEEP_R], o[NR];
#pragma unroll
                    for (int b = 0; b < SWEEP_R; b++) c[b] = s_rc[x][b];
                    o[0] = tr;
#pragma unroll
                    for (int r = 1; r < NR; r++) o[r] = o[r & (r - 1)] ^ c[ctz4(r)];
#pragma unroll
                    for (int r = 0; r < NR; r++) {
                        a[r] = *reinterpret_cast<const C *>(reinterpret_cast<const char *>(sm_a) + o[r]);
                        if (BWD) l[r] = *reinterpret_cast<const C *>(reinterpret_cast<const char *>(sm_l) + o[r]);
                    }
#ifdef TQD_EXP_DOUBLE_EXCH
                    // timing experiment (variant builds only): a second, identity exchange
                    // (same addresses, CTA barriers) to measure the marginal exchange cost
                    __syncthreads();
#pragma unroll
                    for (int r = 0; r < NR; r++) {
                        *reinterpret_cast<C *>(reinterpret_cast<char *>(sm_a) + o[r]) = a[r];
                        if (BWD) *reinterpret_cast<C *>(reinterpret_cast<char *>(sm_l) + o[r]) = l[r];
                    }
                    __syncthreads();
#pragma unroll
                    for (int r = 0; r < NR; r++) {
                        a[r] = *reinterpret_cast<const C *>(reinterpret_cast<const char *>(sm_a) + o[r]);
                        if (BWD) l[r] = *reinterpret_cast<const C *>(reinterpret_cast<const char *>(sm_l) + o[r]);
                    }
#endif
                }
#if TQD_SWEEP_STAGE
                if (stage_ok && s == nseg - 1) {
                    // last exchange: every warp has read it; stage the next tile
                    __syncthreads();
                    if (has_next) stage_issue(next_base);
                } else
#endif
                if (S.xsync[x] & 0x80) __syncwarp();  // the next writes stay in this warp's region
                else __syncthreads();
            }
            const uint32_t tix = s_tix[s * blockDim.x + threadIdx.x];
            const int e = S.seg_begin[s + 1];
            int oi = S.seg_begin[s];
            uint4 h = oi < e ? *reinterpret_cast<const uint4 *>(&s_ops[oi]) : make_uint4(0, 0, 0, 0);
            for (; oi < e; oi++) {
                // header of the next op loads while this one runs
                const uint4 hn = oi + 1 < e ? *reinterpret_cast<const uint4 *>(&s_ops[oi + 1]) : h;
                run_kop<Real, BWD, DB>(h, s_ops[oi], a, l, tix, basefull, tacc + threadIdx.x, S, s_uacc, s_cis);
                h = hn;
            }
        }

        {
            const uint64_t b0 = base | st_thr;
            uint64_t o[NR], c[SWEEP_R];
#pragma unroll
            for (int i = 0; i < SWEEP_R; i++) c[i] = s_stc[i];
            o[0] = b0;
#pragma unroll
            for (int r = 1; r < NR; r++) o[r] = o[r & (r - 1)] + c[ctz4(r)];
            if (BWD && S.no_store == 1) {
                // last reverse sweep: psi / lambda are not needed any more
            } else if (sc.m == 0) {
                // no_store 2: the last reverse sweep before a product prefix keeps lambda only
#pragma unroll
                for (int r = 0; r < NR; r++) {
                    if (!(BWD && S.no_store == 2)) stcs_c(psi + o[r], a[r]);
                    if (BWD) stcs_c(lam + o[r], l[r]);
                }
            } else {
                // fused remap: store to the post-remap owner (peer memory) and position
                const uint64_t lmask = (1ull << sc.n_loc) - 1;
#pragma unroll
                for (int r = 0; r < NR; r++) {
                    const uint64_t P = o[r] | rank_hi;
                    uint64_t flip = 0;
                    for (int i = 0; i < sc.m; i++)
                        if (((P >> sc.gbit[i]) ^ (P >> sc.lbit[i])) & 1ull) flip |= (1ull << sc.gbit[i]) | (1ull << sc.lbit[i]);
                    const uint64_t Q = P ^ flip;
                    const int rr = (int)(Q >> sc.n_loc);
                    reinterpret_cast<C *>(sc.dst_psi[rr])[bidx * bst + (Q & lmask)] = a[r];
                    if (BWD) reinterpret_cast<C *>(sc.dst_lam[rr])[bidx * bst + (Q & lmask)] = l[r];
                }
            }
        }
    }

    if (BWD) {
        __syncthreads();
        const int nw = blockDim.x >> 5;
        for (int i = warp; i < S.n_slots; i += nw) {
            double v = 0.0;
            for (int t = lane; t < (int)blockDim.x; t += 32) v += (double)tacc[i * blockDim.x + t];
            v = warp_sum(v);
            if (lane == 0 && v != 0.0) atomicAdd(&grad[slot_param[S.slot_base + bidx * S.n_slots + i]], v);
        }
    }
}

template <typename Real, bool BWD>
static size_t sweep_smem_bytes(int k, int n_ops, int n_slots, int threads, int nseg, int n_cvals) {
    typedef typename DAcc<Real>::U DU;
    return (size_t)(BWD ? 2 : 1) * ((size_t)1 << k) * sizeof(typename CT<Real>::C) + (size_t)n_ops * sizeof(KOp<Real>) +
           (BWD ? (size_t)n_slots * threads * sizeof(Real) : 0) + (size_t)(3 * nseg - 2) * threads * sizeof(uint32_t) +
           (size_t)2 * threads * sizeof(uint64_t) + (size_t)n_cvals * threads * sizeof(DU);
}

// The dynamic shared-memory cap is a per-function attribute shared by every host
// thread: raise it ONCE per device to the opt-in maximum (a per-launch value would
// race between threads driving different states, e.g. emulated ranks), and let
// each launch / occupancy query pass its own size.
template <typename F> static cudaError_t raise_smem_cap_once(F fn, std::atomic<uint64_t> &done) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    int mx = 0;
    e = cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return e;
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, fn);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, mx - (int)fa.sharedSizeBytes);
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

template <typename Real, bool BWD, bool DB> static std::atomic<uint64_t> &sweep_cap_flag() {
    static std::atomic<uint64_t> f{0};
    return f;
}

// n_cvals < 0: the stage has no diagonal-block runs (plain instantiation)
template <typename Real, bool BWD, bool DB>
cudaError_t launch_sweep_t(const DevStage *d_stage, const void *d_ops, const int32_t *d_slots, void *psi, void *lam,
                           double *grad, uint64_t rank_hi, const ScatterInfo &sc, int k, int W, int n_ops, int n_slots,
                           int nseg, int n_cvals, int grid, cudaStream_t s) {
    typedef typename CT<Real>::C C;
    auto fn = sweep_kernel<Real, BWD, DB>;
    const size_t smem = sweep_smem_bytes<Real, BWD>(k, n_ops, n_slots, 32 << W, nseg, DB ? n_cvals : 0);
    cudaError_t e = raise_smem_cap_once(fn, sweep_cap_flag<Real, BWD, DB>());
    if (e != cudaSuccess) return e;
    fn<<<grid, 32 << W, smem, s>>>(d_stage, (const KOp<Real> *)d_ops, d_slots, (C *)psi, (C *)lam, grad, rank_hi, sc);
    return cudaGetLastError();
}

template <typename Real, bool BWD>
cudaError_t launch_sweep_impl(const DevStage *d_stage, const void *d_ops, const int32_t *d_slots, void *psi, void *lam,
                              double *grad, uint64_t rank_hi, const ScatterInfo &sc, int k, int W, int n_ops,
                              int n_slots, int nseg, int n_cvals, int grid, cudaStream_t s) {
    if (n_cvals >= 0)
        return launch_sweep_t<Real, BWD, true>(d_stage, d_ops, d_slots, psi, lam, grad, rank_hi, sc, k, W, n_ops,
                                               n_slots, nseg, n_cvals, grid, s);
    return launch_sweep_t<Real, BWD, false>(d_stage, d_ops, d_slots, psi, lam, grad, rank_hi, sc, k, W, n_ops, n_slots,
                                            nseg, 0, grid, s);
}

template <typename Real, bool BWD, bool DB>
int sweep_occupancy_t(int k, int W, int n_ops, int n_slots, int nseg, int n_cvals) {
    auto fn = sweep_kernel<Real, BWD, DB>;
    const size_t smem = sweep_smem_bytes<Real, BWD>(k, n_ops, n_slots, 32 << W, nseg, DB ? n_cvals : 0);
    if (raise_smem_cap_once(fn, sweep_cap_flag<Real, BWD, DB>()) != cudaSuccess) {
        cudaGetLastError();
        return 1;
    }
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, 32 << W, smem) != cudaSuccess) {
        cudaGetLastError();
        return 1;
    }
    return nb;
}

template <typename Real, bool BWD>
int sweep_occupancy_impl(int k, int W, int n_ops, int n_slots, int nseg, int n_cvals) {
    return n_cvals >= 0 ? sweep_occupancy_t<Real, BWD, true>(k, W, n_ops, n_slots, nseg, n_cvals)
                        : sweep_occupancy_t<Real, BWD, false>(k, W, n_ops, n_slots, nseg, 0);
}

}  // namespace tqd

#define TQD_INSTANTIATE_SWEEP(REAL, BWD, NAME)                                                                    \
    namespace tqd {                                                                                             \
    cudaError_t launch_sweep_##NAME(const DevStage *d_stage, const void *d_kops, const int32_t *d_slots, void *psi,  \
                                    void *lam, double *grad, uint64_t rank_hi, const ScatterInfo &sc, int k, int W, \
                                    int n_ops, int n_slots, int nseg, int n_cvals, int grid, cudaStream_t s) {    \
        return launch_sweep_impl<REAL, BWD>(d_stage, d_kops, d_slots, psi, lam, grad, rank_hi, sc, k, W, n_ops,    \
                                            n_slots, nseg, n_cvals, grid, s);                                   \
    }                                                                                                           \
    int sweep_occupancy_##NAME(int k, int W, int n_ops, int n_slots, int nseg, int n_cvals) {                    \
        return sweep_occupancy_impl<REAL, BWD>(k, W, n_ops, n_slots, nseg, n_cvals);                             \
    }                                                                                                           \
    }
