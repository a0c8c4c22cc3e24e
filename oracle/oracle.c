/*
 * oracle.c -- plain float64 CPU state-vector simulator (TEST ORACLE).
 *
 * TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this.  It shares nothing with
 * the CUDA path.  See oracle.h for conventions and citations.
 *
 * Everything here is the plain definition written out: one gate at a time,
 * index arithmetic over the full 2^n vector, no fusion, no blocking, no
 * reordering.  The only concession to speed is an OpenMP "parallel for" over
 * independent amplitude groups (each iteration touches a disjoint set of
 * amplitudes, so the result does not depend on the thread count; reductions
 * are the only order-dependent part and are float64).
 *
 * Pins (tests/test_oracle_*.py): brute-force kron-built unitaries (n <= 8),
 * closed forms (<Z> = cos theta, Bell, GHZ, QFT = DFT, Listing 1),
 * parameter shift vs finite differences vs both reverse modes.
 */
#include "oracle.h"

#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef double complex cplx;

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

int orc_num_params(int kind) {
    switch (kind) {
    case ORC_RX: case ORC_RY: case ORC_RZ: return 1;
    case ORC_U3: return 3;
    default: return 0;
    }
}

int orc_arity(int kind) {
    switch (kind) {
    case ORC_CNOT: case ORC_CZ: case ORC_SWAP: case ORC_MAT2: return 2;
    default: return 1;
    }
}

static void put(double *out, int idx, cplx v) { out[2 * idx] = creal(v); out[2 * idx + 1] = cimag(v); }

/* Gate matrices, readings R2-R5 of DESIGN.md (textbook definitions). */
int orc_gate_matrix(int kind, const double *p, const double *m, double *out) {
    const double r2 = 1.0 / sqrt(2.0);
    int dim = orc_arity(kind) == 2 ? 4 : 2;
    for (int i = 0; i < 2 * dim * dim; i++) out[i] = 0.0;
    double c, s;
    switch (kind) {
    case ORC_I: put(out, 0, 1); put(out, 3, 1); break;
    case ORC_X: put(out, 1, 1); put(out, 2, 1); break;
    case ORC_Y: put(out, 1, -I); put(out, 2, I); break;
    case ORC_Z: put(out, 0, 1); put(out, 3, -1); break;
    case ORC_H: put(out, 0, r2); put(out, 1, r2); put(out, 2, r2); put(out, 3, -r2); break;
    case ORC_S: put(out, 0, 1); put(out, 3, I); break;
    case ORC_SDG: put(out, 0, 1); put(out, 3, -I); break;
    case ORC_T: put(out, 0, 1); put(out, 3, cexp(I * M_PI / 4)); break;
    case ORC_TDG: put(out, 0, 1); put(out, 3, cexp(-I * M_PI / 4)); break;
    case ORC_RX: /* exp(-i th X/2) = [[c, -is], [-is, c]] */
        c = cos(p[0] / 2); s = sin(p[0] / 2);
        put(out, 0, c); put(out, 1, -I * s); put(out, 2, -I * s); put(out, 3, c); break;
    case ORC_RY: /* exp(-i th Y/2) = [[c, -s], [s, c]] */
        c = cos(p[0] / 2); s = sin(p[0] / 2);
        put(out, 0, c); put(out, 1, -s); put(out, 2, s); put(out, 3, c); break;
    case ORC_RZ: /* exp(-i th Z/2) = diag(e^{-i th/2}, e^{i th/2}) */
        put(out, 0, cexp(-I * p[0] / 2)); put(out, 3, cexp(I * p[0] / 2)); break;
    case ORC_U3: /* OpenQASM U(th, ph, la), reading R5 */
        c = cos(p[0] / 2); s = sin(p[0] / 2);
        put(out, 0, c); put(out, 1, -cexp(I * p[2]) * s);
        put(out, 2, cexp(I * p[1]) * s); put(out, 3, cexp(I * (p[1] + p[2])) * c); break;
    case ORC_CNOT: /* wires [control, target]; control = MSB of the 4x4 index */
        put(out, 0, 1); put(out, 5, 1); put(out, 11, 1); put(out, 14, 1); break;
    case ORC_CZ: put(out, 0, 1); put(out, 5, 1); put(out, 10, 1); put(out, 15, -1); break;
    case ORC_SWAP: put(out, 0, 1); put(out, 6, 1); put(out, 9, 1); put(out, 15, 1); break;
    case ORC_MAT1: for (int i = 0; i < 8; i++) out[i] = m[i]; break;
    case ORC_MAT2: for (int i = 0; i < 32; i++) out[i] = m[i]; break;
    default: return -1;
    }
    return 0;
}

/* d M / d params[which], differentiated entry by entry from the matrices above. */
int orc_gate_dmatrix(int kind, const double *p, int which, double *out) {
    for (int i = 0; i < 8; i++) out[i] = 0.0;
    double c, s;
    switch (kind) {
    case ORC_RX:
        if (which != 0) return -1;
        c = cos(p[0] / 2); s = sin(p[0] / 2);
        put(out, 0, -s / 2); put(out, 1, -I * c / 2); put(out, 2, -I * c / 2); put(out, 3, -s / 2);
        return 0;
    case ORC_RY:
        if (which != 0) return -1;
        c = cos(p[0] / 2); s = sin(p[0] / 2);
        put(out, 0, -s / 2); put(out, 1, -c / 2); put(out, 2, c / 2); put(out, 3, -s / 2);
        return 0;
    case ORC_RZ:
        if (which != 0) return -1;
        put(out, 0, -I / 2 * cexp(-I * p[0] / 2)); put(out, 3, I / 2 * cexp(I * p[0] / 2));
        return 0;
    case ORC_U3:
        c = cos(p[0] / 2); s = sin(p[0] / 2);
        if (which == 0) {        /* d/d theta */
            put(out, 0, -s / 2); put(out, 1, -cexp(I * p[2]) * c / 2);
            put(out, 2, cexp(I * p[1]) * c / 2); put(out, 3, -cexp(I * (p[1] + p[2])) * s / 2);
        } else if (which == 1) { /* d/d phi */
            put(out, 2, I * cexp(I * p[1]) * s); put(out, 3, I * cexp(I * (p[1] + p[2])) * c);
        } else if (which == 2) { /* d/d lambda */
            put(out, 1, -I * cexp(I * p[2]) * s); put(out, 3, I * cexp(I * (p[1] + p[2])) * c);
        } else {
            return -1;
        }
        return 0;
    default:
        return -1;
    }
}

void orc_init_zero(double *psi, int n) {
    size_t N = (size_t)1 << n;
    memset(psi, 0, 2 * N * sizeof(double));
    psi[0] = 1.0;
}

static inline uint64_t qbit(int n, int q) { return (uint64_t)1 << (n - 1 - q); }

/* Apply a dense 2x2 (complex, row-major) on logical qubit q:
 * for every i with bit_q(i) = 0, j = i + 2^{n-1-q}:
 *   (psi_i, psi_j) <- (M00 psi_i + M01 psi_j, M10 psi_i + M11 psi_j)     */
static void apply1(cplx *psi, int n, int q, const cplx *M) {
    const uint64_t N = (uint64_t)1 << n, b = qbit(n, q);
#pragma omp parallel for schedule(static) if (n >= 14)
    for (int64_t ii = 0; ii < (int64_t)N; ii++) {
        uint64_t i = (uint64_t)ii;
        if (i & b) continue;
        uint64_t j = i | b;
        cplx a0 = psi[i], a1 = psi[j];
        psi[i] = M[0] * a0 + M[1] * a1;
        psi[j] = M[2] * a0 + M[3] * a1;
    }
}

/* Apply a dense 4x4 on (q0, q1); q0 is the MSB of the 4x4 index (R2). */
static void apply2(cplx *psi, int n, int q0, int q1, const cplx *M) {
    const uint64_t N = (uint64_t)1 << n, b0 = qbit(n, q0), b1 = qbit(n, q1);
#pragma omp parallel for schedule(static) if (n >= 14)
    for (int64_t ii = 0; ii < (int64_t)N; ii++) {
        uint64_t i = (uint64_t)ii;
        if (i & (b0 | b1)) continue;
        uint64_t idx[4] = {i, i | b1, i | b0, i | b0 | b1};
        cplx v[4], w[4];
        for (int a = 0; a < 4; a++) v[a] = psi[idx[a]];
        for (int r = 0; r < 4; r++) {
            w[r] = 0;
            for (int a = 0; a < 4; a++) w[r] += M[4 * r + a] * v[a];
        }
        for (int a = 0; a < 4; a++) psi[idx[a]] = w[a];
    }
}

static int check_wires(int n, int kind, const int *w) {
    if (kind < 0 || kind >= ORC_NKINDS) return -1;
    if (w[0] < 0 || w[0] >= n) return -1;
    if (orc_arity(kind) == 2 && (w[1] < 0 || w[1] >= n || w[1] == w[0])) return -1;
    return 0;
}

static int apply_mat(double *psi, int n, int kind, const int *w, const double *mraw) {
    cplx M[16];
    int dim = orc_arity(kind) == 2 ? 4 : 2;
    for (int i = 0; i < dim * dim; i++) M[i] = mraw[2 * i] + I * mraw[2 * i + 1];
    if (dim == 2) apply1((cplx *)psi, n, w[0], M);
    else apply2((cplx *)psi, n, w[0], w[1], M);
    return 0;
}

int orc_apply_gate(double *psi, int n, int kind, const int *w, const double *params, const double *mat) {
    if (check_wires(n, kind, w)) return -1;
    double M[32];
    if (orc_gate_matrix(kind, params, mat, M)) return -1;
    return apply_mat(psi, n, kind, w, M);
}

/* psi <- U^dagger psi (the recompute step x = U^* y of PAPER.md:233-235). */
int orc_apply_gate_dagger(double *psi, int n, int kind, const int *w, const double *params, const double *mat) {
    if (check_wires(n, kind, w)) return -1;
    double M[32], D[32];
    if (orc_gate_matrix(kind, params, mat, M)) return -1;
    int dim = orc_arity(kind) == 2 ? 4 : 2;
    for (int r = 0; r < dim; r++)
        for (int c = 0; c < dim; c++) {        /* D[r][c] = conj(M[c][r]) */
            D[2 * (dim * r + c)] = M[2 * (dim * c + r)];
            D[2 * (dim * r + c) + 1] = -M[2 * (dim * c + r) + 1];
        }
    return apply_mat(psi, n, kind, w, D);
}

int orc_run(int n, int G, const int *kinds, const int *wires, const double *params,
            const double *mats, double *psi) {
    if (n < 1 || n > 40) return -1;
    orc_init_zero(psi, n);
    for (int g = 0; g < G; g++)
        if (orc_apply_gate(psi, n, kinds[g], wires + 2 * g, params + 3 * g, mats + 32 * g)) return -1;
    return 0;
}

/* out = P psi for the Pauli string (x, z) given on logical-qubit masks:
 * (P psi)_{b xor x} = phase(b) psi_b,
 * phase(b) = prod_{q in z} (-1)^{b_q} * prod_{q in x and z} i      (Y = iXZ) */
static void apply_pauli(const cplx *psi, cplx *out, int n, uint64_t xm, uint64_t zm) {
    uint64_t X = 0, Z = 0;
    int ny = 0;
    for (int q = 0; q < n; q++) {
        if ((xm >> q) & 1) X |= qbit(n, q);
        if ((zm >> q) & 1) Z |= qbit(n, q);
        if (((xm & zm) >> q) & 1) ny++;
    }
    cplx iy = 1;
    for (int k = 0; k < ny; k++) iy *= I;
    const uint64_t N = (uint64_t)1 << n;
#pragma omp parallel for schedule(static) if (n >= 14)
    for (int64_t bb = 0; bb < (int64_t)N; bb++) {
        uint64_t b = (uint64_t)bb;
        double sgn = (__builtin_popcountll(b & Z) & 1) ? -1.0 : 1.0;
        out[b ^ X] = iy * sgn * psi[b];
    }
}

static int check_masks(int n, int T, const uint64_t *x, const uint64_t *z) {
    uint64_t lim = n >= 64 ? ~0ull : (((uint64_t)1 << n) - 1);
    for (int t = 0; t < T; t++)
        if ((x[t] & ~lim) || (z[t] & ~lim)) return -1;
    return 0;
}

/* <psi|P_t|psi>, out[t] = c_t * <P_t>. */
int orc_expval(const double *psi_, int n, int T, const uint64_t *x, const uint64_t *z,
               const double *c, double *out) {
    if (check_masks(n, T, x, z)) return -1;
    const cplx *psi = (const cplx *)psi_;
    const uint64_t N = (uint64_t)1 << n;
    cplx *tmp = (cplx *)malloc(N * sizeof(cplx));
    if (!tmp) return -1;
    for (int t = 0; t < T; t++) {
        apply_pauli(psi, tmp, n, x[t], z[t]);
        double acc = 0.0;
#pragma omp parallel for reduction(+ : acc) schedule(static) if (n >= 14)
        for (int64_t b = 0; b < (int64_t)N; b++) acc += creal(conj(psi[b]) * tmp[b]);
        out[t] = (c ? c[t] : 1.0) * acc;
    }
    free(tmp);
    return 0;
}

int orc_count_params(int G, const int *kinds, const int *trainable) {
    int P = 0;
    for (int g = 0; g < G; g++)
        if (trainable[g]) P += orc_num_params(kinds[g]);
    return P;
}

/* lam = sum_t c_t P_t psi */
static int hamiltonian_apply(const cplx *psi, cplx *lam, int n, int T, const uint64_t *x,
                             const uint64_t *z, const double *c) {
    const uint64_t N = (uint64_t)1 << n;
    cplx *tmp = (cplx *)malloc(N * sizeof(cplx));
    if (!tmp) return -1;
    memset(lam, 0, N * sizeof(cplx));
    for (int t = 0; t < T; t++) {
        apply_pauli(psi, tmp, n, x[t], z[t]);
        double ct = c ? c[t] : 1.0;
        for (uint64_t b = 0; b < N; b++) lam[b] += ct * tmp[b];
    }
    free(tmp);
    return 0;
}

static double re_inner(const cplx *a, const cplx *b, int n) { /* Re <a|b> */
    const uint64_t N = (uint64_t)1 << n;
    double acc = 0.0;
#pragma omp parallel for reduction(+ : acc) schedule(static) if (n >= 14)
    for (int64_t i = 0; i < (int64_t)N; i++) acc += creal(conj(a[i]) * b[i]);
    return acc;
}

/* mu <- (dM/dtheta_which) psi, applied like a gate (dM is not unitary). */
static int apply_dgate(const cplx *psi, cplx *mu, int n, int kind, const int *w,
                       const double *params, int which) {
    double D[8];
    if (orc_gate_dmatrix(kind, params, which, D)) return -1;
    memcpy(mu, psi, ((size_t)1 << n) * sizeof(cplx));
    cplx M[4];
    for (int i = 0; i < 4; i++) M[i] = D[2 * i] + I * D[2 * i + 1];
    apply1(mu, n, w[0], M);
    return 0;
}

/* Textbook adjoint (reverse) sweep of PAPER.md:220-236:
 *   lam <- H psi_K
 *   for k = K..1:  psi <- U_k^dag psi                  (x = U^* y)
 *                  g_p = 2 Re <lam | dU_k/dtheta_p | psi>
 *                  lam <- U_k^dag lam                  (dx = U^T dy, R(U)^T = R(U^dag))  */
int orc_adjoint(int n, int G, const int *kinds, const int *wires, const double *params,
                const double *mats, const int *trainable, int T, const uint64_t *x,
                const uint64_t *z, const double *c, double *value, double *grad) {
    if (check_masks(n, T, x, z)) return -1;
    const uint64_t N = (uint64_t)1 << n;
    cplx *psi = (cplx *)malloc(N * sizeof(cplx));
    cplx *lam = (cplx *)malloc(N * sizeof(cplx));
    cplx *mu = (cplx *)malloc(N * sizeof(cplx));
    int rc = -1;
    if (!psi || !lam || !mu) goto done;
    if (orc_run(n, G, kinds, wires, params, mats, (double *)psi)) goto done;
    if (hamiltonian_apply(psi, lam, n, T, x, z, c)) goto done;
    *value = re_inner(psi, lam, n);
    int p = orc_count_params(G, kinds, trainable);
    for (int g = G - 1; g >= 0; g--) {
        const int *w = wires + 2 * g;
        const double *pr = params + 3 * g;
        if (orc_apply_gate_dagger((double *)psi, n, kinds[g], w, pr, mats + 32 * g)) goto done;
        if (trainable[g]) {
            int np = orc_num_params(kinds[g]);
            p -= np;
            for (int k = 0; k < np; k++) {
                if (apply_dgate(psi, mu, n, kinds[g], w, pr, k)) goto done;
                grad[p + k] = 2.0 * re_inner(lam, mu, n);
            }
        }
        if (orc_apply_gate_dagger((double *)lam, n, kinds[g], w, pr, mats + 32 * g)) goto done;
    }
    rc = 0;
done:
    free(psi); free(lam); free(mu);
    return rc;
}

/* Stored-activation reverse mode (what autograd does without the invertible
 * trick): keep every psi_k, no un-application of psi.          */
int orc_adjoint_stored(int n, int G, const int *kinds, const int *wires, const double *params,
                       const double *mats, const int *trainable, int T, const uint64_t *x,
                       const uint64_t *z, const double *c, double *value, double *grad) {
    if (check_masks(n, T, x, z) || n > 16) return -1;
    const uint64_t N = (uint64_t)1 << n;
    cplx *states = (cplx *)malloc((size_t)(G + 1) * N * sizeof(cplx));
    cplx *lam = (cplx *)malloc(N * sizeof(cplx));
    cplx *mu = (cplx *)malloc(N * sizeof(cplx));
    int rc = -1;
    if (!states || !lam || !mu) goto done;
    orc_init_zero((double *)states, n);
    for (int g = 0; g < G; g++) {
        memcpy(states + (size_t)(g + 1) * N, states + (size_t)g * N, N * sizeof(cplx));
        if (orc_apply_gate((double *)(states + (size_t)(g + 1) * N), n, kinds[g], wires + 2 * g,
                           params + 3 * g, mats + 32 * g)) goto done;
    }
    if (hamiltonian_apply(states + (size_t)G * N, lam, n, T, x, z, c)) goto done;
    *value = re_inner(states + (size_t)G * N, lam, n);
    int p = orc_count_params(G, kinds, trainable);
    for (int g = G - 1; g >= 0; g--) {
        const int *w = wires + 2 * g;
        const double *pr = params + 3 * g;
        if (trainable[g]) {
            int np = orc_num_params(kinds[g]);
            p -= np;
            for (int k = 0; k < np; k++) {
                if (apply_dgate(states + (size_t)g * N, mu, n, kinds[g], w, pr, k)) goto done;
                grad[p + k] = 2.0 * re_inner(lam, mu, n);
            }
        }
        if (orc_apply_gate_dagger((double *)lam, n, kinds[g], w, pr, mats + 32 * g)) goto done;
    }
    rc = 0;
done:
    free(states); free(lam); free(mu);
    return rc;
}

static double energy(int n, int G, const int *kinds, const int *wires, const double *params,
                     const double *mats, int T, const uint64_t *x, const uint64_t *z,
                     const double *c, double *psi, double *tmp_out, int *err) {
    if (orc_run(n, G, kinds, wires, params, mats, psi) || orc_expval(psi, n, T, x, z, c, tmp_out)) {
        *err = 1;
        return 0.0;
    }
    double e = 0.0;
    for (int t = 0; t < T; t++) e += tmp_out[t];
    return e;
}

/* g_p = [E(theta_p + s) - E(theta_p - s)] / (2 sin s) with s = pi/2: exact for
 * gates exp(-i theta P/2) and for each U3 angle (U3 = e^{i(ph+la)/2} RZ RY RZ). */
static int shifted(int n, int G, const int *kinds, const int *wires, const double *params,
                   const double *mats, const int *trainable, int T, const uint64_t *x,
                   const uint64_t *z, const double *c, double h, int central_fd, double *grad) {
    if (check_masks(n, T, x, z)) return -1;
    const uint64_t N = (uint64_t)1 << n;
    double *psi = (double *)malloc(2 * N * sizeof(double));
    double *pp = (double *)malloc(3 * (size_t)G * sizeof(double));
    double *tout = (double *)malloc((size_t)(T > 0 ? T : 1) * sizeof(double));
    int rc = -1, err = 0, p = 0;
    if (!psi || !pp || !tout) goto done;
    memcpy(pp, params, 3 * (size_t)G * sizeof(double));
    for (int g = 0; g < G; g++) {
        if (!trainable[g]) continue;
        for (int k = 0; k < orc_num_params(kinds[g]); k++) {
            double th = params[3 * g + k];
            pp[3 * g + k] = th + h;
            double ep = energy(n, G, kinds, wires, pp, mats, T, x, z, c, psi, tout, &err);
            pp[3 * g + k] = th - h;
            double em = energy(n, G, kinds, wires, pp, mats, T, x, z, c, psi, tout, &err);
            pp[3 * g + k] = th;
            grad[p++] = central_fd ? (ep - em) / (2 * h) : (ep - em) / 2.0;
        }
    }
    rc = err ? -1 : 0;
done:
    free(psi); free(pp); free(tout);
    return rc;
}

int orc_param_shift(int n, int G, const int *kinds, const int *wires, const double *params,
                    const double *mats, const int *trainable, int T, const uint64_t *x,
                    const uint64_t *z, const double *c, double *grad) {
    return shifted(n, G, kinds, wires, params, mats, trainable, T, x, z, c, M_PI / 2, 0, grad);
}

int orc_finite_diff(int n, int G, const int *kinds, const int *wires, const double *params,
                    const double *mats, const int *trainable, int T, const uint64_t *x,
                    const uint64_t *z, const double *c, double eps, double *grad) {
    return shifted(n, G, kinds, wires, params, mats, trainable, T, x, z, c, eps, 1, grad);
}

/* ---- shot noise: approximate (Gaussian) sampler, PAPER.md:200-218 -------- */
static uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

double orc_uniform(uint64_t seed, uint64_t k) {
    return (double)(splitmix64(seed ^ (k * 0xD1B54A32D192ED03ull)) >> 11) * 0x1.0p-53;
}

double orc_normal(uint64_t seed, uint64_t i) {
    const double u1 = orc_uniform(seed, 2 * i), u2 = orc_uniform(seed, 2 * i + 1);
    return sqrt(-2.0 * log(1.0 - u1)) * cos(2.0 * M_PI * u2);
}

int orc_gauss_sample(const double *psi_, int n, double shots, uint64_t seed, double *y) {
    if (n < 1 || n > 30 || !(shots > 0)) return -1;
    const cplx *psi = (const cplx *)psi_;
    const uint64_t N = (uint64_t)1 << n, K = N - 1;
    double *u = (double *)malloc(N * sizeof(double));
    double *v = (double *)malloc(N * sizeof(double));
    double *z = (double *)malloc(N * sizeof(double));
    if (!u || !v || !z) { free(u); free(v); free(z); return -1; }
    /* u = sqrt(p);  v~ = e_K - u;  v = v~ / ||v~|| */
    double nv = 0.0;
    for (uint64_t i = 0; i < N; i++) {
        const double p = creal(psi[i]) * creal(psi[i]) + cimag(psi[i]) * cimag(psi[i]);
        u[i] = sqrt(p);
        v[i] = (i == K ? 1.0 : 0.0) - u[i];
        nv += v[i] * v[i];
        z[i] = i == K ? 0.0 : orc_normal(seed, i);
    }
    nv = sqrt(nv);
    for (uint64_t i = 0; i < N; i++) v[i] = nv > 1e-300 ? v[i] / nv : 0.0;
    /* x = S z with S the Householder reflection I - 2 v v^T (reading R21: PAPER.md:209
     * prints I - v v^T, which is a projection and not the factorisation the text asks
     * for; the reflection maps e_K <-> u, so Cov x = S (I - e_K e_K^T) S = I - u u^T);
     * y = shots p + sqrt(shots) D x */
    double vz = 0.0;
    for (uint64_t i = 0; i < N; i++) vz += v[i] * z[i];
    for (uint64_t i = 0; i < N; i++) {
        const double x = z[i] - 2.0 * v[i] * vz;
        y[i] = shots * u[i] * u[i] + sqrt(shots) * u[i] * x;
    }
    free(u); free(v); free(z);
    return 0;
}

int orc_gauss_z(const double *psi, int n, double shots, uint64_t seed, double *out_z) {
    const uint64_t N = (uint64_t)1 << n;
    double *y = (double *)malloc(N * sizeof(double));
    if (!y) return -1;
    int rc = orc_gauss_sample(psi, n, shots, seed, y);
    if (rc) { free(y); return rc; }
    for (int q = 0; q < n; q++) {
        double acc = 0.0;
        for (uint64_t i = 0; i < N; i++) acc += (i & qbit(n, q)) ? -y[i] : y[i];
        out_z[q] = acc / shots;
    }
    free(y);
    return 0;
}
