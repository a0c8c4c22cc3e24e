/*
 * clifford.c -- stabilizer-tableau simulator for Clifford circuits: TEST ORACLE.
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE (same rules as oracle.h: only
 * tests/, smoke() and bench.py's cpu_baseline / reference leg may load it; it
 * shares nothing with the CUDA path).
 *
 * Why: at the benchmark sizes (30 / 33 qubits) the state-vector oracle cannot
 * run, but a circuit of Clifford gates -- H, S, CNOT and everything they
 * generate, including RX / RY / RZ (PAPER.md R4: exp(-i theta P / 2)) at angles
 * theta = k pi / 2 -- maps Pauli operators to Pauli operators, so its expectation
 * values <P> = <0|U^dag P U|0> are exactly 0 or +-1 and follow from the
 * stabilizer tableau in O(n) bit operations per gate and row (Aaronson &
 * Gottesman, "Improved simulation of stabilizer circuits", Phys. Rev. A 70,
 * 052328 (2004): the CHP tableau of n destabilizer and n stabilizer rows, the
 * H / S / CNOT update rules and the rowsum phase rule are written out below in
 * that paper's notation).  Gradients at such angles by the parameter-shift rule
 * dE/dtheta = [E(theta + pi/2) - E(theta - pi/2)] / 2 (exact for exp(-i theta P/2),
 * and per angle for U3; oracle.c shifted()), whose shifted circuits are Clifford
 * again.  This checks what the method computes (PAPER.md:66-72 expectations,
 * PAPER.md:220-236 gradients) on entangled states at full size.
 *
 * Conventions as oracle.h: Pauli masks bit q <-> logical qubit q, (x,z) = (0,0) I,
 * (1,0) X, (0,1) Z, (1,1) Y; CNOT wires = [control, target]; U3 = e^{i(ph+la)/2}
 * RZ(ph) RY(th) RZ(la).  Global phases are irrelevant to <P>.
 * Gates taken: I X Y Z H S SDG CNOT CZ SWAP, RX RY RZ U3 at multiples of pi/2
 * (within 1e-9).  T, TDG, MAT1, MAT2 and other angles: error (-1).
 *
 * Pinned (tests/test_oracle_clifford.py) against the state-vector oracle
 * (orc_run + orc_expval, orc_adjoint) on random Clifford circuits at n <= 9, and
 * against closed forms (GHZ / Bell correlators) at n = 40.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

typedef struct {
    int n;
    uint64_t x[129], z[129];  /* rows 0..n-1 destabilizers, n..2n-1 stabilizers, 2n scratch */
    uint8_t r[129];
} Tab;

static void tab_init(Tab *t, int n) {
    memset(t, 0, sizeof(*t));
    t->n = n;
    for (int i = 0; i < n; i++) {
        t->x[i] = (uint64_t)1 << i;      /* destabilizer X_i */
        t->z[n + i] = (uint64_t)1 << i;  /* stabilizer Z_i: |0..0> */
    }
}

/* CHP rules, every row i of the tableau */
static void tab_h(Tab *t, int a) {
    const uint64_t m = (uint64_t)1 << a;
    for (int i = 0; i < 2 * t->n; i++) {
        const uint64_t xa = t->x[i] & m, za = t->z[i] & m;
        if (xa && za) t->r[i] ^= 1;
        t->x[i] = (t->x[i] & ~m) | za;
        t->z[i] = (t->z[i] & ~m) | xa;
    }
}

static void tab_s(Tab *t, int a) {
    const uint64_t m = (uint64_t)1 << a;
    for (int i = 0; i < 2 * t->n; i++) {
        if ((t->x[i] & m) && (t->z[i] & m)) t->r[i] ^= 1;
        if (t->x[i] & m) t->z[i] ^= m;
    }
}

static void tab_cnot(Tab *t, int a, int b) {
    const uint64_t ma = (uint64_t)1 << a, mb = (uint64_t)1 << b;
    for (int i = 0; i < 2 * t->n; i++) {
        const int xa = (t->x[i] & ma) != 0, zb = (t->z[i] & mb) != 0;
        const int xb = (t->x[i] & mb) != 0, za = (t->z[i] & ma) != 0;
        if (xa && zb && (xb ^ za ^ 1)) t->r[i] ^= 1;
        if (xa) t->x[i] ^= mb;
        if (zb) t->z[i] ^= ma;
    }
}

/* Pauli gates: conjugation only flips signs */
static void tab_pauli(Tab *t, int a, int px, int pz) {
    const uint64_t m = (uint64_t)1 << a;
    for (int i = 0; i < 2 * t->n; i++) {
        int f = 0;
        if (px && (t->z[i] & m)) f ^= 1; /* X anticommutes with Z, Y */
        if (pz && (t->x[i] & m)) f ^= 1; /* Z anticommutes with X, Y */
        t->r[i] ^= (uint8_t)f;
    }
}

/* the exponent of i contributed when multiplying Pauli (x1,z1) into (x2,z2) (CHP g) */
static int chp_g(int x1, int z1, int x2, int z2) {
    if (!x1 && !z1) return 0;
    if (x1 && z1) return z2 - x2;
    if (x1 && !z1) return z2 * (2 * x2 - 1);
    return x2 * (1 - 2 * z2);
}

/* row h <- row i * row h (CHP rowsum) */
static void tab_rowsum(Tab *t, int h, int i) {
    int s = 2 * t->r[h] + 2 * t->r[i];
    for (int q = 0; q < t->n; q++)
        s += chp_g((int)((t->x[i] >> q) & 1), (int)((t->z[i] >> q) & 1), (int)((t->x[h] >> q) & 1),
                   (int)((t->z[h] >> q) & 1));
    s = ((s % 4) + 4) % 4;
    t->r[h] = (uint8_t)(s == 0 ? 0 : 1);
    t->x[h] ^= t->x[i];
    t->z[h] ^= t->z[i];
}

static int anticommute(uint64_t x1, uint64_t z1, uint64_t x2, uint64_t z2) {
    return __builtin_popcountll((x1 & z2) ^ (z1 & x2)) & 1;
}

/* <P> of the stabilizer state: 0 if P anticommutes with a stabilizer, else the
 * sign of P in the stabilizer group (P = +-prod of the stabilizers whose
 * destabilizer partners anticommute with P) */
static int tab_expect(Tab *t, uint64_t px, uint64_t pz) {
    const int n = t->n;
    for (int i = n; i < 2 * n; i++)
        if (anticommute(t->x[i], t->z[i], px, pz)) return 0;
    const int s = 2 * n;
    t->x[s] = t->z[s] = 0;
    t->r[s] = 0;
    for (int i = 0; i < n; i++)
        if (anticommute(t->x[i], t->z[i], px, pz)) tab_rowsum(t, s, i + n);
    if (t->x[s] != px || t->z[s] != pz) return 2; /* cannot happen for a valid tableau */
    return t->r[s] ? -1 : 1;
}

/* theta = k pi/2 -> k mod 4, else -1 */
static int quarter_turns(double th) {
    const double q = th / (M_PI / 2);
    const double k = nearbyint(q);
    if (fabs(q - k) > 1e-9) return -1;
    return (int)(((long long)k % 4 + 4) % 4);
}

static int rz_k(Tab *t, int a, int k) { /* RZ(pi/2) ~ S */
    for (int j = 0; j < k; j++) tab_s(t, a);
    return 0;
}
static int rx_k(Tab *t, int a, int k) { /* RX(pi/2) ~ H S H */
    for (int j = 0; j < k; j++) { tab_h(t, a); tab_s(t, a); tab_h(t, a); }
    return 0;
}
static int ry_k(Tab *t, int a, int k) { /* RY(pi/2) = H Z (Z first) */
    for (int j = 0; j < k; j++) { tab_pauli(t, a, 0, 1); tab_h(t, a); }
    return 0;
}

static int tab_gate(Tab *t, int kind, const int *w, const double *p) {
    const int a = w[0], b = w[1];
    int k;
    switch (kind) {
    case ORC_I: return 0;
    case ORC_X: tab_pauli(t, a, 1, 0); return 0;
    case ORC_Y: tab_pauli(t, a, 1, 1); return 0;
    case ORC_Z: tab_pauli(t, a, 0, 1); return 0;
    case ORC_H: tab_h(t, a); return 0;
    case ORC_S: tab_s(t, a); return 0;
    case ORC_SDG: tab_s(t, a); tab_s(t, a); tab_s(t, a); return 0;
    case ORC_CNOT: tab_cnot(t, a, b); return 0;
    case ORC_CZ: tab_h(t, b); tab_cnot(t, a, b); tab_h(t, b); return 0;
    case ORC_SWAP: tab_cnot(t, a, b); tab_cnot(t, b, a); tab_cnot(t, a, b); return 0;
    case ORC_RX: if ((k = quarter_turns(p[0])) < 0) return -1; return rx_k(t, a, k);
    case ORC_RY: if ((k = quarter_turns(p[0])) < 0) return -1; return ry_k(t, a, k);
    case ORC_RZ: if ((k = quarter_turns(p[0])) < 0) return -1; return rz_k(t, a, k);
    case ORC_U3: {
        const int kt = quarter_turns(p[0]), kp = quarter_turns(p[1]), kl = quarter_turns(p[2]);
        if (kt < 0 || kp < 0 || kl < 0) return -1;
        rz_k(t, a, kl);
        ry_k(t, a, kt);
        rz_k(t, a, kp);
        return 0;
    }
    default: return -1; /* T, TDG, MAT1, MAT2: not Clifford (in general) */
    }
}

static int tab_run(Tab *t, int n, int G, const int *kinds, const int *wires, const double *params) {
    tab_init(t, n);
    for (int g = 0; g < G; g++) {
        const int *w = wires + 2 * g;
        for (int j = 0; j < orc_arity(kinds[g]); j++)
            if (w[j] < 0 || w[j] >= n) return -1;
        if (tab_gate(t, kinds[g], w, params + 3 * g)) return -1;
    }
    return 0;
}

static int clifford_energy(int n, int G, const int *kinds, const int *wires, const double *params, int T,
                           const uint64_t *x, const uint64_t *z, const double *c, double *out_terms, double *e) {
    Tab *t = (Tab *)malloc(sizeof(Tab));
    if (!t) return -1;
    int rc = tab_run(t, n, G, kinds, wires, params);
    double s = 0.0;
    for (int k = 0; k < T && !rc; k++) {
        const int v = tab_expect(t, x[k], z[k]);
        if (v == 2) { rc = -1; break; }
        const double ck = c ? c[k] : 1.0;
        if (out_terms) out_terms[k] = ck * v;
        s += ck * v;
    }
    free(t);
    if (e) *e = s;
    return rc;
}

static int clifford_masks_ok(int n, int T, const uint64_t *x, const uint64_t *z) {
    if (n < 1 || n > 63 || T < 0) return 0;
    const uint64_t lim = (uint64_t)1 << n;
    for (int t = 0; t < T; t++)
        if (x[t] >= lim || z[t] >= lim) return 0;
    return 1;
}

int orc_clifford_expval(int n, int G, const int *kinds, const int *wires, const double *params,
                        int T, const uint64_t *x, const uint64_t *z, const double *c, double *out) {
    if (!clifford_masks_ok(n, T, x, z)) return -1;
    return clifford_energy(n, G, kinds, wires, params, T, x, z, c, out, NULL);
}

int orc_clifford_grad(int n, int G, const int *kinds, const int *wires, const double *params,
                      const int *trainable, int T, const uint64_t *x, const uint64_t *z, const double *c,
                      double *out_value, double *grad) {
    if (!clifford_masks_ok(n, T, x, z)) return -1;
    if (clifford_energy(n, G, kinds, wires, params, T, x, z, c, NULL, out_value)) return -1;
    /* slot order = oracle.c shifted(): gates in order, each trainable gate's angles */
    int P = 0;
    for (int g = 0; g < G; g++)
        if (trainable[g]) P += orc_num_params(kinds[g]);
    int *sg = (int *)malloc((size_t)(P > 0 ? P : 1) * 2 * sizeof(int));
    if (!sg) return -1;
    {
        int p = 0;
        for (int g = 0; g < G; g++)
            if (trainable[g])
                for (int k = 0; k < orc_num_params(kinds[g]); k++) { sg[2 * p] = g; sg[2 * p + 1] = k; p++; }
    }
    int err = 0;
#pragma omp parallel
    {
        double *pp = (double *)malloc(3 * (size_t)(G > 0 ? G : 1) * sizeof(double));
        if (!pp) {
#pragma omp atomic write
            err = 1;
        } else {
            memcpy(pp, params, 3 * (size_t)G * sizeof(double));
#pragma omp for schedule(dynamic, 4)
            for (int p = 0; p < P; p++) {
                const int g = sg[2 * p], k = sg[2 * p + 1];
                const double th = params[3 * g + k];
                double ep = 0.0, em = 0.0;
                pp[3 * g + k] = th + M_PI / 2;
                int e1 = clifford_energy(n, G, kinds, wires, pp, T, x, z, c, NULL, &ep);
                pp[3 * g + k] = th - M_PI / 2;
                int e2 = clifford_energy(n, G, kinds, wires, pp, T, x, z, c, NULL, &em);
                pp[3 * g + k] = th;
                if (e1 || e2) {
#pragma omp atomic write
                    err = 1;
                }
                grad[p] = (ep - em) / 2.0;
            }
            free(pp);
        }
    }
    free(sg);
    return err ? -1 : 0;
}

/* the n stabilizer generators of the final state: sign_k P_k |psi> = |psi>, P_k =
 * (x_out[k], z_out[k]) (Pauli masks as above), sign_k in {+1, -1} */
int orc_clifford_stabilizers(int n, int G, const int *kinds, const int *wires, const double *params,
                             uint64_t *x_out, uint64_t *z_out, int *sign_out) {
    if (n < 1 || n > 63) return -1;
    Tab *t = (Tab *)malloc(sizeof(Tab));
    if (!t) return -1;
    int rc = tab_run(t, n, G, kinds, wires, params);
    for (int k = 0; k < n && !rc; k++) {
        x_out[k] = t->x[n + k];
        z_out[k] = t->z[n + k];
        sign_out[k] = t->r[n + k] ? -1 : 1;
    }
    free(t);
    return rc;
}
