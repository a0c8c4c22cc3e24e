/*
 * oracle.h -- plain float64 CPU state-vector simulator: the TEST ORACLE.
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline / --impl reference
 * leg may load or execute anything under oracle/.  It shares no code, header,
 * table or constant with the CUDA path (paper_2511_19291_b200/csrc), and the
 * CUDA path never calls it.
 *
 * What it computes (all citations are to /root/reference/PAPER.md lines):
 *   - state psi in C^{2^n}, |0..0> initial state
 *   - gate (M, Q) applied as the contraction
 *         Y_{..J..} = sum_L M_{JL} X_{..L..}                (Alg. 1 at 121-134)
 *     written out by index arithmetic, one gate at a time, no fusion
 *   - Pauli expectation <psi|P|psi>
 *   - gradients by the invertible reverse sweep: x = U^* y   (Eq. save_x)
 *   - independent checks: stored-activation reverse mode, parameter shift,
 *     central finite differences.
 *
 * Conventions:
 *   R1  canonical index: logical qubit q <-> index bit (n-1-q)  (MSB-first)
 *   R2  2q matrices: wires[0] is the more significant bit of the 4x4 index
 *   R3  CNOT wires = [control, target]
 *   R4  R_P(theta) = exp(-i theta P / 2)
 *   R5  U3(th,ph,la) = [[c, -e^{i la} s], [e^{i ph} s, e^{i(ph+la)} c]],
 *       c = cos(th/2), s = sin(th/2)
 *   Pauli masks: bit q of x_mask / z_mask <-> logical qubit q;
 *   (x,z) = (0,0) I, (1,0) X, (0,1) Z, (1,1) Y.
 *
 * Gate kind codes (this file's own numbering; the Python harness maps gate
 * NAMES to these codes, it never passes codes from the CUDA side):
 */
#ifndef TQD_ORACLE_H
#define TQD_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    ORC_I = 0, ORC_X, ORC_Y, ORC_Z, ORC_H, ORC_S, ORC_SDG, ORC_T, ORC_TDG,
    ORC_CNOT, ORC_CZ, ORC_SWAP, ORC_MAT1, ORC_MAT2,
    ORC_RX, ORC_RY, ORC_RZ, ORC_U3,
    ORC_NKINDS
};

/* A circuit is passed as parallel arrays of length G:
 *   kinds[g]          gate code
 *   wires[2g..2g+1]   logical wires (second ignored for 1q gates)
 *   params[3g..3g+2]  angles (RX/RY/RZ use params[3g]; U3 uses all three)
 *   mats[32g..32g+31] MAT1: 2x2, MAT2: 4x4 row-major (re,im) pairs
 *   trainable[g]      nonzero: its angles get gradient slots, in recording
 *                     order (U3 contributes theta, phi, lambda)
 * psi is interleaved (re,im) float64, 2^n complex entries.
 * Every function returns 0 on success and -1 on a bad argument.          */

int  orc_num_params(int kind);                       /* 0, 1 or 3 */
int  orc_arity(int kind);                            /* 1 or 2    */
int  orc_gate_matrix(int kind, const double *params, const double *mat_in,
                     double *out /* dim*dim complex, (re,im) */);
int  orc_gate_dmatrix(int kind, const double *params, int which,
                      double *out /* d M / d params[which] */);

void orc_init_zero(double *psi, int n);
int  orc_apply_gate(double *psi, int n, int kind, const int *wires,
                    const double *params, const double *mat);
int  orc_apply_gate_dagger(double *psi, int n, int kind, const int *wires,
                           const double *params, const double *mat);
int  orc_run(int n, int G, const int *kinds, const int *wires, const double *params,
             const double *mats, double *psi_out);

int  orc_expval(const double *psi, int n, int T, const uint64_t *x_mask,
                const uint64_t *z_mask, const double *coeff, double *out /* T */);

int  orc_count_params(int G, const int *kinds, const int *trainable);

/* value = sum_t c_t <psi_K|P_t|psi_K>; grad[p] = d value / d theta_p */
int  orc_adjoint(int n, int G, const int *kinds, const int *wires, const double *params,
                 const double *mats, const int *trainable, int T, const uint64_t *x_mask,
                 const uint64_t *z_mask, const double *coeff, double *value, double *grad);
int  orc_adjoint_stored(int n, int G, const int *kinds, const int *wires, const double *params,
                        const double *mats, const int *trainable, int T, const uint64_t *x_mask,
                        const uint64_t *z_mask, const double *coeff, double *value, double *grad);
int  orc_param_shift(int n, int G, const int *kinds, const int *wires, const double *params,
                     const double *mats, const int *trainable, int T, const uint64_t *x_mask,
                     const uint64_t *z_mask, const double *coeff, double *grad);
int  orc_finite_diff(int n, int G, const int *kinds, const int *wires, const double *params,
                     const double *mats, const int *trainable, int T, const uint64_t *x_mask,
                     const uint64_t *z_mask, const double *coeff, double eps, double *grad);
int  orc_num_threads(void);

/* ---- shot noise, approximate (Gaussian) sampler ----------
 * Counter-based random numbers (the library implements the same DEFINITION in
 * its own code; nothing is shared):
 *   splitmix64(x): x += 0x9E3779B97F4A7C15; x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9;
 *                  x = (x ^ (x >> 27)) * 0x94D049BB133111EB; return x ^ (x >> 31)
 *   uniform(seed, k) = (splitmix64(seed ^ (k * 0xD1B54A32D192ED03)) >> 11) * 2^-53
 *   normal(seed, i)  = sqrt(-2 ln(1 - uniform(seed, 2i))) * cos(2 pi uniform(seed, 2i + 1))
 * orc_gauss_sample: the approximate multinomial sample of `shots` shots over the
 * 2^n canonical outcomes, y = shots p + sqrt(shots) D S z, written out as in the
 * paper: p_i = |psi_i|^2, D = diag(sqrt p), u = sqrt p, v~ = e_K - u with K the
 * last outcome (2^n - 1), v = v~ / ||v~|| (v = 0 if u = e_K), S = I - 2 v v^T (the
 * Householder reflection; reading R21, PAPER.md:209 prints I - v v^T),
 * z_i = normal(seed, i) for i < K and z_K = 0.  out_y: 2^n values.
 * orc_gauss_z: the per-qubit estimates Z_q = (1/shots) sum_i y_i (-1)^{bit of
 * qubit q in i} (measure_allZ with shots). */
double orc_uniform(uint64_t seed, uint64_t k);
double orc_normal(uint64_t seed, uint64_t i);
int  orc_gauss_sample(const double *psi, int n, double shots, uint64_t seed, double *out_y);
int  orc_gauss_z(const double *psi, int n, double shots, uint64_t seed, double *out_z);

/* ---- Clifford circuits at full size (clifford.c; stabilizer tableau) --------
 * Gates I X Y Z H S SDG CNOT CZ SWAP and RX / RY / RZ / U3 at multiples of pi/2;
 * anything else returns -1 (mats are not read).  n <= 63.
 * orc_clifford_expval: out[t] = c_t <P_t> (each <P_t> in {-1, 0, +1}), c NULL = 1.
 * orc_clifford_grad:   value = sum_t c_t <P_t>; grad by parameter shift (+-pi/2),
 *                      slot order as orc_param_shift.                        */
int  orc_clifford_expval(int n, int G, const int *kinds, const int *wires, const double *params,
                         int T, const uint64_t *x_mask, const uint64_t *z_mask, const double *coeff,
                         double *out);
int  orc_clifford_grad(int n, int G, const int *kinds, const int *wires, const double *params,
                       const int *trainable, int T, const uint64_t *x_mask, const uint64_t *z_mask,
                       const double *coeff, double *value, double *grad);
/* the n stabilizer generators of the final state: sign[k] P_k |psi> = |psi> */
int  orc_clifford_stabilizers(int n, int G, const int *kinds, const int *wires, const double *params,
                              uint64_t *x_out, uint64_t *z_out, int *sign_out);

#ifdef __cplusplus
}
#endif
#endif
