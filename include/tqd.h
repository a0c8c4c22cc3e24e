/*
 * tqd.h -- C ABI of the B200-native sharded state-vector forward + adjoint
 * gradient path (arXiv 2511.19291, "TorchQuantumDistributed").
 *
 * The library (paper_2511_19291_b200/libtqd.so) applies a gate circuit to a
 * complex 2^n state vector sharded over GPUs, computes Pauli expectation values,
 * and computes their parameter gradients with the invertible reverse sweep.
 * Every step runs in hand-written CUDA kernels for sm_100a plus NCCL for the
 * qubit-remap exchange; there is no CPU fallback.
 *
 * Citations are PAPER.md line numbers with the
 * section / algorithm / equation they fall in.  Readings of ambiguous passages
 * (R1..R20) are listed in DESIGN.md.
 *
 * Conventions
 *   - Status: every call returns int; 0 = TQD_OK, < 0 = error (enum below).
 *     The message of the last error of the calling thread is returned by
 *     tqd_last_error().  After a CUDA or NCCL error the context is poisoned:
 *     every later call on it returns TQD_ERR_STATE.
 *   - Qubits: logical qubit q in [0, n).  Canonical amplitude index: qubit q is
 *     bit (n-1-q) (MSB-first, reading R1; qubit q is tensor
 *     dimension q of X in C^{2x...x2}, row-major).
 *   - Pauli masks: bit q of x_mask / z_mask <-> logical qubit q;
 *     (x,z) = (0,0) I, (1,0) X, (0,1) Z, (1,1) Y.
 *   - Ownership: handles are library-owned and freed with *_destroy / *_free.
 *     Input arrays are copied and never retained.  Output arrays are
 *     caller-owned HOST memory.  A caller-provided device buffer (dev_buf) stays
 *     owned by the caller and must outlive the state.  The CUDA stream is
 *     borrowed.
 *   - Collectives: tqd_state_init, tqd_expval, tqd_adjoint_grad and
 *     tqd_get_amplitudes are collective over the context's ranks: every rank
 *     calls them in the same order with the same arguments (and records the
 *     same gates).
 *   - Laziness: tqd_apply_gate only records the gate on the state's tape (no
 *     device work, like the deferred MoveDim^{-1} of Alg. 2).
 *     Execution happens in tqd_expval, tqd_adjoint_grad, tqd_get_amplitudes.
 */
#ifndef TQD_ABI_H_
#define TQD_ABI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tqd_ctx tqd_ctx;     /* one per process = one GPU; owns NCCL comm + stream */
typedef struct tqd_state tqd_state; /* sharded state + gate tape + qubit map pi          */

/* Amplitude precision. Complex64 = interleaved float (re, im); complex128 = double. */
typedef enum { TQD_C64 = 0, TQD_C128 = 1 } tqd_dtype;

/* Gate kinds ("universal gate set using single-qubit Pauli rotation
 * gates and the two-qubit CNOT", plus the fixed gates and custom unitaries it
 * allows; north star adds CZ and U3).
 *   1q fixed:  I X Y Z H S SDG T TDG                  (textbook matrices)
 *   2q fixed:  CNOT (wires = [control, target], R3), CZ, SWAP
 *   custom:    MAT1 (2x2), MAT2 (4x4): row-major (re, im) doubles; must be
 *              unitary ("users should take care to ensure they are
 *              unitary"): ||M M^dag - I||_max <= 1e-10 (C128) / 1e-5 (C64)
 *   rotation:  RX RY RZ = exp(-i theta P / 2) (R4), 1 parameter
 *              U3(theta, phi, lambda) = [[c, -e^{il} s], [e^{ip} s, e^{i(p+l)} c]]
 *              (R5), 3 parameters.
 * For 2q gates wires[0] is the more significant bit of the 4x4 index (R2). */
typedef enum {
    TQD_I = 0, TQD_X, TQD_Y, TQD_Z, TQD_H, TQD_S, TQD_SDG, TQD_T, TQD_TDG,
    TQD_CNOT, TQD_CZ, TQD_SWAP,
    TQD_MAT1, TQD_MAT2,
    TQD_RX, TQD_RY, TQD_RZ, TQD_U3,
    TQD_NUM_GATES
} tqd_gate;

enum {
    TQD_OK = 0,
    TQD_ERR_ARG = -1,         /* NULL pointer, bad wire / arity / parameter count / size */
    TQD_ERR_QUBITS = -2,      /* n < log2(world) + 2, n > 62, or shard too large */
    TQD_ERR_WORLD = -3,       /* world not a power of two, rank out of range */
    TQD_ERR_NOT_UNITARY = -4, /* MAT1 / MAT2 fails the unitarity tolerance */
    TQD_ERR_OOM = -5,         /* device allocation failed / dev_buf too small */
    TQD_ERR_CUDA = -6,        /* CUDA runtime error (context poisoned) */
    TQD_ERR_NCCL = -7,        /* NCCL error (context poisoned) */
    TQD_ERR_UNSUPPORTED = -8, /* valid request this build does not implement */
    TQD_ERR_STATE = -9        /* poisoned context, consumed state, wrong call order */
};

/* Options (tqd_state_set_option).  Defaults are tuned for B200. */
typedef enum {
    TQD_OPT_TILE_QUBITS = 0,  /* k: amplitudes per fused-sweep tile = 2^k (9..12; default 12) */
    TQD_OPT_SMALL_MAX = 1,    /* n_loc <= this runs the single-CTA whole-state kernel (default 8:
                               * from 9 local qubits a one-tile fused sweep is faster, e.g.
                               * cfg1 10q c128 fwd+grad 0.29 -> 0.17 ms) */
    TQD_OPT_PROFILE = 2,      /* 1: time every kernel with CUDA events (see tqd_metrics) */
    TQD_OPT_GRID_CTAS = 3,    /* persistent CTAs per launch (0 = auto: SMs x resident CTAs) */
    TQD_OPT_USE_GRAPH = 4,    /* 1: replays of a cached plan (tqd_state_rewind, or a re-recorded
                               * tape of the same structure) launch the forward and reverse
                               * sweep sequences as CUDA graphs (one rank, PROFILE off;
                               * default 0)                                               */
    TQD_OPT_FUSED_REMAP = 5,  /* 1: a FORWARD remap right after a sweep is fused into it: the
                               * sweep stores straight into the owners' lambda buffers over
                               * peer memory (idle until the adjoint seed; allocated on
                               * first use: the with_adjoint budget of tqd_state_bytes) and
                               * the buffers swap roles (default 1); 0: every remap runs
                               * pack -> all-to-all -> unpack through the bounded staging
                               * (always the case for adjoint remaps: psi and lambda live) */
    TQD_OPT_ABSORB_TAIL = 6,  /* 1 (default): tqd_adjoint_grad and tqd_expval with Z-string
                               * terms absorb the circuit's trailing diagonal / permutation
                               * gates (RZ, CZ, CP, X, Y, CNOT, SWAP ...) into the observable by
                               * conjugation (Heisenberg picture, E = <psi|U^dag H U|psi>)
                               * instead of applying (and un-applying) them; same values and
                               * gradients (absorbed trainable gates are diagonal: gradient 0).
                               * After tqd_expval the absorbed gates stay pending: a later
                               * readback / sample / non-Z observable applies them.
                               * 0: apply every gate.                                      */
    TQD_OPT_STAGING_BYTES = 7, /* world > 1: bytes of the exchange staging (send + receive
                               * halves; remap blocks and X/Y partner shards move through it
                               * in chunks).  0 (default) = min(1 GiB, 2 x shard).  Tests
                               * force a few KiB so the chunk loop iterates.               */
    TQD_OPT_PRODUCT_PREFIX = 9, /* 2 (default): auto = 1 from 22 local qubits when the plan of
                               * the remaining gates is cheaper (planner cost model), else 0;
                               * 1: every qubit's leading 1-qubit gates (before its first
                               * entangling gate) act on |0>; fixed 2-qubit gates that keep
                               * the product (SWAP; diagonal or controlled gates with one
                               * qubit in a parameter-independent basis state) join them.  A
                               * state (>= 11 local qubits, any batch and world size) starts
                               * from that product state (one write pass instead of their
                               * sweeps) and the adjoint finishes their gradients from
                               * lambda's environments at the prefix boundary (one read pass);
                               * same values and gradients.  0: sweep every gate.
                               * Other values: TQD_ERR_ARG.                                  */
    TQD_OPT_CIRCUIT_MAX = 8,   /* single-GPU states of <= this many qubits (0..12; default 10)
                               * run tqd_adjoint_grad with Z-string terms as ONE kernel launch:
                               * forward gates, lambda = H psi and the reverse sweep in one
                               * CTA's shared memory per state (0 = staged sweeps only)     */
    TQD_OPT_CIRCUIT_LAYOUT = 10, /* 0 (default): the single launch runs gate by gate (2 amplitudes
                               * per thread, 16 warps); 1 (experiment): for 8..10 local qubits
                               * and circuits of 1-qubit, diagonal, controlled-1-qubit and SWAP
                               * gates, a register-layout kernel (8 amplitudes per thread, 4
                               * warps, layout exchanges through swizzled shared memory;
                               * metric circuit_layout_launches).  Same results; measured
                               * slower (latency-bound at 4 warps). */
} tqd_option;

/* Execution metrics, cumulative since tqd_state_init / tqd_state_reset.
 * Byte counts are ALGORITHMIC (what the method must move, DESIGN.md section
 * "Algorithmic bytes"), not DRAM counters. */
typedef struct tqd_metrics {
    uint64_t fwd_sweeps;        /* fused forward sweep launches                      */
    uint64_t bwd_sweeps;        /* fused adjoint sweep launches                      */
    uint64_t remaps;            /* global<->local qubit remaps (all-to-all rounds)   */
    uint64_t gates_applied;     /* gates applied in forward sweeps                   */
    uint64_t gates_unapplied;   /* gates un-applied in adjoint sweeps                */
    uint64_t hbm_bytes;         /* algorithmic HBM bytes of all kernels              */
    uint64_t a2a_bytes;         /* bytes this rank sent to other ranks               */
    double   fwd_sweep_ms;      /* summed kernel time of forward sweeps (PROFILE=1)  */
    double   bwd_sweep_ms;      /* summed kernel time of adjoint sweeps (PROFILE=1)  */
    double   other_ms;          /* init / expval / lambda-init / gather (PROFILE=1)  */
    double   a2a_ms;            /* remap exchange time (PROFILE=1)                   */
    uint64_t fwd_sweep_bytes;   /* algorithmic bytes of forward sweeps               */
    uint64_t bwd_sweep_bytes;   /* algorithmic bytes of adjoint sweeps               */
    uint64_t peak_device_bytes; /* state buffers + scratch held by this state        */
    uint64_t kernel_launches;   /* library kernels launched                          */
    uint64_t h2d_bytes;         /* host->device bytes (plan descriptors, masks)      */
    uint64_t d2h_bytes;         /* device->host bytes (values, gradients, amplitudes) */
    uint64_t fused_remaps;      /* remaps done by the preceding sweep's peer-memory stores */
    uint64_t plans_reused;      /* executions that reused the plan of a structurally equal tape */
    uint64_t gates_absorbed;    /* trailing gates absorbed into Z observables (TQD_OPT_ABSORB_TAIL) */
    uint64_t gates_prefix;      /* gates written as the product-state prefix (TQD_OPT_PRODUCT_PREFIX;
                                   counted in gates_applied too)                      */
    uint64_t circuit_layout_launches; /* single-launch circuits run by the register-layout kernel */
} tqd_metrics;

/* --- context ------------------------------------------------------------- */

/* Writes a 128-byte NCCL unique id into out128 (call on rank 0, broadcast the
 * bytes to the other ranks by any means, e.g. torch.distributed). */
int tqd_nccl_unique_id(void *out128);

/* Writes a 128-byte LOOPBACK id: a world of W ranks emulated inside one
 * process on one device (test facility for 1-GPU machines).  Every rank calls
 * tqd_ctx_create(W, rank, device, id, ...) from its own host thread; the remap
 * blocks then move by device-to-device copies between the ranks' buffers after
 * host barriers, and sums are reduced on the host in rank order.  No kernel of
 * one rank waits on another rank's kernel.  The device work of every rank (rank-
 * bit conditioned sweeps, remap pack / unpack, sharded reductions, readback) is
 * the same as with NCCL; only the transport differs. */
int tqd_loopback_id(void *out128);

/* Create the per-process context.  world must be a power of two (sharding
 * log2 d qubits over d accelerators, §4.2); 0 <= rank < world.
 * nccl_id: the 128 bytes from tqd_nccl_unique_id or tqd_loopback_id
 * (ignored, may be NULL, iff world == 1).  cuda_stream: a cudaStream_t to run on (borrowed) or NULL for
 * a library-created stream.  Collective over the world when world > 1. */
int tqd_ctx_create(int world, int rank, int cuda_device, const void *nccl_id,
                   void *cuda_stream, tqd_ctx **out);
int tqd_ctx_destroy(tqd_ctx *ctx);

/* --- state --------------------------------------------------------------- */

/* Device bytes per rank for an n-qubit state of dtype dt on `world` ranks:
 * the shard psi (2^{n - log2 world} amplitudes), plus lambda for the adjoint
 * when with_adjoint != 0, plus the bounded exchange staging when world > 1
 * (min(1 GiB, 2 shards); e.g. 36 qubits complex64 on 8 GPUs with the adjoint:
 * 2 x 64 GiB + 1 GiB).  Scratch of a few MiB (descriptors, reductions) is extra.
 * The with_adjoint = 0 figure holds for forward-only work with
 * TQD_OPT_FUSED_REMAP = 0 (fused forward remaps store into the lambda buffer). */
int tqd_state_bytes(int n_qubits, tqd_dtype dt, int world, int with_adjoint, size_t *bytes_per_rank);

/* Allocate and initialise |0...0> (reset_states):
 * amplitude 1 at canonical index 0 on the rank that owns it.  The qubit map
 * pi starts as the identity: logical qubit q at physical bit n-1-q, so logical
 * qubits 0..g-1 (g = log2 world) are the sharded ("global") ones.
 * dev_buf: NULL = the library allocates; else a device buffer of buf_bytes
 * >= tqd_state_bytes(..., with_adjoint=1) that the library carves up.
 * Errors: TQD_ERR_QUBITS when n > 62, or (world > 1) n < g + 2 (PAPER.md:162
 * "at least two unsharded dimensions"); TQD_ERR_OOM.  Collective. */
int tqd_state_init(tqd_ctx *ctx, int n_qubits, tqd_dtype dt, void *dev_buf, size_t buf_bytes,
                   tqd_state **out);
/* A BATCH of `batch` states of n qubits that share one gate tape (PAPER.md:157:
 * the first tensor dimension is the batch; the paper's profiled workload is a
 * batch of 16 states whose encoder angles differ).  Every state
 * starts in |0...0>.  Gates recorded with tqd_apply_gate act identically on all
 * states (one gradient slot per parameter: the gradient is the sum over the
 * batch); tqd_apply_gate_batch records per-state parameters.  Outputs index the
 * batch first: tqd_expval writes out[b * n_terms + t]; tqd_get_amplitudes reads
 * the index space [0, batch * 2^n) as b * 2^n + i; tqd_adjoint_grad takes
 * coeff[b * n_terms + t] (NULL = all 1) and returns E = sum_b sum_t c_bt <P_t>_b.
 * Memory: batch x the single-state buffers.  Collective. */
int tqd_state_init_batch(tqd_ctx *ctx, int n_qubits, tqd_dtype dt, int batch, tqd_state **out);

/* Back to |0...0>, empty tape, pi = identity.  Collective (device memset). */
int tqd_state_reset(tqd_state *st);
/* Back to |0...0> and pi = identity but KEEP the recorded tape: the next
 * tqd_expval / tqd_adjoint_grad re-executes the same circuit with the plan and
 * device descriptors already resident (no re-planning, no upload).  For
 * repeated evaluation of one circuit (benchmarks, optimisers that re-record
 * only when parameters change).  Collective. */
int tqd_state_rewind(tqd_state *st);
int tqd_state_free(tqd_state *st);
int tqd_state_set_option(tqd_state *st, int option, int64_t value);

/* Record gate g on `wires` (n_wires = 1 or 2, distinct, < n).  params: 0, 1 or
 * 3 angles (NULL iff 0).  matrix: MAT1 2x2 / MAT2 4x4 row-major (re, im)
 * doubles, NULL otherwise.  trainable != 0 gives each angle a gradient slot in
 * recording order.  No device work (lazy).  Errors: TQD_ERR_ARG,
 * TQD_ERR_NOT_UNITARY, TQD_ERR_STATE (state consumed by tqd_adjoint_grad). */
int tqd_apply_gate(tqd_state *st, tqd_gate g, const int *wires, int n_wires,
                   const double *params, const double *matrix, int trainable);

/* Record G gates at once, in order, exactly as G tqd_apply_gate calls would
 * (same validation, same gradient slots), from host parallel arrays (caller
 * owned, read during the call only): kinds[G] (tqd_gate), wires[2G] (second
 * entry ignored for 1-qubit kinds), params[3G] (first gate_num_params used),
 * mats[32G] (MAT1 2x2 / MAT2 4x4 row-major re,im; ignored for other kinds),
 * trainable[G].  One call per circuit instead of one per gate (the circuit
 * building of Listing 1, recorded lazily).  All-or-nothing: on error no
 * gate is recorded.  G = 0 is a no-op.  Errors: as tqd_apply_gate. */
int tqd_apply_circuit(tqd_state *st, int G, const int *kinds, const int *wires, const double *params,
                      const double *mats, const int *trainable);

/* Record a parameterised 1-qubit gate (RX, RY, RZ or U3) with PER-STATE
 * parameters: params[b * np + i] for batch element b (np = 1, or 3 for U3), e.g.
 * the encoder rotation carrying each state's input.  trainable != 0 gives the
 * gate batch * np gradient slots, element b's at slot0 + b * np + i (the input
 * gradients of Adam-on-inputs).  Errors: TQD_ERR_ARG for another
 * kind, n_wires != 1, NULL params. */
int tqd_apply_gate_batch(tqd_state *st, tqd_gate g, const int *wires, int n_wires, const double *params,
                         int trainable);

/* Shape of a state: qubits, batch size (1 for tqd_state_init) and dtype
 * (tqd_dtype); NULL outputs are skipped.  Bindings size the caller-owned arrays
 * of tqd_expval / tqd_adjoint_grad / tqd_apply_gate_batch from it (the ABI takes
 * no array lengths). */
int tqd_state_info(const tqd_state *st, int *n_qubits, int *batch, int *dtype);

/* Number of gradient slots recorded so far. */
int tqd_num_params(const tqd_state *st, int *out);

/* Execute pending gates, then out[t] = c_t <psi|P_t|psi> (
 * measure_allZ), c_t = 1 when coeff is NULL.  Pauli string
 * t: X on the qubits of x_mask[t], Z on z_mask[t], Y where both bits are set
 * (bit q = logical qubit q).  A term whose X/Y part touches sharded qubits pairs
 * this shard with the partner rank's (rank XOR those rank bits): one whole-shard
 * exchange per distinct such x mask.  Collective. */
int tqd_expval(tqd_state *st, int n_terms, const uint64_t *x_mask, const uint64_t *z_mask,
               const double *coeff, double *out);

/* Execute pending gates, then E = sum_t c_t <psi|P_t|psi> and
 * out_grad[p] = dE/dtheta_p for every gradient slot p (n_grad must equal
 * tqd_num_params), by the invertible reverse sweep of PAPER.md:220-236 (§4.4):
 * lambda = H psi, then per gate in reverse: g += 2 Re <lambda|(dU)U^dag|psi>,
 * psi <- U^dag psi (x = U^* y), lambda <- U^dag lambda
 * (dx = U^T dy in the real representation, Eq. save_x).
 * This is the VJP of any loss of the expectation values (choose c_t = dL/dE_t,
 * e.g. sign(E_t) for Listing 2's out.abs().sum()).
 * General Pauli strings (as tqd_expval), at most 64 terms: Z strings seed
 * lambda in one pass; X / Y strings add c_t P_t psi per x mask (with the partner
 * rank's shard when the x mask has rank bits).
 * CONSUMES the state: afterwards only tqd_state_reset / tqd_state_free /
 * tqd_get_metrics are allowed.  Collective. */
int tqd_adjoint_grad(tqd_state *st, int n_terms, const uint64_t *x_mask, const uint64_t *z_mask,
                     const double *coeff, double *out_value, double *out_grad, int n_grad);

/* Shot noise, exact sampler: `shots` measurements of all
 * qubits.  out[b * shots + k] = the canonical outcome (basis index, MSB-first) of
 * shot k of batch element b, identical on every rank.  Hierarchical multinomial:
 * the groups are the ranks' shards; every rank learns the groups' masses q_j (one
 * small all-reduce), draws the same uniforms u_k = uniform(seed + b, k) (counter-
 * based, R22), assigns shot k to group j (y ~ Multinomial(shots, q)) and
 * samples the outcomes of its own shots conditionally from its shard (inverse CDF
 * over chunk masses, then inside the chunk on the device).  at most 2^32 shots.
 * Collective. */
int tqd_sample(tqd_state *st, uint64_t shots, uint64_t seed, uint64_t *out);

/* Shot noise, approximate sampler: the multinomial sample of
 * `shots` measurements of all qubits is replaced by its Gaussian limit
 * y = shots p + sqrt(shots) D S z over the 2^n canonical outcomes (D = diag sqrt p,
 * S the Householder reflection mapping e_K <-> sqrt p, K = 2^n - 1; reading R21),
 * with z_i = normal(seed + b, i) from the counter-based generator of DESIGN.md
 * §8c (splitmix64 + Box-Muller, indexed by the canonical outcome i, so the result
 * does not depend on the sharding).  out[b * n + q] = (1/shots) sum_i y_i (-1)^{q
 * bit of i}: the noisy <Z_q> estimate of measure_allZ(shots).
 * y is never materialised: the estimates follow from O(n) global sums.
 * Collective. */
int tqd_sample_gaussian_z(tqd_state *st, double shots, uint64_t seed, double *out);

/* The differentiable (reparameterised) counterpart: value
 * L = sum_b sum_q coeff[b * n + q] Zhat_{b,q} (coeff NULL = all 1) with the same
 * z as tqd_sample_gaussian_z(seed), and out_grad[p] = dL/dtheta_p by the adjoint
 * sweep seeded with lambda = dL/dpsi*.  CONSUMES the state.  Collective. */
int tqd_adjoint_grad_gaussian(tqd_state *st, double shots, uint64_t seed, const double *coeff, double *out_value,
                              double *out_grad, int n_grad);

/* Execute pending gates and copy amplitudes [first, first+count) in CANONICAL
 * order (MoveDim^{-1} of PAPER.md:116-119 applied through pi) to host_out
 * (count complex values of the state's dtype, interleaved re, im).  Every rank
 * receives the values.  Collective. */
int tqd_get_amplitudes(tqd_state *st, uint64_t first, uint64_t count, void *host_out);

int tqd_get_metrics(const tqd_state *st, tqd_metrics *out);
int tqd_reset_metrics(tqd_state *st);

/* Message of the calling thread's last error ("" if none). */
const char *tqd_last_error(void);

/* Library build string (arch, CUDA / NCCL versions). */
const char *tqd_version(void);

/* Diagnostic, host only (no GPU, no device work): run the planner on a circuit
 * and write its stages (tile bits, layouts, ops, remaps, qubit map pi before /
 * after each stage) as JSON into json_out (cap bytes, NUL-terminated).
 * Circuit as parallel arrays of length G: kinds[G] (tqd_gate), wires[2G],
 * params[3G], mats[32G] (MAT1/MAT2 row-major re,im), trainable[G].
 * k: tile qubits; small_max: as TQD_OPT_SMALL_MAX; c128: dtype flag.
 * *needed receives the JSON size + 1.  TQD_ERR_ARG if cap is too small. */
int tqd_debug_plan(int n, int world, int k, int small_max, int c128, int G, const int *kinds, const int *wires,
                   const double *params, const double *mats, const int *trainable, char *json_out, size_t cap,
                   size_t *needed);

/* Diagnostic, host only (no GPU): the observable absorption that
 * tqd_adjoint_grad applies with TQD_OPT_ABSORB_TAIL (Heisenberg picture,
 * E = <psi|U^dag H U|psi>; PAPER.md:226-231 seed, PAPER.md:308 Z observables).
 * Circuit as in tqd_debug_plan; T Z-string masks z_in[T] (bit q = logical
 * qubit q).  Writes the first absorbed gate index to *tail_begin (G if none),
 * the conjugated masks z_out[T] and signs sign_out[T] (+1 / -1): then
 * sum_t c_t <Z_{z_in[t]}> after all G gates equals
 * sum_t c_t sign_out[t] <Z_{z_out[t]}> after gates [0, *tail_begin).
 * TQD_ERR_ARG on bad sizes or NULL pointers; caller-owned arrays. */
int tqd_debug_absorb(int n, int G, const int *kinds, const int *wires, const double *params, const double *mats,
                     const int *trainable, int T, const uint64_t *z_in, uint64_t *z_out, double *sign_out,
                     int *tail_begin);

/* Diagnostic, host only: one rank's remap exchange schedule (PAPER.md:164, 261:
 * interchange global qubit positions gpos[0..m) with local positions
 * lpos[0..m) and redistribute).  Rank `rank` packs its local amplitudes into
 * 2^m blocks by the values of the lpos-bits (block b, remaining local bits in
 * ascending position order inside a block); block b goes to rank peer_out[b];
 * the block received from that peer is unpacked as block recv_block_out[b]
 * (its values become the lpos-bits).  Arrays of 2^m ints, caller-owned. */
int tqd_debug_remap_schedule(int rank, int n_loc, int m, const int *gpos, const int *lpos, int *peer_out,
                             int *recv_block_out);

/* Experiment (PAPER.md:91 custom unitaries): apply a dense
 * 2^m x 2^m complex unitary U (row-major (re, im) doubles, m = 6) to the m LOWEST
 * bits of a 2^n-amplitude complex64 state (13 <= n <= 33) on the tensor cores:
 * tcgen05.mma kind::tf32 with TMEM accumulators, precision = 3 (3xTF32 split,
 * fp32-level accuracy) or 1 (plain TF32).  Canonical index i = row * 2^m + c, the
 * block acts on c.  psi_in / psi_out: host complex64 arrays of 2^n (NULL: zeros /
 * no readback).  Then `iters` more applications are timed with CUDA events:
 * *ms_out = average ms per application.  Allocates its own device buffers on
 * `device`; not part of the circuit path.  Errors: TQD_ERR_ARG, TQD_ERR_OOM,
 * TQD_ERR_CUDA. */
int tqd_debug_dense_block(int device, int n, int m, int precision, const double *U, const void *psi_in, void *psi_out,
                          int iters, double *ms_out);

#ifdef __cplusplus
}
#endif
#endif /* TQD_ABI_H_ */
