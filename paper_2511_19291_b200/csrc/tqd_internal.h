// tqd_internal.h -- descriptors shared by the host planner and the sm_100a kernels.
//
// A circuit is executed as a list of STAGES (Alg. 2 + §4.2 in
// B200 form):
//   SWEEP  one fused pass over the local shard.  The shard is cut into tiles of
//          2^k amplitudes: the k "tile-local" bits t = 0..k-1 sit at physical
//          positions ld_phys[t] (t = 0..4 are always physical bits 0..4 so that
//          one warp instruction reads one 256 B run).  Inside a CTA the tile is
//          distributed as   lanes (5 bits) x warps (W bits) x registers (R bits).
//          A LAYOUT says which tile-local bit each lane / warp / register bit
//          holds.  Gates run on register bits only (their targets); controls and
//          diagonal gates may sit on any bit.  Between segments the CTA changes
//          layout through shared memory (one STS + one LDS per amplitude).  The
//          store may move tile bits to other tile positions (st_phys), which is
//          how the qubit map pi changes for free.
//   SMALL  the whole local shard in one CTA's shared memory (n_loc small);
//          gate-by-gate, one launch for a whole run of local gates.
//   REMAP  exchange of global (rank) qubit positions with local positions over
//          NCCL ("interchanging qubit positions" +
//          "redistribute across devices", the NCCL all-to-all).
#pragma once
#include <stdint.h>

namespace tqd {

constexpr int KMAX = 16;    // max tile bits
constexpr int RMAX = 5;     // max register bits
constexpr int WMAX = 4;     // max warp bits (16 warps = 512 threads)
#ifndef TQD_SWEEP_R
#define TQD_SWEEP_R 4  // register bits per thread in the sweep kernels (experiment knob)
#endif
constexpr int LANE_BITS = 5;
constexpr int MAXSEG = 8;   // layouts per sweep stage
constexpr int NAFF = 8;     // base-controlled affine terms per exchange
constexpr int MAX_STAGE_OPS = 128;   // placed gates per sweep stage (bounds the kernel-op table in shared memory)
constexpr int MAX_STAGE_SLOTS = 32;   // gradient slots per stage (per-thread fp32 accumulators in shared memory)

enum OpKind : uint8_t {
    OP_NONE = 0,
    OP_U1 = 1,  // general complex 2x2 on register bit t0 (optional control)
    OP_R1 = 2,  // real 2x2 on register bit t0 (RY, H, ...) (optional control)
    OP_P1 = 3,  // [[0, a], [b, 0]] on register bit t0 (X, Y, CNOT's target) (optional control)
    OP_D1 = 4,  // diag(d0, d1) on bit b0 (any bit) (optional control)
    OP_U2 = 5,  // general complex 4x4 on register bits (t0 = MSB, t1)
    OP_D2 = 6,  // diag(d00, d01, d10, d11) on bits (b0 = MSB, b1)
};

enum BitKind : uint8_t {
    BK_NONE = 0,
    BK_REG = 1,   // register bit idx of the current layout
    BK_TIX = 2,   // tile-local bit idx held by a lane or warp bit (per-thread constant)
    BK_BASE = 3,  // physical position idx outside the tile (incl. global = rank bits)
};

enum GenKind : uint8_t {
    GEN_NONE = 0,
    GEN_X = 1,     // G = -(i/2) X   (RX)
    GEN_Y = 2,     // G = -(i/2) Y   (RY)
    GEN_Z = 3,     // G = -(i/2) Z   (RZ, on a D1 op)
    GEN_FULL = 4,  // G = (dU/dtheta) U^dag, general 2x2 (U3)
};

struct BitRef {
    uint8_t kind;
    uint8_t idx;
};

// One gate in device form.  Matrices are float64; float kernels convert on use.
// For backward ops the matrix is already U^dagger and g[] holds the generators
// G_p = (dU/dtheta_p) U^dag of the ORIGINAL gate.
struct alignas(16) DevOp {
    uint8_t kind;       // OpKind
    uint8_t t0, t1;     // SWEEP: register-bit indices; SMALL: physical positions
    uint8_t ngen;       // generators (gradient slots) carried by this op
    BitRef ctrl;        // control bit (must be 1) or BK_NONE
    BitRef b0, b1;      // D1 / D2 bits
    uint8_t gkind[3];   // GenKind per generator
    uint8_t pad0[5];
    int32_t slot[3];    // SWEEP: stage-local slot; SMALL: global parameter index
    int32_t pad1;
    double m[32];       // U1: 4 complex; R1: 4 real; P1: a, b; D1: d0, d1; U2: 16 complex; D2: 4 complex
    double g[3][8];     // generator matrices (2x2 complex, row-major re,im)
};

// ---- sweep-kernel ops (v2): what the fused sweep kernel executes, staged in
// shared memory in the kernel's precision.  Consecutive single-qubit gates on
// register bits are fused into one K_LAYER op (one 2x2 per register bit, the
// mask is a compile-time dispatch), so the runtime dispatch cost is paid once
// per layer, not once per gate.
enum KKind : uint8_t {
    K_NOP = 0,
    K_LAYER = 1,  // per active register bit b: 2x2 m[8b..8b+7] (type ltype)
    K_CX = 2,     // X on register bit t0 (CNOT target), control creg / ctrl
    K_CU = 3,     // general 2x2 on register bit t0, control creg / ctrl
    K_PHASE = 4,  // diag(d0, d1) selected by a lane/warp/base bit b0 (+ RZ generator)
    K_D2 = 5,     // diag 2q on bits b0 (MSB), b1 (any kind)
    K_U2 = 6,     // 4x4 on register bits t0 (MSB), t1
    K_DBLK = 7,   // merged run of diagonal gates: phase polynomial (see DTerm)
};
enum LType : uint8_t { LT_GEN = 0, LT_REAL = 1, LT_DIAG = 2 };
constexpr int KOP_MAXGEN = 4;

// dense dispatch codes: one flat switch (jump table) in the kernel
enum KCode : uint8_t {
    KC_NOP = 0,
    KC_REAL = 0,    // KC_REAL + mask (1..15): real 2x2 per active register bit
    KC_GEN = 15,    // KC_GEN + mask (16..30): complex 2x2 per active register bit
    KC_DIAG = 31,   // 16-phase table
    KC_CU = 32,     // KC_CU + t0 (32..35)
    KC_PHASE = 36,
    KC_D2 = 37,
    KC_U2 = 38,     // KC_U2 + u2_index(t0, t1) (38..49)
    KC_DBLK = 50,   // diagonal block: applies the run ending here
    KC_DDATA = 51,  // diagonal block: more terms of the run (no work when dispatched)
    KC_COUNT = 52,
};

// Diagonal block (K_DBLK): a run of diagonal gates (CP, CZ, Z / S / T / RZ on
// non-register bits, diagonal MAT1 / MAT2) is one phase function of the index
// bits, exp(i Phi(b)) with Phi a quadratic polynomial over GF(2) bits.  The part
// that depends only on the register bits is a uniform 16-entry table (m[], as a
// diagonal layer); the rest is a list of terms in g[] (t0 = count, <= DBLK_TERMS):
//   a = REG bit r, b = lane/warp/base bit X (or none): Phi += ang * r * X
//   a, b both lane/warp/base bits (b may be none):    Phi += ang * A * B
// Angles are fixed-point fractions of a full turn (2^32 / 2^64 = 2 pi), so sums
// wrap exactly mod 2 pi; the kernel turns the per-thread sums into phases with
// sincospi.  gbits = register bits that carry cross terms.
constexpr int DBLK_TERMS = 16;
// A run is zero or more KC_DDATA kops followed by the applying KC_DBLK kop; the
// run's terms are ordered [C | U | M] across its kops (per kop: nC, nU, nM):
//   C: lane / warp bits only (no base bit): per-thread constants, summed once per
//      kernel into a per-thread table (rows c_off.., DevStage::n_cvals rows);
//   U: base bits only (no lane / warp bit): uniform over the CTA per tile, summed
//      once per tile by one thread per value into u_acc (rows u_off..);
//   M: lane / warp x base products: summed by every thread per tile.
// The run's C rows / U values: 1 + popc(xm): th, then al[b] for b in xm.
constexpr int DBLK_CCAP_F32 = 16;  // per-thread C rows per adjoint stage (shared memory: rows x threads x 4 B)
constexpr int DBLK_CCAP_F64 = 4;   // (x 8 B); both <= 16 KB at 256 threads; forward stages: 3x
constexpr int DBLK_UCAP = 64;      // per-tile U values per stage
template <typename Real> struct DTerm;
template <> struct DTerm<float> {
    uint32_t ang;
    BitRef a, b;
};
template <> struct DTerm<double> {
    uint64_t ang;
    BitRef a, b;
    uint8_t pad[4];
};
inline int u2_index(int t0, int t1) { return t0 * 3 + (t1 > t0 ? t1 - 1 : t1); }

// The first 16 bytes are the dispatch header (prefetched one op ahead).
template <typename Real> struct alignas(16) KOp {
    uint8_t code;               // KCode
    uint8_t ngen;               // backward: generators (gradient slots)
    uint8_t creg;               // register-bit control, 0xff = none
    uint8_t t0;                 // K_CU target register bit
    uint8_t gbits;              // generator register bits, 2 bits each
    uint8_t gmask;              // layer fast path: register bits carrying the layer's own generator
                                // (real layer: -(i/2) Y per bit, diagonal layer: -(i/2) Z per bit)
    BitRef ctrl;                // lane / warp / base control, BK_NONE = none
    BitRef b0, b1;              // K_PHASE / K_D2 bits
    uint16_t gkinds;            // GenKind of each generator, 4 bits each
    uint8_t kind, ltype;        // host / debug only
    int16_t slot[KOP_MAXGEN];   // stage-local slot
    uint8_t mask, t1;           // host / debug only
    uint8_t gbit[KOP_MAXGEN];   // host view of gbits
    uint8_t gkind[KOP_MAXGEN];  // host view of gkinds
    uint16_t soff[KOP_MAXGEN];  // gradient accumulator offsets slot * threads; indexed by register
                                // bit when gmask != 0, else by generator
    uint8_t pad1[6];
    Real m[64];                 // 16-byte aligned (offset 48); complex entries as (re, 0, im, im)
    Real g[KOP_MAXGEN][8];      // generators (2x2 complex)
};

struct DevLayout {
    uint8_t reg[RMAX];
    uint8_t lane[LANE_BITS];
    uint8_t warp[WMAX];
    uint8_t pad[1];
};

struct DevStage {
    int32_t k, R, W, nseg;
    int64_t n_tiles;
    uint8_t ld_phys[KMAX];      // physical position of tile-local bit t at load
    uint8_t st_phys[KMAX];      // physical position of tile-local bit t at store
    uint8_t tile_sorted[KMAX];  // the tile's physical positions, ascending
    uint32_t swz[KMAX];         // shared-memory address vector of tile-local bit t (plain layouts)
    // exchange s (segment s -> s+1): shared-memory address vectors of tile-local
    // bit t on the write side (layout s) and the read side (layout s+1); the
    // permutation gates of the stage (CNOT, X) are folded into these maps
    uint32_t wcol[MAXSEG][KMAX];
    uint32_t rcol[MAXSEG][KMAX];
    uint32_t wcst[MAXSEG], rcst[MAXSEG];
    uint8_t naff[MAXSEG];
    uint8_t aff_read[MAXSEG];   // 1: affine terms apply to the read side
    uint8_t aff_pos[MAXSEG][NAFF];
    uint32_t aff_vec[MAXSEG][NAFF];
    uint8_t xsync[MAXSEG];      // exchange x: bits 0..3 = warp-index bits kept (write -> read sync only
                                // among warps sharing them), bit 7 = the sync after its reads may be __syncwarp
    int32_t seg_begin[MAXSEG + 1];
    DevLayout lay[MAXSEG];
    int32_t op_base, n_ops;     // into the launch's DevOp array
    int32_t slot_base, n_slots; // into the launch's slot -> parameter table
    int32_t lam_init;           // backward only: 1 = build lambda = H psi on load
    int32_t flags;              // kernel variant bits (SWF_*)
    int32_t batch;              // states in the batch: op / slot tables repeat per state (n_ops, n_slots each)
    int32_t no_store;           // backward only, last reverse stage: 1 = psi / lambda not needed afterwards,
                                // 2 = lambda only (product prefix: its environments give gradients)
    int32_t n_cvals, n_uvals;   // diagonal blocks: per-thread C rows, per-tile U values (see DTerm)
    int32_t n_dblk;             // applying diagonal-block kops in the stage
};

// sweep-kernel variant bits (DevStage::flags)
enum : int32_t { SWF_NONE = 0 };  // 4: timing only (wrong results)

// Fused sweep -> remap (PAPER.md:164 redistribution fused into the preceding sweep):
// the sweep's store writes every amplitude straight to its post-remap owner and
// position, through peer memory (NVLink P2P / CUDA IPC; the loopback world: same
// device).  Full index P -> P' = P with bits gbit[i] <-> lbit[i] swapped; rank
// P' >> n_loc, offset P' & lmask.  m = 0: plain in-place store.
constexpr int SCATTER_MAX_RANKS = 64;
struct ScatterInfo {
    int32_t m;
    int32_t n_loc;
    uint8_t gbit[8];  // full-index positions (>= n_loc) of the swapped rank bits
    uint8_t lbit[8];  // local positions they swap with
    uint64_t dst_psi[SCATTER_MAX_RANKS];  // destination shard of psi on every rank
    uint64_t dst_lam[SCATTER_MAX_RANKS];  // (adjoint) destination shard of lambda
};

// Z-string observable in PHYSICAL masks (full index incl. rank bits)
// lambda-init form: h(b) = cst - 2 sum_p w[p] bit_p(b) + sum_t c_t (-1)^{popc(b & z_t)}
// (single-qubit Z terms folded into per-position weights, the rest listed)
// ---- single-launch layout circuit (circuit_l3_kernel, 8..10 local qubits) --------
// The whole state in registers: 8 amplitudes per thread (3 register bits, then 5
// lane bits and n_loc - 8 warp bits = the thread index bits).  A LAYOUT assigns a
// physical bit to every slot (0..2 register, 3.. thread bit slot-3).  Gates run on
// register slots (diagonal gates and controls on any slot); an exchange (L3_X)
// moves to a new layout through XOR-swizzled shared memory: amplitude with physical
// index x is stored at S(x) = (x & ~low) | F(x), F linear with F|low invertible,
// chosen per exchange so that both layouts' lane bits hit distinct banks
// (abi.cpp encode_l3).  Exchange row e: per thread xtab[e][tid] = S(thread part of
// the old layout) | S(thread part of the new layout) << 16, uniform
// xreg[e][0..7] = S(register part r, old), [8..15] = S(register part r, new);
// rows 0 / 1: the plain (unswizzled) initial / seed layouts.
enum L3Type : uint8_t { L3_U1 = 1, L3_D1 = 2, L3_D2 = 3, L3_X = 4 };
enum L3Form : uint8_t { L3F_GEN = 0, L3F_REAL = 1, L3F_SWAP = 2 };
struct alignas(16) L3Op {
    uint8_t type, j, ck, ci;      // U1: target register slot; control kind (0 none, 1 register slot, 2 thread bit), index
    uint8_t d0k, d0i, d1k, d1i;   // D1 / D2 bits: kind (1 register slot, 2 thread bit), index (d0 = MSB of the D2 index)
    uint8_t ngen, form;           // adjoint generators; U1 form (L3Form)
    uint16_t xi;                  // X: exchange row
    uint8_t gk[3], pad0;          // GenKind per generator
    uint16_t acc[3], gi;          // per generator: accumulator; GEN_FULL: gtab row of generator p = gi + p
    uint32_t pad1[2];
    double m[8];                  // U1: 2x2 complex row-major (re, im); D1: d0, d1; D2: d00, d01, d10, d11
};

struct ZTerms {
    int T;
    uint64_t z[64];
    double c[64];
    double w[64];
    double cst;
};

// canonical index -> physical index through pi (readback)
struct GatherMap {
    int n, n_loc;
    uint64_t rank;
    uint8_t phys_of_canon_bit[64];  // canonical bit b -> physical position
};

}  // namespace tqd
