// plan.h -- host-side gate tape + fusion / remap planner (no CUDA dependency).
//
// This is the bookkeeping layer of PAPER.md §4.1-4.2 done B200-first: instead
// of physically moving tensor dimensions (MoveDim, Alg. 1) the planner keeps a
// qubit map pi (logical qubit -> physical bit position, the "second tensor
// [that] keeps track of exactly how the qubits are arranged") and
// groups consecutive gates into fused SWEEP stages whose tiles contain the
// gates' target bits.  Gates whose target is a sharded (global) qubit trigger a
// REMAP stage that interchanges global and local positions.
#pragma once
#include <complex>
#include <cstdint>
#include <string>
#include <vector>

#include "tqd_internal.h"

namespace tqd {

typedef std::complex<double> cd;

enum GateClass {
    CL_IDENT = 0,  // identity: dropped
    CL_DIAG1,      // diagonal 1q (Z S T RZ, diagonal MAT1)
    CL_DIAG2,      // diagonal 2q (CZ, diagonal MAT2 e.g. CP)
    CL_U1,         // non-diagonal 1q
    CL_CTRL1,      // controlled 1q: control w[0], target w[1] (CNOT, controlled MAT2)
    CL_U2,         // general 2q
    CL_SWAP,       // SWAP: relabel of pi, no device work
};

struct GateRec {
    int kind = 0;
    int nw = 1;
    int w[2] = {0, 0};   // CL_CTRL1: [control, target]
    int ow[2] = {0, 0};  // wires as recorded
    double p[3] = {0, 0, 0};
    cd M[16];          // gate matrix (2x2 or 4x4 row-major)
    int trainable = 0;
    int slot0 = -1;    // first gradient slot (recording order) or -1
    int cls = CL_IDENT;
    cd sub[4];         // CL_CTRL1: the 2x2 applied to the target when control = 1
    int ngen = 0;
    uint8_t gkind[3] = {0, 0, 0};
    cd G[3][4];        // generators (dU/dtheta_p) U^dag
    // batched gate (per-state parameters in a batch of states, e.g. encoder inputs):
    // structure decided by the kind alone so that every batch element encodes to the
    // same kernel ops; the tape holds element 0, the state keeps all B records
    int batched = 0;
};

// build matrix, class and generators; returns 0 or a TQD_ERR_* code
int make_gate(int kind, const int *wires, int n_wires, const double *params, const double *matrix, int trainable,
              bool c128, GateRec &out, std::string &err);
int gate_num_params(int kind);
int gate_arity(int kind);

// op before device encoding: physical positions resolved at placement time
struct POp {
    int gate = -1;
    int kind = OP_NONE;
    int tp0 = -1, tp1 = -1;  // target positions (register bits needed)
    int cp = -1;             // control position
    int dp0 = -1, dp1 = -1;  // diagonal bit positions
    cd m[16];                // forward matrix in op form (see DevOp)
    int plain = 0;           // OP_P1: plain swap
    int seg = 0;             // sweep segment
    int wp0 = -1, wp1 = -1;  // diagnostics: positions of the gate's wires[0], wires[1] at placement
    int perm = 0;            // 1: CNOT / X on a tile bit, realised as an index map (no arithmetic)
};

// GF(2)-affine map on tile-local indices accumulated from the permutation gates
// (CNOT, X) of one segment: x -> A x + c + sum_j [bit p_j of the full index] v_j
struct TileMap {
    uint32_t col[KMAX];               // A e_t
    uint32_t cst = 0;                 // c
    std::vector<std::pair<int, uint32_t>> aff;  // (physical position p_j outside the tile, v_j)
    bool identity() const;
};

struct Layout {
    int reg[RMAX];
    int lane[LANE_BITS];
    int warp[WMAX];
};

struct SweepPlan {
    int k = 0, R = 0, W = 0;
    std::vector<int> ld_phys, st_phys;  // per tile-local bit
    std::vector<Layout> lays;
    std::vector<int> seg_begin;         // size lays+1
    std::vector<POp> ops;               // in execution order, seg ascending
    std::vector<uint32_t> swz;
    std::vector<TileMap> maps;          // per segment: permutation gates applied after its ops
    std::vector<uint8_t> xwarp;         // per exchange s -> s+1: 1 = warp-local (same warp bits, map keeps them)
    std::vector<uint8_t> xumask;        // per exchange: warp-index bits kept (groups of 2^(W - popc) warps)
    std::vector<uint32_t> perm_tgt;     // per segment: tile bits targeted by its permutation gates
    int n_gates = 0;                    // gates applied (incl. relabels / identities)
    int n_arith = 0;                    // ops needing arithmetic (kernel launch needed if > 0 or maps)
};

struct SmallPlan {
    std::vector<POp> ops;
    int n_gates = 0;
};

struct RemapPlan {
    int m = 0;
    int gpos[8];  // global physical positions
    int lpos[8];  // local physical positions they swap with
};

enum StageType { ST_SWEEP = 0, ST_SMALL = 1, ST_REMAP = 2 };

struct Stage {
    int type = ST_SWEEP;
    SweepPlan sw;
    SmallPlan sm;
    RemapPlan rm;
    std::vector<int> pos_before, pos_after;  // pi around the stage
};

struct PlanConfig {
    int n = 0, n_loc = 0;
    int k = 12;        // tile bits
    int R = 4;         // register bits
    int small_max = 10;
    bool c128 = false;
    int swz_bits = 4;  // shared-memory conflict-free bits (4 for 8 B elems, 3 for 16 B)
    int c_low = 4;     // physical bits 0..c_low-1 pinned in every tile (2^c_low-amplitude runs)
    int max_ops = MAX_STAGE_OPS;      // per sweep stage (shared-memory budget of the kernel)
    int max_slots = MAX_STAGE_SLOTS;  // gradient slots per sweep stage
    int seg_min_gates = -1;  // trailing-segment trim (plan_sweep); -1: plan_circuit tries the default and 0
};

// Plan the gates `pending` (indices into gates, in recording order) starting
// from qubit map pos (logical -> physical).  Appends stages, updates pos.
uint64_t plan_signature(const std::vector<GateRec> &gates, const PlanConfig &cfg);
void refresh_plan_values(std::vector<Stage> &stages, const std::vector<GateRec> &gates);
int plan_circuit(const std::vector<GateRec> &gates, std::vector<int> pending, std::vector<int> &pos,
                 const PlanConfig &cfg, std::vector<Stage> &out, std::string &err);
// estimated cost of a stage list in 30-q sweep pairs (sweeps + 0.24 per layout
// exchange + 2 per remap)
double plan_cost(const std::vector<Stage> &stages);

// Encode a sweep stage into device descriptors (forward or backward order).
template <typename Real>
// skip_below (backward only): gates with a smaller tape index precede every
// trainable gate; their (non-permutation) ops are left out of the reverse sweep
void encode_sweep_k(const SweepPlan &sp, const std::vector<GateRec> &gates, bool bwd, int n_loc, DevStage &ds,
                    std::vector<KOp<Real>> &ops, std::vector<int32_t> &slot_param, int skip_below = 0);
void encode_small(const SmallPlan &sp, const std::vector<GateRec> &gates, bool bwd, std::vector<DevOp> &ops,
                  int skip_below = 0);

std::string plan_to_json(const std::vector<Stage> &stages, const PlanConfig &cfg);

}  // namespace tqd
