// plan.cpp -- gate records, fusion planner and device encoding (host only).
//
// See plan.h.  The planner's choices never change results, only the layout and
// the number of HBM sweeps / exchanges.
#include "plan.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <cstdlib>
#include <sstream>

#include "../../include/tqd.h"

namespace tqd {

static const cd I1(0.0, 1.0);

int gate_num_params(int kind) {
    switch (kind) {
    case TQD_RX: case TQD_RY: case TQD_RZ: return 1;
    case TQD_U3: return 3;
    default: return 0;
    }
}

int gate_arity(int kind) {
    switch (kind) {
    case TQD_CNOT: case TQD_CZ: case TQD_SWAP: case TQD_MAT2: return 2;
    default: return 1;
    }
}

// Textbook matrices (readings R2-R5).
static void base_matrix(int kind, const double *p, const double *mat, cd *M) {
    for (int i = 0; i < 16; i++) M[i] = 0.0;
    const double r2 = 1.0 / std::sqrt(2.0);
    double c, s;
    switch (kind) {
    case TQD_I: M[0] = 1; M[3] = 1; break;
    case TQD_X: M[1] = 1; M[2] = 1; break;
    case TQD_Y: M[1] = -I1; M[2] = I1; break;
    case TQD_Z: M[0] = 1; M[3] = -1; break;
    case TQD_H: M[0] = r2; M[1] = r2; M[2] = r2; M[3] = -r2; break;
    case TQD_S: M[0] = 1; M[3] = I1; break;
    case TQD_SDG: M[0] = 1; M[3] = -I1; break;
    case TQD_T: M[0] = 1; M[3] = std::polar(1.0, M_PI / 4); break;
    case TQD_TDG: M[0] = 1; M[3] = std::polar(1.0, -M_PI / 4); break;
    case TQD_RX: c = std::cos(p[0] / 2); s = std::sin(p[0] / 2);
        M[0] = c; M[1] = -I1 * s; M[2] = -I1 * s; M[3] = c; break;
    case TQD_RY: c = std::cos(p[0] / 2); s = std::sin(p[0] / 2);
        M[0] = c; M[1] = -s; M[2] = s; M[3] = c; break;
    case TQD_RZ: M[0] = std::polar(1.0, -p[0] / 2); M[3] = std::polar(1.0, p[0] / 2); break;
    case TQD_U3: c = std::cos(p[0] / 2); s = std::sin(p[0] / 2);
        M[0] = c; M[1] = -std::polar(1.0, p[2]) * s; M[2] = std::polar(1.0, p[1]) * s;
        M[3] = std::polar(1.0, p[1] + p[2]) * c; break;
    case TQD_CNOT: M[0] = 1; M[5] = 1; M[11] = 1; M[14] = 1; break;
    case TQD_CZ: M[0] = 1; M[5] = 1; M[10] = 1; M[15] = -1; break;
    case TQD_SWAP: M[0] = 1; M[6] = 1; M[9] = 1; M[15] = 1; break;
    case TQD_MAT1: for (int i = 0; i < 4; i++) M[i] = cd(mat[2 * i], mat[2 * i + 1]); break;
    case TQD_MAT2: for (int i = 0; i < 16; i++) M[i] = cd(mat[2 * i], mat[2 * i + 1]); break;
    default: break;
    }
}

// dU/dtheta_which for the parametric kinds
static void dmatrix(int kind, const double *p, int which, cd *D) {
    for (int i = 0; i < 4; i++) D[i] = 0.0;
    double c, s;
    switch (kind) {
    case TQD_RX: c = std::cos(p[0] / 2); s = std::sin(p[0] / 2);
        D[0] = -s / 2; D[1] = -I1 * c / 2.0; D[2] = -I1 * c / 2.0; D[3] = -s / 2; break;
    case TQD_RY: c = std::cos(p[0] / 2); s = std::sin(p[0] / 2);
        D[0] = -s / 2; D[1] = -c / 2; D[2] = c / 2; D[3] = -s / 2; break;
    case TQD_RZ: D[0] = -I1 / 2.0 * std::polar(1.0, -p[0] / 2); D[3] = I1 / 2.0 * std::polar(1.0, p[0] / 2); break;
    case TQD_U3: c = std::cos(p[0] / 2); s = std::sin(p[0] / 2);
        if (which == 0) {
            D[0] = -s / 2; D[1] = -std::polar(1.0, p[2]) * c / 2.0; D[2] = std::polar(1.0, p[1]) * c / 2.0;
            D[3] = -std::polar(1.0, p[1] + p[2]) * s / 2.0;
        } else if (which == 1) {
            D[2] = I1 * std::polar(1.0, p[1]) * s; D[3] = I1 * std::polar(1.0, p[1] + p[2]) * c;
        } else {
            D[1] = -I1 * std::polar(1.0, p[2]) * s; D[3] = I1 * std::polar(1.0, p[1] + p[2]) * c;
        }
        break;
    default: break;
    }
}

static bool is_zero(cd z) { return z.real() == 0.0 && z.imag() == 0.0; }
static bool is_one(cd z) { return z.real() == 1.0 && z.imag() == 0.0; }

int make_gate(int kind, const int *wires, int n_wires, const double *params, const double *matrix, int trainable,
              bool c128, GateRec &g, std::string &err) {
    if (kind < 0 || kind >= TQD_NUM_GATES) { err = "unknown gate kind"; return TQD_ERR_ARG; }
    if (n_wires != gate_arity(kind)) { err = "wrong number of wires for gate"; return TQD_ERR_ARG; }
    if (!wires) { err = "wires is NULL"; return TQD_ERR_ARG; }
    const int np = gate_num_params(kind);
    if (np > 0 && !params) { err = "params is NULL for a parametric gate"; return TQD_ERR_ARG; }
    if ((kind == TQD_MAT1 || kind == TQD_MAT2) && !matrix) { err = "matrix is NULL for MAT1/MAT2"; return TQD_ERR_ARG; }
    g = GateRec();
    g.kind = kind;
    g.nw = n_wires;
    for (int i = 0; i < n_wires; i++) g.w[i] = g.ow[i] = wires[i];
    for (int i = 0; i < np; i++) {
        g.p[i] = params[i];
        if (!std::isfinite(params[i])) { err = "non-finite gate parameter"; return TQD_ERR_ARG; }
    }
    base_matrix(kind, g.p, matrix, g.M);
    const int dim = n_wires == 2 ? 4 : 2;
    if (kind == TQD_MAT1 || kind == TQD_MAT2) {
        double worst = 0;
        for (int r = 0; r < dim; r++)
            for (int c = 0; c < dim; c++) {
                cd acc = 0;
                for (int q = 0; q < dim; q++) acc += g.M[dim * r + q] * std::conj(g.M[dim * c + q]);
                if (r == c) acc -= 1.0;
                if (!std::isfinite(acc.real()) || !std::isfinite(acc.imag())) worst = 1e300;
                worst = std::max(worst, std::abs(acc));
            }
        const double tol = c128 ? 1e-10 : 1e-5;
        if (worst > tol) {
            err = "custom matrix is not unitary (||M M^dag - I||_max = " + std::to_string(worst) + ")";
            return TQD_ERR_NOT_UNITARY;
        }
    }
    g.trainable = (trainable && np > 0) ? 1 : 0;

    // class
    if (g.trainable) {
        g.cls = kind == TQD_RZ ? CL_DIAG1 : CL_U1;
    } else if (dim == 2) {
        bool diag = is_zero(g.M[1]) && is_zero(g.M[2]);
        if (diag && is_one(g.M[0]) && is_one(g.M[3])) g.cls = CL_IDENT;
        else g.cls = diag ? CL_DIAG1 : CL_U1;
    } else if (kind == TQD_SWAP) {
        g.cls = CL_SWAP;
    } else {
        bool diag = true;
        for (int r = 0; r < 4; r++)
            for (int c = 0; c < 4; c++)
                if (r != c && !is_zero(g.M[4 * r + c])) diag = false;
        bool ident = diag;
        for (int r = 0; r < 4; r++) if (!is_one(g.M[5 * r])) ident = false;
        if (ident) g.cls = CL_IDENT;
        else if (diag) g.cls = CL_DIAG2;
        else {
            // controlled on wires[0]: block diag(I, U) in the (w0 MSB) basis
            bool c0 = is_one(g.M[0]) && is_one(g.M[5]) && is_zero(g.M[1]) && is_zero(g.M[4]);
            for (int r = 0; r < 2 && c0; r++)
                for (int c = 2; c < 4; c++)
                    if (!is_zero(g.M[4 * r + c]) || !is_zero(g.M[4 * c + r])) c0 = false;
            // controlled on wires[1]: indices {0,2} identity, {1,3} carry U
            bool c1 = is_one(g.M[0]) && is_one(g.M[10]) && is_zero(g.M[2]) && is_zero(g.M[8]);
            for (int r : {0, 2})
                for (int c : {1, 3})
                    if (!is_zero(g.M[4 * r + c]) || !is_zero(g.M[4 * c + r])) c1 = false;
            if (c0) {
                g.cls = CL_CTRL1;
                g.sub[0] = g.M[10]; g.sub[1] = g.M[11]; g.sub[2] = g.M[14]; g.sub[3] = g.M[15];
            } else if (c1) {
                g.cls = CL_CTRL1;
                g.sub[0] = g.M[5]; g.sub[1] = g.M[7]; g.sub[2] = g.M[13]; g.sub[3] = g.M[15];
                std::swap(g.w[0], g.w[1]);  // store as [control, target]
            } else {
                g.cls = CL_U2;
            }
        }
    }

    // generators G_p = (dU/dtheta_p) U^dag (anti-Hermitian)
    if (g.trainable) {
        g.ngen = np;
        for (int i = 0; i < np; i++) {
            cd D[4];
            dmatrix(kind, g.p, i, D);
            for (int r = 0; r < 2; r++)
                for (int c = 0; c < 2; c++) {
                    cd acc = 0;
                    for (int q = 0; q < 2; q++) acc += D[2 * r + q] * std::conj(g.M[2 * c + q]);
                    g.G[i][2 * r + c] = acc;
                }
            g.gkind[i] = kind == TQD_RX ? GEN_X : kind == TQD_RY ? GEN_Y : kind == TQD_RZ ? GEN_Z : GEN_FULL;
        }
    }
    return TQD_OK;
}

// ---------------------------------------------------------------------------
// planning helpers

// logical wires with roles: targets (need register residency = non-diagonal
// action) and diagonal wires (controls, diagonal gates)
static void roles(const GateRec &g, int *tq, int &ntq, int *dq, int &ndq) {
    ntq = ndq = 0;
    switch (g.cls) {
    case CL_U1: tq[ntq++] = g.w[0]; break;
    case CL_CTRL1: tq[ntq++] = g.w[1]; dq[ndq++] = g.w[0]; break;
    case CL_U2: tq[ntq++] = g.w[0]; tq[ntq++] = g.w[1]; break;
    case CL_DIAG1: dq[ndq++] = g.w[0]; break;
    case CL_DIAG2: dq[ndq++] = g.w[0]; dq[ndq++] = g.w[1]; break;
    case CL_SWAP: tq[ntq++] = g.w[0]; tq[ntq++] = g.w[1]; break;  // roles only; relabel, no residency
    default: break;
    }
}

static bool real_mat(const cd *m, int n) {
    for (int i = 0; i < n; i++) if (m[i].imag() != 0.0) return false;
    return true;
}

// op form of a 1q matrix (trainable / batched gates: by kind, so it never depends on values)
static int op1_form(const cd *m, int trainable_kind, int &plain) {
    plain = 0;
    if (trainable_kind == TQD_RX || trainable_kind == TQD_U3) return OP_U1;
    if (trainable_kind == TQD_RY) return OP_R1;
    if (is_zero(m[0]) && is_zero(m[3])) {
        plain = is_one(m[1]) && is_one(m[2]);
        return OP_P1;
    }
    return real_mat(m, 4) ? OP_R1 : OP_U1;
}

// Build the op (physical positions) for a placed gate.
static POp make_pop(const GateRec &g, int gi, const std::vector<int> &pos) {
    POp o;
    o.gate = gi;
    o.wp0 = pos[g.ow[0]];
    if (g.nw == 2) o.wp1 = pos[g.ow[1]];
    auto set1 = [&](const cd *m, int trainable_kind) {
        for (int i = 0; i < 4; i++) o.m[i] = m[i];
        o.kind = op1_form(m, trainable_kind, o.plain);
    };
    switch (g.cls) {
    case CL_U1:
        o.tp0 = pos[g.w[0]];
        set1(g.M, (g.trainable || g.batched) ? g.kind : -1);
        break;
    case CL_CTRL1:
        o.tp0 = pos[g.w[1]];
        o.cp = pos[g.w[0]];
        set1(g.sub, -1);
        break;
    case CL_U2:
        o.kind = OP_U2;
        o.tp0 = pos[g.w[0]];
        o.tp1 = pos[g.w[1]];
        for (int i = 0; i < 16; i++) o.m[i] = g.M[i];
        break;
    case CL_DIAG1:
        o.kind = OP_D1;
        o.dp0 = pos[g.w[0]];
        o.m[0] = g.M[0];
        o.m[1] = g.M[3];
        break;
    case CL_DIAG2:
        o.kind = OP_D2;
        o.dp0 = pos[g.w[0]];
        o.dp1 = pos[g.w[1]];
        for (int i = 0; i < 4; i++) o.m[i] = g.M[5 * i];
        break;
    default:
        o.kind = OP_NONE;
        break;
    }
    return o;
}

struct Item {      // placed gate (op or relabel) during sweep planning
    int gate;
    POp op;        // kind OP_NONE for relabel / identity
    int relabel_a = -1, relabel_b = -1;  // physical positions swapped (SWAP relabel)
    std::vector<int> npos;  // positions touched non-diagonally
    std::vector<int> dpos;  // positions touched diagonally
    std::vector<int> need;  // tile-local bits that must be register-resident
};

static int next_target_use(const std::vector<GateRec> &gates, const std::vector<int> &rest, int q) {
    for (size_t i = 0; i < rest.size(); i++) {
        const GateRec &g = gates[rest[i]];
        int tq[2], dq[2], nt, nd;
        roles(g, tq, nt, dq, nd);
        if (g.cls == CL_SWAP) continue;
        for (int j = 0; j < nt; j++)
            if (tq[j] == q) return (int)i;
    }
    return 1 << 30;
}

static int gf2_rank(std::vector<uint32_t> v) {
    int r = 0;
    for (int bit = 31; bit >= 0; bit--) {
        int piv = -1;
        for (size_t i = r; i < v.size(); i++)
            if ((v[i] >> bit) & 1) { piv = (int)i; break; }
        if (piv < 0) continue;
        std::swap(v[r], v[piv]);
        for (size_t i = 0; i < v.size(); i++)
            if ((int)i != r && ((v[i] >> bit) & 1)) v[i] ^= v[r];
        r++;
    }
    return r;
}

bool TileMap::identity() const {
    if (cst || !aff.empty()) return false;
    for (int t = 0; t < KMAX; t++)
        if (col[t] != (1u << t)) return false;
    return true;
}

static TileMap identity_map() {
    TileMap m;
    for (int t = 0; t < KMAX; t++) m.col[t] = 1u << t;
    return m;
}

// x_t ^= x_c (or ^= 1, or ^= a bit outside the tile), composed after m
static void map_apply_perm(TileMap &m, int t, int c_tile, int c_pos) {
    auto tr = [&](uint32_t v) { return (c_tile >= 0 && ((v >> c_tile) & 1)) ? v ^ (1u << t) : v; };
    for (int j = 0; j < KMAX; j++) m.col[j] = tr(m.col[j]);
    m.cst = tr(m.cst);
    for (auto &a : m.aff) a.second = tr(a.second);
    if (c_tile < 0) {
        if (c_pos < 0) {
            m.cst ^= 1u << t;
        } else {
            bool found = false;
            for (auto &a : m.aff)
                if (a.first == c_pos) { a.second ^= 1u << t; found = true; }
            if (!found) m.aff.push_back({c_pos, 1u << t});
        }
    }
}

static uint32_t lin(const uint32_t *cols, uint32_t v) {
    uint32_t r = 0;
    for (int t = 0; v; t++, v >>= 1)
        if (v & 1) r ^= cols[t];
    return r;
}

// Shared-memory swizzle: address(y) = y ^ F(y's high bits) in the low SW bits.
// Chosen so that, for every exchange, the lane bits 0..SW-1 of the write and of
// the read side hit distinct banks (SW = 4 for 8 B elements, 3 for 16 B).
static std::vector<uint32_t> choose_swizzle(int k, int SW, const std::vector<std::vector<uint32_t>> &sets) {
    std::vector<uint32_t> best(k), cur(k);
    int best_ok = -1;
    uint64_t rng = 0x9E3779B97F4A7C15ull;
    auto next = [&]() { rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17; return rng; };
    for (int trial = 0; trial < 4000; trial++) {
        for (int t = 0; t < k; t++) {
            uint32_t f = 0;
            if (t >= SW && trial > 0) f = (uint32_t)(next() & ((1u << SW) - 1));
            cur[t] = (1u << t) ^ f;
        }
        int ok = 0;
        for (const auto &set : sets) {
            std::vector<uint32_t> v;
            for (uint32_t y : set) v.push_back(lin(cur.data(), y) & ((1u << SW) - 1));
            if (gf2_rank(v) == SW) ok++;
        }
        if (ok > best_ok) { best_ok = ok; best = cur; }
        if (ok == (int)sets.size()) break;
    }
    return best;
}

// Dry run of the next stage's placement (phase 1 of plan_sweep, logical qubits):
// how many gates it would place if `lanes` (logical qubits) sit at physical bits
// 0..4.  Used to choose which qubits a stage leaves on the always-resident bits.
static int simulate_next_stage(const std::vector<GateRec> &gates, const std::vector<int> &remaining,
                               const std::vector<int> &pos, int n_loc, int k, const int *lanes, int nl, int max_items) {
    const int n = (int)pos.size();
    std::vector<char> in_tile(n, 0), blocked(n, 0);
    int tsize = 0;
    for (int i = 0; i < nl; i++) { in_tile[lanes[i]] = 1; tsize++; }
    int placed = 0, scanned = 0;
    for (int gi : remaining) {
        if (++scanned > 4 * n + 64) break;
        const GateRec &g = gates[gi];
        bool blk = false;
        for (int j = 0; j < g.nw; j++) if (blocked[g.w[j]]) blk = true;
        int tq[2], dq[2], nt, nd;
        roles(g, tq, nt, dq, nd);
        int add[2], na = 0;
        if (!blk && g.cls != CL_SWAP)
            for (int j = 0; j < nt && !blk; j++) {
                const int qq = tq[j];
                if (pos[qq] >= n_loc) blk = true;
                else if (!in_tile[qq]) add[na++] = qq;
            }
        if (!blk && tsize + na > k) blk = true;
        if (blk) {
            for (int j = 0; j < g.nw; j++) blocked[g.w[j]] = 1;
            continue;
        }
        for (int j = 0; j < na; j++) { in_tile[add[j]] = 1; tsize++; }
        if (++placed >= max_items) break;
    }
    return placed;
}

// Plan one fused sweep stage.  Returns false if nothing could be placed.
static bool plan_sweep(const std::vector<GateRec> &gates, std::vector<int> &pending, std::vector<int> &pos,
                       const PlanConfig &cfg, Stage &st) {
    const int n = cfg.n, n_loc = cfg.n_loc;
    const int k = std::min(cfg.k, n_loc);
    const int R = cfg.R;
    const int W = k - LANE_BITS - R;
    if (W < 0 || W > WMAX) return false;

    std::vector<int> tile_of(n_loc, -1), tphys;
    const int C = cfg.c_low;  // physical bits 0..C-1 are in every tile (contiguous 2^C-amplitude runs)
    for (int p = 0; p < C; p++) { tile_of[p] = p; tphys.push_back(p); }
    std::vector<char> blocked(n, 0);
    std::vector<int> wpos = pos;               // working map (relabels)
    std::vector<int> wlq(n);
    for (int q = 0; q < n; q++) wlq[wpos[q]] = q;
    std::vector<Item> items;
    std::vector<int> rest;
    int n_nondiag = 0, n_slots = 0;
    const int cap_nondiag = R * (MAXSEG - 2);
    // kernel-op budget of the stage (cfg.max_ops, shared memory): every op-emitting
    // item costs <= 1 kop plus <= 1 for the diagonal-block run it may split; merged
    // diagonal gates (no targets, no gradient) cost <= 3 terms of DBLK_TERMS per
    // K_DBLK; + one run per segment
    int n_kop_items = 0, n_diag_merge = 0;
    auto kop_estimate = [&](int items_, int diag_) { return 2 * items_ + MAXSEG + (3 * diag_ + DBLK_TERMS - 1) / DBLK_TERMS; };
    std::vector<int> aff_pos;  // distinct control positions outside the tile of folded CNOTs

    for (size_t ii = 0; ii < pending.size(); ii++) {
        const int gi = pending[ii];
        const GateRec &g = gates[gi];
        bool blk = false;
        for (int j = 0; j < g.nw; j++)
            if (blocked[g.w[j]]) blk = true;
        int tq[2], dq[2], nt, nd;
        roles(g, tq, nt, dq, nd);
        const bool merge_diag = g.cls != CL_SWAP && nt == 0 && g.ngen == 0;
        if (!blk && g.cls != CL_SWAP &&
            kop_estimate(n_kop_items + (merge_diag ? 0 : 1), n_diag_merge + (merge_diag ? 1 : 0)) > cfg.max_ops - 1)
            blk = true;
        if (!blk && n_slots + g.ngen > cfg.max_slots) blk = true;
        std::vector<int> newbits;
        if (!blk && g.cls != CL_SWAP && nt > 0) {
            if (n_nondiag >= cap_nondiag) blk = true;
            for (int j = 0; j < nt && !blk; j++) {
                const int p = wpos[tq[j]];
                if (p >= n_loc) { blk = true; break; }
                if (tile_of[p] < 0 && std::find(newbits.begin(), newbits.end(), p) == newbits.end()) newbits.push_back(p);
            }
            if (!blk && (int)(tphys.size() + newbits.size()) > k) blk = true;
        }
        if (blk) {
            for (int j = 0; j < g.nw; j++) blocked[g.w[j]] = 1;
            rest.push_back(gi);
            continue;
        }
        for (int p : newbits) { tile_of[p] = (int)tphys.size(); tphys.push_back(p); }
        Item it;
        it.gate = gi;
        if (g.cls == CL_SWAP) {
            const int a = wpos[g.w[0]], b = wpos[g.w[1]];
            it.relabel_a = a;
            it.relabel_b = b;
            it.npos = {a, b};
            std::swap(wpos[g.w[0]], wpos[g.w[1]]);
            wlq[wpos[g.w[0]]] = g.w[0];
            wlq[wpos[g.w[1]]] = g.w[1];
        } else {
            it.op = make_pop(g, gi, wpos);
            for (int j = 0; j < nt; j++) it.npos.push_back(wpos[tq[j]]);
            for (int j = 0; j < nd; j++) it.dpos.push_back(wpos[dq[j]]);
            // X / CNOT with the target in the tile: a GF(2)-affine index map,
            // folded into the next layout change (no register residency needed)
            if (it.op.kind == OP_P1 && it.op.plain && !g.trainable) {
                const int cpos = it.op.cp;
                const bool outside = cpos >= 0 && (cpos >= n_loc || tile_of[cpos] < 0);
                if (!outside) it.op.perm = 1;
                else if (std::count(aff_pos.begin(), aff_pos.end(), cpos) || (int)aff_pos.size() < NAFF) {
                    it.op.perm = 1;
                    if (!std::count(aff_pos.begin(), aff_pos.end(), cpos)) aff_pos.push_back(cpos);
                }
            }
            if (merge_diag) n_diag_merge++;
            else if (!it.op.perm) n_kop_items++;
            if (!it.op.perm)
                for (int j = 0; j < nt; j++) it.need.push_back(tile_of[wpos[tq[j]]]);
            if (nt && !it.op.perm) n_nondiag++;
            n_slots += g.ngen;
        }
        items.push_back(it);
    }
    if (items.empty()) return false;

    // fill the tile to k bits
    for (int p = 0; p < n_loc && (int)tphys.size() < k; p++)
        if (tile_of[p] < 0) { tile_of[p] = (int)tphys.size(); tphys.push_back(p); }

    // ---- list scheduling into register layouts (segments) ----
    const int m = (int)items.size();
    auto is_perm = [&](int i) { return items[i].op.perm != 0; };
    std::vector<std::vector<int>> succ(m);
    std::vector<int> indeg(m, 0), ready_seg(m, 0);
    for (int j = 0; j < m; j++)
        for (int i = 0; i < j; i++) {
            bool conflict = false;
            for (int p : items[j].npos) {
                if (std::count(items[i].npos.begin(), items[i].npos.end(), p) ||
                    std::count(items[i].dpos.begin(), items[i].dpos.end(), p)) conflict = true;
            }
            for (int p : items[j].dpos)
                if (std::count(items[i].npos.begin(), items[i].npos.end(), p)) conflict = true;
            if (conflict) { succ[i].push_back(j); indeg[j]++; }
        }
    std::vector<char> done(m, 0);
    std::vector<int> order, seg_of(m, -1);
    std::vector<std::vector<int>> segregs(1);
    auto subset = [](const std::vector<int> &a, const std::vector<int> &b) {
        for (int x : a) if (!std::count(b.begin(), b.end(), x)) return false;
        return true;
    };
    // segments per stage: every layout change moves psi (and lambda) through shared
    // memory (~1.4 ms per forward / ~3.5 ms per adjoint exchange at
    // 30 qubits); TQD_PLAN_MAX_SEGS caps them (experiment knob, default MAXSEG)
    static const int env_segs = [] {
        const char *e = getenv("TQD_PLAN_MAX_SEGS");
        return e ? std::max(2, std::min(MAXSEG, atoi(e))) : MAXSEG;
    }();
    const int max_segs = env_segs;
    int nseg = 1;
    while ((int)order.size() < m) {
        const int cs = nseg - 1;
        std::vector<int> &cur = segregs[cs];
        auto eligible = [&](int i) { return !done[i] && indeg[i] == 0 && ready_seg[i] <= cs; };
        int pick = -1;
        // permutation gates first (free), then ops whose targets are already resident
        for (int i = 0; i < m && pick < 0; i++)
            if (eligible(i) && is_perm(i)) pick = i;
        for (int i = 0; i < m && pick < 0; i++)
            if (eligible(i) && subset(items[i].need, cur)) pick = i;
        if (pick < 0) {
            for (int i = 0; i < m && pick < 0; i++) {
                if (!eligible(i)) continue;
                std::vector<int> u = cur;
                bool ok = true;
                for (int x : items[i].need) {
                    if (cs == 0 && x < C) ok = false;
                    if (!std::count(u.begin(), u.end(), x)) u.push_back(x);
                }
                if (ok && (int)u.size() <= R) { cur = u; pick = i; }
            }
        }
        if (pick < 0) {
            if (nseg >= max_segs) break;
            segregs.push_back({});
            nseg++;
            continue;
        }
        done[pick] = 1;
        order.push_back(pick);
        seg_of[pick] = cs;
        for (int j : succ[pick]) {
            indeg[j]--;
            const int rs = (is_perm(pick) && !is_perm(j)) ? cs + 1 : cs;
            ready_seg[j] = std::max(ready_seg[j], rs);
        }
    }
    // drop empty trailing segments
    auto last_used = [&]() {
        int ls = 0;
        for (int i : order) ls = std::max(ls, seg_of[i]);
        return ls;
    };
    // a layout change costs a fixed share of the sweep (~1.4 ms per
    // forward and ~3.5 ms per adjoint exchange at 30 qubits, a whole sweep pair
    // ~13.7 ms for ~24 gates): a trailing segment beyond the third that carries
    // fewer than seg_min_gates gates is cheaper as part of the next stage.  Its items
    // are last in dependency order, so handing them back keeps the rest closed.
    {
        static const int seg_min_default = [] {  // measured: 6 -> 1029 vs 1058 ms per cfg-3 step
            const char *e = getenv("TQD_PLAN_SEG_MIN_GATES");
            return e ? atoi(e) : 6;
        }();
        const int seg_min_gates = cfg.seg_min_gates >= 0 ? cfg.seg_min_gates : seg_min_default;
        static const int seg_keep = [] {  // segments always kept (experiment knob)
            const char *e = getenv("TQD_PLAN_SEG_KEEP");
            return e ? std::max(1, atoi(e)) : 3;
        }();
        for (;;) {
            const int ls = last_used();
            if (ls < seg_keep || seg_min_gates <= 0) break;
            int cnt = 0;
            for (int i : order) if (seg_of[i] == ls) cnt++;
            if (cnt >= seg_min_gates) break;
            std::vector<int> keep;
            for (int i : order) {
                if (seg_of[i] == ls) { done[i] = 0; seg_of[i] = -1; }
                else keep.push_back(i);
            }
            order = keep;
        }
    }
    // permutation gates left in the last segment would need a final map at the
    // store (uncoalesced): hand them back to the next stage, unless the stage
    // has nothing else (then a trailing empty segment realises them)
    {
        const int ls = last_used();
        bool any_arith = false;
        for (int i : order) if (!is_perm(i)) any_arith = true;
        if (any_arith) {
            std::vector<int> keep;
            for (int i : order) {
                if (is_perm(i) && seg_of[i] == ls) { done[i] = 0; seg_of[i] = -1; }
                else keep.push_back(i);
            }
            order = keep;
            nseg = last_used() + 1;
        } else {
            nseg = std::max(2, last_used() + 2);
            if (nseg > MAXSEG) nseg = MAXSEG;
        }
        while ((int)segregs.size() < nseg) segregs.push_back({});
        segregs.resize(nseg);
    }

    // items not scheduled go back to pending (closed under successors)
    std::vector<int> dropped;
    for (int i = 0; i < m; i++)
        if (!done[i]) dropped.push_back(items[i].gate);

    // final qubit map after the kept relabels
    std::vector<int> fpos = pos;
    for (int oi : order) {
        const Item &it = items[oi];
        if (it.relabel_a >= 0) {
            int qa = -1, qb = -1;
            for (int q = 0; q < n; q++) {
                if (fpos[q] == it.relabel_a) qa = q;
                if (fpos[q] == it.relabel_b) qb = q;
            }
            std::swap(fpos[qa], fpos[qb]);
        }
    }

    // remaining gates (dropped + blocked), in recording order
    std::vector<int> remaining = rest;
    remaining.insert(remaining.end(), dropped.begin(), dropped.end());
    std::sort(remaining.begin(), remaining.end());

    // ---- layouts ----
    SweepPlan &sp = st.sw;
    sp.k = k; sp.R = R; sp.W = W;
    sp.ld_phys = tphys;
    sp.lays.assign(nseg, Layout());
    std::vector<int> fl(n_loc, -1);  // logical qubit at physical position after relabels
    for (int q = 0; q < n; q++) if (fpos[q] < n_loc) fl[fpos[q]] = q;
    // register bits of every layout
    std::vector<std::vector<int>> regs_of(nseg);
    for (int s = 0; s < nseg; s++) {
        std::vector<int> regs = segregs[s];
        for (int t = 0; t < k && (int)regs.size() < R; t++) {
            if (s == 0 && t < C) continue;
            if (!std::count(regs.begin(), regs.end(), t)) regs.push_back(t);
        }
        regs_of[s] = regs;
    }
    auto others_of = [&](int s) {
        std::vector<int> o;
        for (int t = 0; t < k; t++) if (!std::count(regs_of[s].begin(), regs_of[s].end(), t)) o.push_back(t);
        return o;
    };
    // lanes 0..C-1 hold the pinned low bits at load (layout 0) and the bits that
    // land on physical 0..C-1 at store (last layout): choose the latter so that the
    // NEXT stage places the most gates (dry run over all C-subsets of the free bits);
    // with one segment the pinned bits stay put
    std::vector<int> last_pin, last_pref;  // pinned lanes of the last layout, then preferred order
    {
        const int s = nseg - 1;
        std::vector<std::pair<long long, int>> cand;
        for (int t : others_of(s)) {
            if (nseg == 1 && t < C) continue;
            const int q = fl[tphys[t]];
            cand.push_back({(long long)next_target_use(gates, remaining, q), t});
        }
        std::sort(cand.begin(), cand.end());
        if (nseg == 1) {
            for (int t = 0; t < C; t++) last_pin.push_back(t);
        } else {
            const int no = (int)cand.size();
            std::vector<int> best_pick;
            int best = -1;
            for (int m = 0; m < (1 << no); m++) {
                if (__builtin_popcount(m) != C) continue;
                int lqc[LANE_BITS], c = 0;
                std::vector<int> pick;
                for (int i = 0; i < no; i++)
                    if ((m >> i) & 1) { lqc[c++] = fl[tphys[cand[i].second]]; pick.push_back(i); }
                const int sc = simulate_next_stage(gates, remaining, fpos, n_loc, k, lqc, C, cfg.max_ops - 1);
                if (sc > best) { best = sc; best_pick = pick; }
            }
            for (int i : best_pick) last_pin.push_back(cand[i].second);
            for (size_t i = 0; i < cand.size(); i++)
                if (!std::count(best_pick.begin(), best_pick.end(), (int)i)) last_pref.push_back(cand[i].second);
        }
    }
    // Warp bits per layout, chosen so that as many layout changes as possible keep
    // the SAME warp bits: such an exchange moves data only inside each warp
    // (__syncwarp instead of a CTA barrier).  Exchange s is
    // warp-local iff W_s == W_{s+1} and no permutation gate of segment s targets a
    // warp bit (its map then preserves the warp bits).  Dynamic programme over the
    // layouts; candidates = W-subsets of the non-register, non-pinned bits.
    std::vector<uint32_t> perm_tgt(nseg, 0);
    for (int oi : order)
        if (is_perm(oi) && seg_of[oi] >= 0 && tile_of[items[oi].op.tp0] >= 0)
            perm_tgt[seg_of[oi]] |= 1u << tile_of[items[oi].op.tp0];
    std::vector<std::vector<uint32_t>> wc(nseg);
    for (int s = 0; s < nseg; s++) {
        uint32_t avail = 0;
        for (int t : others_of(s)) avail |= 1u << t;
        if (s == 0) avail &= ~((1u << C) - 1);
        if (s == nseg - 1) for (int t : last_pin) avail &= ~(1u << t);
        for (uint32_t m = 0; m < (1u << k); m++)
            if ((m & ~avail) == 0 && __builtin_popcount(m) == W) wc[s].push_back(m);
        if (wc[s].empty()) wc[s].push_back(0);  // unreachable for W <= k - R - 5
    }
    std::vector<std::vector<int>> cost(nseg), from(nseg);
    for (int s = 0; s < nseg; s++) {
        cost[s].assign(wc[s].size(), 0);
        from[s].assign(wc[s].size(), 0);
        if (s == 0) continue;
        for (size_t b = 0; b < wc[s].size(); b++) {
            int bc = 1 << 30, bf = 0;
            for (size_t a = 0; a < wc[s - 1].size(); a++) {
                // warp bits kept by the layout change (and by its permutation map):
                // the exchange then splits into independent groups of 2^(W - kept) warps
                const int kept = __builtin_popcount(wc[s - 1][a] & wc[s][b] & ~perm_tgt[s - 1]);
                const int c = cost[s - 1][a] + (W - kept);
                if (c < bc) { bc = c; bf = (int)a; }
            }
            cost[s][b] = bc;
            from[s][b] = bf;
        }
    }
    std::vector<uint32_t> wsel(nseg, 0);
    {
        int b = 0;
        for (size_t i = 1; i < cost[nseg - 1].size(); i++)
            if (cost[nseg - 1][i] < cost[nseg - 1][b]) b = (int)i;
        for (int s = nseg - 1; s >= 0; s--) {
            wsel[s] = wc[s][b];
            b = from[s][b];
        }
    }
    std::vector<int> prev_warps;
    for (int s = 0; s < nseg; s++) {
        const std::vector<int> &regs = regs_of[s];
        std::vector<int> warps, lanes;
        // warp order: bits shared with the previous layout keep their warp-index position
        if (s == 0) {
            for (int t = 0; t < k; t++) if ((wsel[s] >> t) & 1) warps.push_back(t);
        } else {
            warps.assign(W, -1);
            for (int i = 0; i < W; i++)
                if ((wsel[s] >> prev_warps[i]) & 1) warps[i] = prev_warps[i];
            for (int t = 0; t < k; t++) {
                if (!((wsel[s] >> t) & 1) || std::count(warps.begin(), warps.end(), t)) continue;
                for (int i = 0; i < W; i++) if (warps[i] < 0) { warps[i] = t; break; }
            }
        }
        prev_warps = warps;
        if (s == 0) for (int t = 0; t < C; t++) lanes.push_back(t);
        if (s == nseg - 1 && s != 0) lanes = last_pin;
        if (s == nseg - 1 && s != 0)
            for (int t : last_pref)
                if ((int)lanes.size() < LANE_BITS && !((wsel[s] >> t) & 1)) lanes.push_back(t);
        for (int t : others_of(s))
            if ((int)lanes.size() < LANE_BITS && !((wsel[s] >> t) & 1) && !std::count(lanes.begin(), lanes.end(), t))
                lanes.push_back(t);
        Layout &L = sp.lays[s];
        for (int i = 0; i < R; i++) L.reg[i] = regs[i];
        for (int i = 0; i < LANE_BITS; i++) L.lane[i] = lanes[i];
        for (int i = 0; i < WMAX; i++) L.warp[i] = i < W ? warps[i] : 0;
    }
    // per exchange: warp-index bits kept (same tile bit at the same warp position,
    // not a permutation target of the segment) -> independent warp groups
    sp.perm_tgt = perm_tgt;
    sp.xumask.assign(nseg, 0);
    sp.xwarp.assign(nseg, 0);
    for (int s = 0; s + 1 < nseg; s++) {
        uint8_t um = 0;
        for (int i = 0; i < W; i++)
            if (sp.lays[s].warp[i] == sp.lays[s + 1].warp[i] && !((perm_tgt[s] >> sp.lays[s].warp[i]) & 1)) um |= 1 << i;
        sp.xumask[s] = um;
        sp.xwarp[s] = um == (1 << W) - 1 ? 1 : 0;
    }
    // output permutation sigma: last layout's lanes land on physical 0..4
    sp.st_phys.assign(k, -1);
    {
        const Layout &L = sp.lays[nseg - 1];
        std::vector<char> used(n_loc, 0);
        for (int i = 0; i < C; i++) { sp.st_phys[L.lane[i]] = i; used[i] = 1; }
        std::vector<int> freep;
        for (int t = C; t < k; t++) {
            bool moved = sp.st_phys[t] >= 0;
            if (!moved) { sp.st_phys[t] = tphys[t]; used[tphys[t]] = 1; }
        }
        for (int t = C; t < k; t++) if (!used[tphys[t]]) freep.push_back(tphys[t]);
        size_t fi = 0;
        for (int t = 0; t < C; t++)
            if (sp.st_phys[t] < 0) sp.st_phys[t] = freep[fi++];
    }
    // ops in schedule order with segment ids; per-segment permutation maps
    sp.seg_begin.assign(nseg + 1, 0);
    sp.maps.assign(nseg, identity_map());
    sp.n_gates = 0;
    sp.n_arith = 0;
    for (size_t i = 0; i < order.size(); i++) {
        const Item &it = items[order[i]];
        sp.n_gates++;
        if (it.op.kind == OP_NONE) continue;
        POp o = it.op;
        o.seg = seg_of[order[i]];
        if (o.perm) {
            const int t = tile_of[o.tp0];
            const int ct = (o.cp >= 0 && o.cp < n_loc) ? tile_of[o.cp] : -1;
            map_apply_perm(sp.maps[o.seg], t, ct, ct >= 0 ? -1 : o.cp);
        } else {
            sp.n_arith++;
        }
        sp.ops.push_back(o);
    }
    // ops sorted by segment (stable: schedule order inside a segment)
    std::stable_sort(sp.ops.begin(), sp.ops.end(), [](const POp &a, const POp &b) { return a.seg < b.seg; });
    for (int s = 0, oi = 0; s <= nseg; s++) {
        while (oi < (int)sp.ops.size() && sp.ops[oi].seg < s) oi++;
        sp.seg_begin[s] = oi;
    }
    sp.seg_begin[nseg] = (int)sp.ops.size();
    // swizzle: per exchange, the write side's lane vectors (through the map)
    // and the read side's lane vectors must be bank-conflict free
    {
        std::vector<std::vector<uint32_t>> sets;
        const int SW = cfg.swz_bits;
        for (int s = 0; s + 1 < nseg; s++) {
            std::vector<uint32_t> w, r;
            for (int i = 0; i < SW; i++) {
                w.push_back(sp.maps[s].col[sp.lays[s].lane[i]]);
                r.push_back(1u << sp.lays[s + 1].lane[i]);
            }
            sets.push_back(w);
            sets.push_back(r);
        }
        sp.swz = choose_swizzle(k, SW, sets);
    }

    // new qubit map: relabels, then sigma on the tile
    st.pos_before = pos;
    std::vector<int> npos = fpos;
    for (int q = 0; q < n; q++) {
        const int p = fpos[q];
        if (p < n_loc && tile_of[p] >= 0) npos[q] = sp.st_phys[tile_of[p]];
    }
    if (sp.ops.empty()) npos = fpos;  // no launch: no sigma
    pos = npos;
    st.pos_after = npos;
    pending = remaining;
    return true;
}

static bool plan_small(const std::vector<GateRec> &gates, std::vector<int> &pending, std::vector<int> &pos,
                       const PlanConfig &cfg, Stage &st) {
    const int n = cfg.n, n_loc = cfg.n_loc;
    std::vector<char> blocked(n, 0);
    std::vector<int> rest;
    st.pos_before = pos;
    SmallPlan &sp = st.sm;
    sp.n_gates = 0;
    for (size_t ii = 0; ii < pending.size(); ii++) {
        const int gi = pending[ii];
        const GateRec &g = gates[gi];
        bool blk = false;
        for (int j = 0; j < g.nw; j++) if (blocked[g.w[j]]) blk = true;
        int tq[2], dq[2], nt, nd;
        roles(g, tq, nt, dq, nd);
        if (!blk && g.cls != CL_SWAP)
            for (int j = 0; j < nt; j++) if (pos[tq[j]] >= n_loc) blk = true;
        if (blk) {
            for (int j = 0; j < g.nw; j++) blocked[g.w[j]] = 1;
            rest.push_back(gi);
            continue;
        }
        sp.n_gates++;
        if (g.cls == CL_SWAP) { std::swap(pos[g.w[0]], pos[g.w[1]]); continue; }
        POp o = make_pop(g, gi, pos);
        if (o.kind != OP_NONE) sp.ops.push_back(o);
    }
    if (sp.n_gates == 0) return false;
    pending = rest;
    st.pos_after = pos;
    return true;
}

static void plan_remap(const std::vector<GateRec> &gates, const std::vector<int> &pending, std::vector<int> &pos,
                       const PlanConfig &cfg, Stage &st) {
    const int n = cfg.n, n_loc = cfg.n_loc;
    std::vector<int> need;  // global physical positions needed as targets soon
    for (size_t i = 0; i < pending.size() && i < (size_t)(4 * n); i++) {
        const GateRec &g = gates[pending[i]];
        if (g.cls == CL_SWAP) continue;
        int tq[2], dq[2], nt, nd;
        roles(g, tq, nt, dq, nd);
        for (int j = 0; j < nt; j++) {
            const int p = pos[tq[j]];
            if (p >= n_loc && !std::count(need.begin(), need.end(), p)) need.push_back(p);
        }
    }
    std::sort(need.begin(), need.end());
    // Belady: evict the local qubits whose next target use is furthest away
    std::vector<std::pair<long long, int>> cand;
    std::vector<int> lq(n);
    for (int q = 0; q < n; q++) lq[pos[q]] = q;
    for (int p = 0; p < n_loc; p++)
        cand.push_back({-(long long)next_target_use(gates, pending, lq[p]), -p});
    std::sort(cand.begin(), cand.end());
    RemapPlan &rm = st.rm;
    rm.m = (int)need.size();
    std::vector<int> lp;
    for (int i = 0; i < rm.m; i++) lp.push_back(-cand[i].second);
    std::sort(lp.begin(), lp.end());
    st.pos_before = pos;
    for (int i = 0; i < rm.m; i++) {
        rm.gpos[i] = need[i];
        rm.lpos[i] = lp[i];
        const int qa = lq[need[i]], qb = lq[lp[i]];
        std::swap(pos[qa], pos[qb]);
        lq[pos[qa]] = qa;
        lq[pos[qb]] = qb;
    }
    st.pos_after = pos;
}

// Plan reuse across parameter changes (training loops re-record the same circuit
// with new angles): the plan depends on the gates' structure only -- kinds, wires,
// trainability, classes and op forms -- never on parameter values beyond those.
uint64_t plan_signature(const std::vector<GateRec> &gates, const PlanConfig &cfg) {
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](uint64_t v) { h = (h ^ v) * 1099511628211ull; };
    const int c[] = {cfg.n, cfg.n_loc, cfg.k, cfg.R, cfg.small_max, cfg.c128 ? 1 : 0, cfg.swz_bits, cfg.c_low,
                     cfg.max_ops, cfg.max_slots};
    for (int v : c) mix((uint64_t)(int64_t)v);
    for (const GateRec &g : gates) {
        mix((uint64_t)g.kind); mix((uint64_t)g.nw); mix((uint64_t)g.ow[0]); mix((uint64_t)g.ow[1]);
        mix((uint64_t)g.w[0]); mix((uint64_t)g.w[1]); mix((uint64_t)g.trainable); mix((uint64_t)g.batched);
        mix((uint64_t)g.cls); mix((uint64_t)g.ngen);
        int plain = 0;
        if (g.cls == CL_U1) mix((uint64_t)op1_form(g.M, (g.trainable || g.batched) ? g.kind : -1, plain) * 2 + plain);
        if (g.cls == CL_CTRL1) mix((uint64_t)op1_form(g.sub, -1, plain) * 2 + plain);
        if (g.kind == TQD_MAT1 || g.kind == TQD_MAT2)  // constants: exact bits
            for (int i = 0; i < (g.nw == 2 ? 16 : 4); i++) {
                double re = g.M[i].real(), im = g.M[i].imag();
                uint64_t a, b;
                memcpy(&a, &re, 8); memcpy(&b, &im, 8);
                mix(a); mix(b);
            }
    }
    return h;
}

// new parameter values into a reused plan (same signature): op matrices only
void refresh_plan_values(std::vector<Stage> &stages, const std::vector<GateRec> &gates) {
    for (Stage &st : stages) {
        std::vector<POp> *ops = st.type == ST_SWEEP ? &st.sw.ops : st.type == ST_SMALL ? &st.sm.ops : nullptr;
        if (!ops) continue;
        for (POp &o : *ops) {
            const GateRec &g = gates[o.gate];
            switch (g.cls) {
            case CL_U1: for (int i = 0; i < 4; i++) o.m[i] = g.M[i]; break;
            case CL_CTRL1: for (int i = 0; i < 4; i++) o.m[i] = g.sub[i]; break;
            case CL_U2: for (int i = 0; i < 16; i++) o.m[i] = g.M[i]; break;
            case CL_DIAG1: o.m[0] = g.M[0]; o.m[1] = g.M[3]; break;
            case CL_DIAG2: for (int i = 0; i < 4; i++) o.m[i] = g.M[5 * i]; break;
            default: break;
            }
        }
    }
}

static int plan_circuit_once(const std::vector<GateRec> &gates, std::vector<int> pending, std::vector<int> &pos,
                             const PlanConfig &cfg, std::vector<Stage> &out, std::string &err) {
    int guard = 0;
    while (!pending.empty()) {
        if (++guard > 1000000) { err = "planner did not converge"; return TQD_ERR_STATE; }
        Stage st;
        bool ok;
        if (cfg.n_loc <= cfg.small_max) {
            st.type = ST_SMALL;
            ok = plan_small(gates, pending, pos, cfg, st);
        } else {
            st.type = ST_SWEEP;
            ok = plan_sweep(gates, pending, pos, cfg, st);
        }
        if (ok) {
            out.push_back(std::move(st));
            continue;
        }
        if (cfg.n_loc == cfg.n) { err = "planner made no progress on a single-rank state"; return TQD_ERR_STATE; }
        Stage rs;
        rs.type = ST_REMAP;
        plan_remap(gates, pending, pos, cfg, rs);
        if (rs.rm.m == 0) { err = "planner made no progress"; return TQD_ERR_STATE; }
        out.push_back(std::move(rs));
    }
    return TQD_OK;
}

// The trailing-segment trim of plan_sweep (fewer layout exchanges) helps layered
// circuits (HEA: 65 sweeps / 149 exchanges vs 65 / 157 untrimmed) but can cascade on
// sequential chains (the paper's CNOT + RY ladder at 24 q: 66 sweeps vs 23).  Plan
// both ways and keep the cheaper one: cost in sweep pairs = sweeps + 0.24 exchanges
// (an exchange pair measured at ~0.24 of a 30-q sweep pair) + 2 per
// remap.
double plan_cost(const std::vector<Stage> &v) {
    double c = 0.0;
    for (const Stage &s : v) {
        if (s.type == ST_SWEEP) c += 1.0 + 0.24 * (double)(s.sw.lays.size() - 1);
        else if (s.type == ST_REMAP) c += 2.0;
        else c += 1.0;
    }
    return c;
}

int plan_circuit(const std::vector<GateRec> &gates, std::vector<int> pending, std::vector<int> &pos,
                 const PlanConfig &cfg, std::vector<Stage> &out, std::string &err) {
    if (cfg.seg_min_gates >= 0 || cfg.n_loc <= cfg.small_max)
        return plan_circuit_once(gates, pending, pos, cfg, out, err);
    auto cost = [](const std::vector<Stage> &v) { return plan_cost(v); };
    static const int seg_min_default = [] {  // (TQD_PLAN_SEG_MIN_GATES: experiment knob)
        const char *e = getenv("TQD_PLAN_SEG_MIN_GATES");
        return e ? std::max(0, atoi(e)) : 6;
    }();
    PlanConfig ca = cfg, cb = cfg;
    ca.seg_min_gates = seg_min_default;
    cb.seg_min_gates = 0;
    std::vector<int> pa = pos, pb = pos;
    std::vector<Stage> sa, sb;
    int rc = plan_circuit_once(gates, pending, pa, ca, sa, err);
    if (rc) return rc;
    if (ca.seg_min_gates == 0) {
        pos = pa;
        for (auto &s : sa) out.push_back(std::move(s));
        return TQD_OK;
    }
    rc = plan_circuit_once(gates, pending, pb, cb, sb, err);
    if (rc) return rc;
    const bool use_b = cost(sb) < cost(sa);
    pos = use_b ? pb : pa;
    for (auto &s : (use_b ? sb : sa)) out.push_back(std::move(s));
    return TQD_OK;
}

// ---------------------------------------------------------------------------
// device encoding

static void put(double *m, int i, cd v) { m[2 * i] = v.real(); m[2 * i + 1] = v.imag(); }

static void fill_matrix(DevOp &d, const POp &o, bool dag) {
    switch (o.kind) {
    case OP_U1:
        if (!dag) for (int i = 0; i < 4; i++) put(d.m, i, o.m[i]);
        else { put(d.m, 0, std::conj(o.m[0])); put(d.m, 1, std::conj(o.m[2])); put(d.m, 2, std::conj(o.m[1])); put(d.m, 3, std::conj(o.m[3])); }
        break;
    case OP_R1:
        if (!dag) { d.m[0] = o.m[0].real(); d.m[1] = o.m[1].real(); d.m[2] = o.m[2].real(); d.m[3] = o.m[3].real(); }
        else { d.m[0] = o.m[0].real(); d.m[1] = o.m[2].real(); d.m[2] = o.m[1].real(); d.m[3] = o.m[3].real(); }
        break;
    case OP_P1:  // [[0,a],[b,0]]^dag = [[0, conj b], [conj a, 0]]
        if (!dag) { put(d.m, 0, o.m[1]); put(d.m, 1, o.m[2]); }
        else { put(d.m, 0, std::conj(o.m[2])); put(d.m, 1, std::conj(o.m[1])); }
        d.t1 = (uint8_t)o.plain;
        break;
    case OP_D1:
        put(d.m, 0, dag ? std::conj(o.m[0]) : o.m[0]);
        put(d.m, 1, dag ? std::conj(o.m[1]) : o.m[1]);
        break;
    case OP_U2:
        for (int r = 0; r < 4; r++)
            for (int c = 0; c < 4; c++) put(d.m, 4 * r + c, dag ? std::conj(o.m[4 * c + r]) : o.m[4 * r + c]);
        break;
    case OP_D2:
        for (int i = 0; i < 4; i++) put(d.m, i, dag ? std::conj(o.m[i]) : o.m[i]);
        break;
    default: break;
    }
}

static void fill_gens(DevOp &d, const GateRec &g) {
    d.ngen = (uint8_t)g.ngen;
    for (int i = 0; i < g.ngen; i++) {
        d.gkind[i] = g.gkind[i];
        for (int j = 0; j < 4; j++) put(d.g[i], j, g.G[i][j]);
    }
}

// The 2x2 an op applies to its target / diagonal bit (forward or adjoint form).
// batched 1q gates: the op's matrix is the batch element's (same op form)
static POp pop_for(const POp &o, const GateRec &g) {
    if (!g.batched) return o;
    POp r = o;
    if (o.kind == OP_D1) { r.m[0] = g.M[0]; r.m[1] = g.M[3]; }
    else for (int i = 0; i < 4; i++) r.m[i] = g.M[i];
    return r;
}

static void op_matrix2(const POp &o, bool dag, cd *M) {
    cd F[4];
    switch (o.kind) {
    case OP_U1: case OP_R1: F[0] = o.m[0]; F[1] = o.m[1]; F[2] = o.m[2]; F[3] = o.m[3]; break;
    case OP_P1: F[0] = 0.0; F[1] = o.m[1]; F[2] = o.m[2]; F[3] = 0.0; break;
    case OP_D1: F[0] = o.m[0]; F[1] = 0.0; F[2] = 0.0; F[3] = o.m[1]; break;
    default: F[0] = 1.0; F[1] = 0.0; F[2] = 0.0; F[3] = 1.0; break;
    }
    if (!dag) { for (int i = 0; i < 4; i++) M[i] = F[i]; }
    else { M[0] = std::conj(F[0]); M[1] = std::conj(F[2]); M[2] = std::conj(F[1]); M[3] = std::conj(F[3]); }
}

template <typename Real>
void encode_sweep_k(const SweepPlan &sp, const std::vector<GateRec> &gates, bool bwd, int n_loc, DevStage &ds,
                    std::vector<KOp<Real>> &ops, std::vector<int32_t> &slot_param, int skip_below) {
    memset(&ds, 0, sizeof(ds));
    const int nseg = (int)sp.lays.size();
    const int R = sp.R;
    ds.k = sp.k; ds.R = sp.R; ds.W = sp.W; ds.nseg = nseg;
    {
        static const char *fe = getenv("TQD_EXPERIMENT_FLAGS");  // timing experiments only
        ds.flags = fe ? atoi(fe) : 0;
    }
    ds.n_tiles = (int64_t)1 << (n_loc - sp.k);
    std::vector<int> sorted = sp.ld_phys;
    std::sort(sorted.begin(), sorted.end());
    for (int t = 0; t < sp.k; t++) {
        ds.ld_phys[t] = (uint8_t)(bwd ? sp.st_phys[t] : sp.ld_phys[t]);
        ds.st_phys[t] = (uint8_t)(bwd ? sp.ld_phys[t] : sp.st_phys[t]);
        ds.tile_sorted[t] = (uint8_t)sorted[t];
        ds.swz[t] = sp.swz[t];
    }
    std::vector<int> tile_of(n_loc, -1);
    for (int t = 0; t < sp.k; t++) tile_of[sp.ld_phys[t]] = t;
    ds.op_base = (int)ops.size();
    ds.slot_base = (int)slot_param.size();
    int nslots = 0;
    // complex coefficient e at m[4i..4i+3] as (re, 0, im, im): the kernel does a
    // complex multiply with one packed FMUL2 + one FFMA2 (swapped / negated halves)
    auto pute = [](KOp<Real> &k, int i, cd v) {
        k.m[4 * i] = (Real)v.real();
        k.m[4 * i + 1] = 0;
        k.m[4 * i + 2] = (Real)v.imag();
        k.m[4 * i + 3] = (Real)v.imag();
    };
    const int threads = 32 << sp.W;
    int n_cvals = 0, n_uvals = 0;  // diagonal-block C rows / U values of this stage
    // the forward sweep has shared memory to spare (one state tile): more C rows
    const int ccap = (sizeof(Real) == 4 ? DBLK_CCAP_F32 : DBLK_CCAP_F64) * (bwd ? 1 : 3);
    auto finalize = [threads](KOp<Real> &k) {
        switch (k.kind) {
        case K_LAYER:
            k.code = (uint8_t)(k.ltype == LT_DIAG ? KC_DIAG : k.ltype == LT_REAL ? KC_REAL + k.mask : KC_GEN + k.mask);
            break;
        case K_CU: k.code = (uint8_t)(KC_CU + k.t0); break;
        case K_PHASE: k.code = KC_PHASE; break;
        case K_D2: k.code = KC_D2; break;
        case K_DBLK: k.code = KC_DBLK; break;
        case K_U2: k.code = (uint8_t)(KC_U2 + u2_index(k.t0, k.t1)); break;
        default: k.code = KC_NOP; break;
        }
        k.gbits = 0;
        k.gkinds = 0;
        for (int i = 0; i < k.ngen; i++) {
            k.gbits |= (uint8_t)((k.gbit[i] & 3) << (2 * i));
            k.gkinds |= (uint16_t)((k.gkind[i] & 15) << (4 * i));
        }
        // layer fast path: every generator is the layer type's own (RY on a real
        // layer, RZ on a diagonal layer), at most one per register bit
        k.gmask = 0;
        if (k.kind == K_LAYER && k.ngen > 0 && (k.ltype == LT_REAL || k.ltype == LT_DIAG)) {
            const int want = k.ltype == LT_REAL ? GEN_Y : GEN_Z;
            int gm = 0;
            bool ok = true;
            for (int i = 0; i < k.ngen; i++) {
                if (k.gkind[i] != want || ((gm >> k.gbit[i]) & 1)) ok = false;
                gm |= 1 << k.gbit[i];
            }
            if (ok) k.gmask = (uint8_t)gm;
        }
        for (int i = 0; i < KOP_MAXGEN; i++) k.soff[i] = 0;
        for (int i = 0; i < k.ngen; i++)
            k.soff[k.gmask ? k.gbit[i] : i] = (uint16_t)(k.slot[i] * threads);
    };
    auto newop = [](int kind) {
        KOp<Real> k;
        memset(&k, 0, sizeof(k));
        k.kind = (uint8_t)kind;
        k.creg = 0xff;
        return k;
    };
    auto add_gen = [&](KOp<Real> &k, const GateRec &g, int i, int bit) {
        const int j = k.ngen++;
        k.gbit[j] = (uint8_t)bit;
        k.gkind[j] = g.gkind[i];
        for (int q = 0; q < 4; q++) { k.g[j][2 * q] = (Real)g.G[i][q].real(); k.g[j][2 * q + 1] = (Real)g.G[i][q].imag(); }
        k.slot[j] = (int16_t)nslots++;
        slot_param.push_back(g.slot0 + i);
    };
    for (int s = 0; s < nseg; s++) {
        const int fs = bwd ? nseg - 1 - s : s;
        const Layout &L = sp.lays[fs];
        DevLayout &DL = ds.lay[s];
        for (int i = 0; i < R; i++) DL.reg[i] = (uint8_t)L.reg[i];
        for (int i = 0; i < LANE_BITS; i++) DL.lane[i] = (uint8_t)L.lane[i];
        for (int i = 0; i < WMAX; i++) DL.warp[i] = (uint8_t)L.warp[i];
        ds.seg_begin[s] = (int)ops.size() - ds.op_base;
        auto regidx = [&](int p) {
            if (p < 0 || p >= n_loc || tile_of[p] < 0) return -1;
            for (int i = 0; i < R; i++) if (L.reg[i] == tile_of[p]) return i;
            return -1;
        };
        auto bref = [&](int p) {
            BitRef r;
            r.kind = BK_NONE; r.idx = 0;
            if (p < 0) return r;
            const int t = p < n_loc ? tile_of[p] : -1;
            const int ri = regidx(p);
            if (ri >= 0) { r.kind = BK_REG; r.idx = (uint8_t)ri; }
            else if (t >= 0) { r.kind = BK_TIX; r.idx = (uint8_t)t; }
            else { r.kind = BK_BASE; r.idx = (uint8_t)p; }
            return r;
        };
        // current fused layer: single-qubit gates on register bits, one matrix
        // type per layer (real / diagonal / general) so the kernel's cheapest
        // variant applies (real: packed f32x2 FMA, diagonal: one complex multiply
        // per amplitude with the host-built table of 16 phase products)
        bool active = false;
        int mask = 0, ltype = LT_GEN;
        cd LM[RMAX][4];
        KOp<Real> layer = newop(K_LAYER);
        auto mtype = [](const cd *M) {
            if (M[1] == cd(0.0) && M[2] == cd(0.0)) return (int)LT_DIAG;
            for (int q = 0; q < 4; q++) if (M[q].imag() != 0.0) return (int)LT_GEN;
            return (int)LT_REAL;
        };
        auto flush = [&]() {
            if (!active) return;
            layer.mask = (uint8_t)mask;
            layer.ltype = (uint8_t)ltype;
            if (ltype == LT_DIAG) {
                for (int r = 0; r < (1 << R); r++) {
                    cd ph = 1.0;
                    for (int bb = 0; bb < R; bb++)
                        if ((mask >> bb) & 1) ph *= ((r >> bb) & 1) ? LM[bb][3] : LM[bb][0];
                    pute(layer, r, ph);
                }
            } else {
                for (int bb = 0; bb < R; bb++) {
                    if (!((mask >> bb) & 1)) continue;
                    Real *m = layer.m + 8 * bb;
                    if (ltype == LT_REAL) {
                        for (int q = 0; q < 4; q++) m[q] = (Real)LM[bb][q].real();
                    } else {
                        for (int q = 0; q < 4; q++) pute(layer, 4 * bb + q, LM[bb][q]);
                    }
                }
            }
            finalize(layer);
            ops.push_back(layer);
            active = false;
            mask = 0;
            layer = newop(K_LAYER);
        };
        const int b = sp.seg_begin[fs], e = sp.seg_begin[fs + 1];
        static const bool skip_ops = getenv("TQD_EXPERIMENT_SKIP_OPS") != nullptr;  // timing experiment only
        // Single-qubit gates on register bits are queued per bit and emitted as
        // layers: each layer takes the front gate of every bit whose front has the
        // chosen type (gates on different bits commute, same-bit order is kept);
        // the forward also composes consecutive same-type gates on one bit.  Any
        // other op (controlled / 2q / phase on a non-register bit) drains the queues.
        struct QG { cd M[4]; int t; int gate; int batched; };
        std::vector<QG> q[RMAX];
        size_t qh[RMAX] = {0, 0, 0, 0, 0};
        auto drain = [&]() {
            for (;;) {
                int cnt[3] = {0, 0, 0};
                for (int bb = 0; bb < R; bb++)
                    if (qh[bb] < q[bb].size()) cnt[q[bb][qh[bb]].t]++;
                if (!cnt[0] && !cnt[1] && !cnt[2]) break;
                int T = LT_REAL;
                for (int tt : {LT_DIAG, LT_GEN})
                    if (cnt[tt] > cnt[T]) T = tt;
                if (!cnt[T]) T = cnt[LT_DIAG] ? LT_DIAG : LT_GEN;
                active = true;
                ltype = T;
                for (int bb = 0; bb < R; bb++) {
                    if (qh[bb] >= q[bb].size() || q[bb][qh[bb]].t != T) continue;
                    const GateRec &gg = gates[q[bb][qh[bb]].gate];
                    if (bwd && layer.ngen + gg.ngen > KOP_MAXGEN) continue;
                    for (int c = 0; c < 4; c++) LM[bb][c] = q[bb][qh[bb]].M[c];
                    mask |= 1 << bb;
                    if (bwd && gg.ngen)
                        for (int i = 0; i < gg.ngen; i++) add_gen(layer, gg, i, bb);
                    qh[bb]++;
                    // forward: fold following gates on this bit while the product keeps the type
                    // (never across batched gates: their type must not depend on values)
                    const bool took_batched = q[bb][qh[bb] - 1].batched != 0;
                    while (!bwd && !took_batched && qh[bb] < q[bb].size() && !q[bb][qh[bb]].batched) {
                        const cd *Mn = q[bb][qh[bb]].M;
                        cd Pm[4];
                        Pm[0] = Mn[0] * LM[bb][0] + Mn[1] * LM[bb][2];
                        Pm[1] = Mn[0] * LM[bb][1] + Mn[1] * LM[bb][3];
                        Pm[2] = Mn[2] * LM[bb][0] + Mn[3] * LM[bb][2];
                        Pm[3] = Mn[2] * LM[bb][1] + Mn[3] * LM[bb][3];
                        if (mtype(Pm) != T) break;
                        for (int c = 0; c < 4; c++) LM[bb][c] = Pm[c];
                        qh[bb]++;
                    }
                }
                flush();
            }
            for (int bb = 0; bb < R; bb++) { q[bb].clear(); qh[bb] = 0; }
        };
        // Diagonal blocks: diagonal gates off the register-bit queues (K_PHASE /
        // K_D2 forms) are kept as pending phase-polynomial terms Phi += ang * x * y
        // (x, y: register / lane-warp / base bits or none) and emitted as K_DBLK
        // runs (DTerm): lane / warp / base terms accumulate in per-thread fixed-point
        // registers over chained kops, the last kop of a run converts them and
        // applies exp(i Phi) with the register-only part as a 16-entry table.
        // Pending terms commute with every queued gate: queueing a gate on register
        // bit b first emits the pending terms that involve b (the others stay
        // pending), and a diagonal gate involving a register bit with queued gates
        // drains the queues first.
        struct DT { BitRef a, b; double ang; };
        std::vector<DT> dpend;
        double dconst = 0;  // global phase of the pending terms
        auto dref_less = [](BitRef x, BitRef y) { return x.kind != y.kind ? x.kind < y.kind : x.idx < y.idx; };
        const BitRef none = {BK_NONE, 0};
        auto dadd = [&](BitRef x, BitRef y, double ang) {  // Phi += ang * x * y (y may be BK_NONE)
            if (std::abs(std::remainder(ang, 2 * M_PI)) < 1e-15) return;
            // normal order: a register bit first, else the smaller reference; none last
            if (y.kind == BK_REG && x.kind != BK_REG) std::swap(x, y);
            else if (x.kind != BK_REG && y.kind != BK_NONE && x.kind != BK_NONE && dref_less(y, x)) std::swap(x, y);
            else if (x.kind == BK_REG && y.kind == BK_REG && y.idx < x.idx) std::swap(x, y);
            for (DT &t : dpend)
                if (t.a.kind == x.kind && t.a.idx == x.idx && t.b.kind == y.kind && t.b.idx == y.idx) {
                    t.ang += ang;
                    return;
                }
            dpend.push_back({x, y, ang});
        };
        auto involves = [](const DT &t, int rb) {
            return (t.a.kind == BK_REG && t.a.idx == rb) || (t.b.kind == BK_REG && t.b.idx == rb);
        };
        auto turn = [](double ang, double scale) {  // fraction of a full turn, fixed point
            double f = ang / (2 * M_PI);
            f -= std::floor(f);
            const long double v = (long double)f * (long double)scale;
            return v >= (long double)scale ? (long double)0 : v;
        };
        // emit terms (and a global phase) as one K_DBLK run; per kop the terms are
        // ordered [C | U | M] (tqd_internal.h): C and U sums are precomputed by the
        // kernel (per thread once, per tile once) while the budgets last
        auto cls_of = [](const DT &t) {  // 0 = C (no base bit), 1 = U (no lane/warp bit), 2 = M
            const bool has_base = t.a.kind == BK_BASE || t.b.kind == BK_BASE;
            const bool has_tix = t.a.kind == BK_TIX || t.b.kind == BK_TIX;
            return has_base ? (has_tix ? 2 : 1) : 0;
        };
        auto emit_dblk = [&](const std::vector<DT> &terms, double cst) {
            std::vector<double> tab(1 << R, cst);
            std::vector<DT> other;
            for (const DT &t : terms) {
                if (t.a.kind == BK_REG && (t.b.kind == BK_REG || t.b.kind == BK_NONE)) {
                    for (int r = 0; r < (1 << R); r++)
                        if (((r >> t.a.idx) & 1) && (t.b.kind == BK_NONE || ((r >> t.b.idx) & 1))) tab[r] += t.ang;
                } else {
                    other.push_back(t);
                }
            }
            bool ident = true;
            for (double v : tab)
                if (std::abs(std::remainder(v, 2 * M_PI)) > 1e-15) ident = false;
            if (ident && other.empty()) return;
            // cheap forms first: register bits only -> a diagonal layer; plus at most six
            // single-bit terms on lane / warp / base bits -> K_PHASE ops (one multiply per
            // amplitude each, no per-tile work, the plain kernel instantiation: the
            // diagonal-block instantiation costs ~2 ms more per 30-qubit sweep)
            bool simple = other.size() <= 6;
            for (const DT &t : other)
                if (t.a.kind == BK_REG || t.b.kind != BK_NONE) simple = false;
            if (simple) {
                if (!ident) {
                    KOp<Real> k = newop(K_LAYER);
                    k.ltype = LT_DIAG;
                    k.mask = (uint8_t)((1 << R) - 1);
                    for (int r = 0; r < (1 << R); r++) pute(k, r, std::polar(1.0, tab[r]));
                    finalize(k);
                    ops.push_back(k);
                }
                for (const DT &t : other) {
                    KOp<Real> k = newop(K_PHASE);
                    k.b0 = t.a;
                    pute(k, 0, cd(1.0));
                    pute(k, 1, std::polar(1.0, t.ang));
                    finalize(k);
                    ops.push_back(k);
                }
                return;
            }
            uint8_t xm = 0;
            for (const DT &t : other)
                if (t.a.kind == BK_REG) xm |= (uint8_t)(1u << t.a.idx);
            // run-level classes; C / U sums precomputed by the kernel while the stage
            // budgets last (rows th, al[b] for b in xm), the rest evaluated per tile (M)
            std::vector<DT> cl[3];
            for (const DT &t : other) cl[cls_of(t)].push_back(t);
            const int rows = 1 + __builtin_popcount(xm);
            uint8_t coff = 0xff, uoff = 0xff;
            if (!cl[0].empty() && n_cvals + rows <= ccap) { coff = (uint8_t)n_cvals; n_cvals += rows; }
            else { cl[2].insert(cl[2].end(), cl[0].begin(), cl[0].end()); cl[0].clear(); }
            if (!cl[1].empty() && n_uvals + rows <= DBLK_UCAP) { uoff = (uint8_t)n_uvals; n_uvals += rows; }
            else { cl[2].insert(cl[2].end(), cl[1].begin(), cl[1].end()); cl[1].clear(); }
            std::vector<std::pair<int, DT>> seq;  // (class, term) in [C | U | M] order
            for (int c = 0; c < 3; c++)
                for (const DT &t : cl[c]) seq.push_back({c, t});
            // chunks of DBLK_TERMS: data kops (KC_DDATA, never dispatched to work) and the
            // applying kop last (KC_DBLK), which reads the whole run's C / U / M sums
            const int nk = std::max<int>(1, (int)((seq.size() + DBLK_TERMS - 1) / DBLK_TERMS));
            for (int kk = 0; kk < nk; kk++) {
                const size_t i0 = (size_t)kk * DBLK_TERMS;
                const size_t cnt = std::min<size_t>(DBLK_TERMS, seq.size() - std::min(seq.size(), i0));
                const bool last = kk == nk - 1;
                KOp<Real> k = newop(K_DBLK);
                for (int r = 0; r < (1 << R); r++) pute(k, r, last ? std::polar(1.0, tab[r]) : cd(1.0));
                finalize(k);
                if (!last) k.code = KC_DDATA;
                int ncls[3] = {0, 0, 0};
                DTerm<Real> *tm = reinterpret_cast<DTerm<Real> *>(k.g);
                for (size_t jx = 0; jx < cnt; jx++) {
                    const DT &t = seq[i0 + jx].second;
                    ncls[seq[i0 + jx].first]++;
                    DTerm<Real> d;
                    memset(&d, 0, sizeof(d));
                    if (sizeof(Real) == 4) d.ang = (uint32_t)(uint64_t)turn(t.ang, 4294967296.0);
                    else d.ang = (decltype(d.ang))turn(t.ang, 18446744073709551616.0);
                    d.a = t.a;
                    d.b = t.b;
                    tm[jx] = d;
                }
                // header bytes (unused by this kind): 2 flags (2: identity table), 3 data kops
                // before the applying one, 4 xm, 5 c_off, 6 u_off, 8..10 nC nU nM
                k.creg = (uint8_t)(last && ident ? 2 : 0);
                k.t0 = (uint8_t)(last ? nk - 1 : 0);
                k.gbits = xm;
                k.gmask = coff;
                k.ctrl.kind = uoff;
                k.ctrl.idx = 0;
                k.b0.kind = (uint8_t)ncls[0];
                k.b0.idx = (uint8_t)ncls[1];
                k.b1.kind = (uint8_t)ncls[2];
                k.b1.idx = 0;
                ops.push_back(k);
            }
        };
        auto flush_dblk = [&]() {  // all pending terms
            if (dpend.empty() && std::abs(std::remainder(dconst, 2 * M_PI)) < 1e-15) { dpend.clear(); dconst = 0; return; }
            emit_dblk(dpend, dconst);
            dpend.clear();
            dconst = 0;
        };
        auto flush_bit = [&](int rb) {  // the pending terms that involve register bit rb
            std::vector<DT> sel, keep;
            for (const DT &t : dpend) (involves(t, rb) ? sel : keep).push_back(t);
            if (sel.empty()) return;
            emit_dblk(sel, 0.0);
            dpend.swap(keep);
        };
        for (int jj = 0; jj < e - b && !skip_ops; jj++) {
            const POp &o0 = sp.ops[bwd ? e - 1 - jj : b + jj];
            if (o0.perm) continue;  // folded into the layout-change maps below
            // reverse sweep: gates before the earliest trainable gate (tape order) are
            // never needed -- every later gate sharing a qubit with one of them is
            // placed after it, so the skipped ones commute with all that remain
            if (bwd && o0.gate < skip_below) continue;
            const GateRec &g = gates[o0.gate];
            const POp o = pop_for(o0, g);
            const bool has_gen = bwd && g.ngen > 0;
            int bit = -1;
            if ((o.kind == OP_U1 || o.kind == OP_R1 || o.kind == OP_P1) && o.cp < 0) bit = regidx(o.tp0);
            else if (o.kind == OP_D1 && o.cp < 0) bit = regidx(o.dp0);
            if (bit >= 0) {
                QG qg;
                op_matrix2(o, bwd, qg.M);
                qg.t = mtype(qg.M);
                if (g.trainable && g.kind == TQD_RZ) qg.t = LT_DIAG;  // RZ gradients are batched on diagonal layers
                qg.batched = g.batched;
                if (g.batched) qg.t = g.kind == TQD_RY ? LT_REAL : g.kind == TQD_RZ ? LT_DIAG : LT_GEN;  // by kind
                qg.gate = o.gate;
                flush_bit(bit);
                q[bit].push_back(qg);
                continue;
            }
            // (batched gates keep their own K_PHASE op: a run's kop structure depends on
            // the values -- zero terms vanish -- and must be equal for every batch element)
            if ((o.kind == OP_D1 && o.cp < 0 && !has_gen && !g.batched) || o.kind == OP_D2) {
                // theta(u, v) = a + b u + c v + d u v with theta_uv = arg d[2u + v] (u = MSB bit)
                const BitRef u = bref(o.dp0), v = o.kind == OP_D2 ? bref(o.dp1) : none;
                bool busy = false;  // a register bit of this gate has queued gates: they go first
                for (BitRef x : {u, v})
                    if (x.kind == BK_REG && qh[x.idx] < q[x.idx].size()) busy = true;
                if (busy) drain();
                if (o.kind == OP_D1) {
                    cd M1[4];
                    op_matrix2(o, bwd, M1);
                    const double t0 = std::arg(M1[0]), t1 = std::arg(M1[3]);
                    dconst += t0;
                    dadd(u, none, t1 - t0);
                } else {
                    double th[4];
                    for (int qq = 0; qq < 4; qq++) th[qq] = std::arg(bwd ? std::conj(o.m[qq]) : o.m[qq]);
                    dconst += th[0];
                    dadd(u, none, th[2] - th[0]);
                    dadd(v, none, th[1] - th[0]);
                    dadd(u, v, th[3] - th[2] - th[1] + th[0]);
                }
                continue;
            }
            drain();
            flush_dblk();
            KOp<Real> k = newop(K_NOP);
            cd M[4];
            switch (o.kind) {
            case OP_U1: case OP_R1: case OP_P1: {
                // controlled 1q (CNOT, controlled MAT2); targets are always register bits
                op_matrix2(o, bwd, M);
                k.kind = K_CU;
                k.t0 = (uint8_t)regidx(o.tp0);
                const int cr = regidx(o.cp);
                if (cr >= 0) k.creg = (uint8_t)cr;
                else if (o.cp >= 0) k.ctrl = bref(o.cp);
                for (int q = 0; q < 4; q++) pute(k, q, M[q]);
                break;
            }
            case OP_D1: {
                op_matrix2(o, bwd, M);
                k.kind = K_PHASE;
                k.b0 = bref(o.dp0);
                pute(k, 0, M[0]);
                pute(k, 1, M[3]);
                if (has_gen) add_gen(k, g, 0, 0);
                break;
            }
            case OP_D2: {
                k.kind = K_D2;
                k.b0 = bref(o.dp0);
                k.b1 = bref(o.dp1);
                for (int q = 0; q < 4; q++) pute(k, q, bwd ? std::conj(o.m[q]) : o.m[q]);
                break;
            }
            case OP_U2: {
                k.kind = K_U2;
                k.t0 = (uint8_t)regidx(o.tp0);
                k.t1 = (uint8_t)regidx(o.tp1);
                for (int r = 0; r < 4; r++)
                    for (int c = 0; c < 4; c++) pute(k, 4 * r + c, bwd ? std::conj(o.m[4 * c + r]) : o.m[4 * r + c]);
                break;
            }
            default: continue;
            }
            finalize(k);
            ops.push_back(k);
        }
        drain();
        flush_dblk();
    }
    ds.seg_begin[nseg] = (int)ops.size() - ds.op_base;
    ds.n_ops = (int)ops.size() - ds.op_base;
    ds.n_cvals = n_cvals;
    ds.n_uvals = n_uvals;
    ds.n_dblk = 0;
    for (int i = ds.op_base; i < (int)ops.size(); i++)
        if (ops[i].code == KC_DBLK) ds.n_dblk++;
    ds.n_slots = nslots;
    // exchange synchronisation (kernel order x; fwd segment f = x, adjoint f = nseg-2-x).
    // Write -> read: warps that keep their warp-index bits U_x only exchange among the
    // group of warps sharing those bits (named barrier per group; U = all -> __syncwarp).
    // Read -> next write: a warp's next writes land in the region it just read iff the
    // map that relates them keeps the warp bits of the layout in between (forward: the
    // next exchange's map, applied on its write side; adjoint: this exchange's map,
    // applied on its read side); then __syncwarp suffices.  The tile's last exchange
    // always ends with a CTA barrier (the next tile restarts at layout 0).
    {
        auto wset = [&](int fs) {
            uint32_t m = 0;
            for (int i = 0; i < sp.W; i++) m |= 1u << sp.lays[fs].warp[i];
            return m;
        };
        for (int x = 0; x + 1 < nseg; x++) {
            const int f = bwd ? nseg - 2 - x : x;
            uint8_t v = (uint8_t)(sp.xumask[f] & 0x0f);
            bool tail = false;
            if (x + 2 < nseg) {
                if (!bwd) tail = !(sp.perm_tgt[x + 1] & wset(x + 1));
                else tail = !(sp.perm_tgt[f] & wset(f));  // kernel layout x+1 = fwd layout f
                // a group barrier (named barrier per warp group) must not be entered
                // while other warps still wait in this exchange's group barriers: keep
                // the CTA barrier before a partially-kept exchange
                const int fn = bwd ? f - 1 : x + 1;
                const uint8_t un = sp.xumask[fn];
                if (un != 0 && un != (1 << sp.W) - 1) tail = false;
            }
            if (ds.flags & 1) { v = 0; tail = false; }  // experiment: CTA barriers everywhere
            ds.xsync[x] = v | (tail ? 0x80 : 0);
        }
    }
    // layout changes: forward exchange s applies the map of forward segment s on
    // the write side; the adjoint (exchange from forward layout f+1 to f) applies
    // it on the read side (amp_pre[x] = amp_post[A x + b])
    const uint32_t *swz = sp.swz.data();
    for (int x = 0; x + 1 < nseg; x++) {
        const int f = bwd ? nseg - 2 - x : x;
        const TileMap &M = sp.maps[f];
        uint32_t *mcol = bwd ? ds.rcol[x] : ds.wcol[x];
        uint32_t *pcol = bwd ? ds.wcol[x] : ds.rcol[x];
        for (int t = 0; t < sp.k; t++) {
            mcol[t] = lin(swz, M.col[t]);
            pcol[t] = swz[t];
        }
        (bwd ? ds.rcst[x] : ds.wcst[x]) = lin(swz, M.cst);
        (bwd ? ds.wcst[x] : ds.rcst[x]) = 0;
        ds.aff_read[x] = bwd ? 1 : 0;
        ds.naff[x] = (uint8_t)M.aff.size();
        for (size_t i = 0; i < M.aff.size() && i < (size_t)NAFF; i++) {
            ds.aff_pos[x][i] = (uint8_t)M.aff[i].first;
            ds.aff_vec[x][i] = lin(swz, M.aff[i].second);
        }
    }
}

template void encode_sweep_k<float>(const SweepPlan &, const std::vector<GateRec> &, bool, int, DevStage &,
                                    std::vector<KOp<float>> &, std::vector<int32_t> &, int);
template void encode_sweep_k<double>(const SweepPlan &, const std::vector<GateRec> &, bool, int, DevStage &,
                                     std::vector<KOp<double>> &, std::vector<int32_t> &, int);

void encode_small(const SmallPlan &sp, const std::vector<GateRec> &gates, bool bwd, std::vector<DevOp> &ops,
                  int skip_below) {
    const int m = (int)sp.ops.size();
    for (int jj = 0; jj < m; jj++) {
        if (bwd && sp.ops[m - 1 - jj].gate < skip_below) continue;  // as in encode_sweep_k
        const POp o = pop_for(sp.ops[bwd ? m - 1 - jj : jj], gates[sp.ops[bwd ? m - 1 - jj : jj].gate]);
        DevOp d;
        memset(&d, 0, sizeof(d));
        d.kind = (uint8_t)o.kind;
        if (o.tp0 >= 0) d.t0 = (uint8_t)o.tp0;
        if (o.tp1 >= 0) d.t1 = (uint8_t)o.tp1;
        auto bref = [&](int p) {
            BitRef r;
            r.kind = p < 0 ? BK_NONE : BK_BASE;
            r.idx = (uint8_t)(p < 0 ? 0 : p);
            return r;
        };
        d.ctrl = bref(o.cp);
        d.b0 = bref(o.dp0);
        d.b1 = bref(o.dp1);
        fill_matrix(d, o, bwd);
        if (o.kind == OP_P1) d.t1 = (uint8_t)o.tp1;  // small kernel ignores t1 for P1
        if (bwd && gates[o.gate].ngen) {
            fill_gens(d, gates[o.gate]);
            for (int i = 0; i < d.ngen; i++) d.slot[i] = gates[o.gate].slot0 + i;
        }
        ops.push_back(d);
    }
}

// ---------------------------------------------------------------------------
std::string plan_to_json(const std::vector<Stage> &stages, const PlanConfig &cfg) {
    std::ostringstream os;
    os << "{\"n\":" << cfg.n << ",\"n_loc\":" << cfg.n_loc << ",\"k\":" << cfg.k << ",\"R\":" << cfg.R
       << ",\"stages\":[";
    for (size_t si = 0; si < stages.size(); si++) {
        const Stage &st = stages[si];
        if (si) os << ",";
        os << "{\"type\":\"" << (st.type == ST_SWEEP ? "sweep" : st.type == ST_SMALL ? "small" : "remap") << "\"";
        os << ",\"pos_before\":[";
        for (size_t i = 0; i < st.pos_before.size(); i++) os << (i ? "," : "") << st.pos_before[i];
        os << "],\"pos_after\":[";
        for (size_t i = 0; i < st.pos_after.size(); i++) os << (i ? "," : "") << st.pos_after[i];
        os << "]";
        auto op_json = [&](const POp &o) {
            os << "{\"gate\":" << o.gate << ",\"kind\":" << o.kind << ",\"tp0\":" << o.tp0 << ",\"tp1\":" << o.tp1
               << ",\"cp\":" << o.cp << ",\"dp0\":" << o.dp0 << ",\"dp1\":" << o.dp1 << ",\"seg\":" << o.seg
               << ",\"wp0\":" << o.wp0 << ",\"wp1\":" << o.wp1 << ",\"perm\":" << o.perm << "}";
        };
        if (st.type == ST_SWEEP) {
            const SweepPlan &sp = st.sw;
            os << ",\"k\":" << sp.k << ",\"R\":" << sp.R << ",\"W\":" << sp.W << ",\"n_gates\":" << sp.n_gates
               << ",\"c_low\":" << cfg.c_low;
            os << ",\"ld_phys\":[";
            for (int t = 0; t < sp.k; t++) os << (t ? "," : "") << sp.ld_phys[t];
            os << "],\"st_phys\":[";
            for (int t = 0; t < sp.k; t++) os << (t ? "," : "") << sp.st_phys[t];
            os << "],\"swz\":[";
            for (int t = 0; t < sp.k; t++) os << (t ? "," : "") << sp.swz[t];
            os << "],\"xwarp\":[";
            for (size_t s = 0; s < sp.xwarp.size(); s++) os << (s ? "," : "") << (int)sp.xwarp[s];
            os << "],\"xumask\":[";
            for (size_t s = 0; s < sp.xumask.size(); s++) os << (s ? "," : "") << (int)sp.xumask[s];
            os << "],\"layouts\":[";
            for (size_t s = 0; s < sp.lays.size(); s++) {
                const Layout &L = sp.lays[s];
                os << (s ? "," : "") << "{\"reg\":[";
                for (int i = 0; i < sp.R; i++) os << (i ? "," : "") << L.reg[i];
                os << "],\"lane\":[";
                for (int i = 0; i < LANE_BITS; i++) os << (i ? "," : "") << L.lane[i];
                os << "],\"warp\":[";
                for (int i = 0; i < sp.W; i++) os << (i ? "," : "") << L.warp[i];
                os << "]}";
            }
            os << "],\"ops\":[";
            for (size_t i = 0; i < sp.ops.size(); i++) { if (i) os << ","; op_json(sp.ops[i]); }
            os << "]";
        } else if (st.type == ST_SMALL) {
            os << ",\"n_gates\":" << st.sm.n_gates << ",\"ops\":[";
            for (size_t i = 0; i < st.sm.ops.size(); i++) { if (i) os << ","; op_json(st.sm.ops[i]); }
            os << "]";
        } else {
            os << ",\"m\":" << st.rm.m << ",\"gpos\":[";
            for (int i = 0; i < st.rm.m; i++) os << (i ? "," : "") << st.rm.gpos[i];
            os << "],\"lpos\":[";
            for (int i = 0; i < st.rm.m; i++) os << (i ? "," : "") << st.rm.lpos[i];
            os << "]";
        }
        os << "}";
    }
    os << "]}";
    return os.str();
}

}  // namespace tqd
