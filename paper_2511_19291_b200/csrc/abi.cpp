// abi.cpp -- the C ABI of include/tqd.h: contexts, states, the execution engine
// (plan -> encode -> launch), the NCCL remap exchange and the reductions.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tqd.h"
#include "comm.h"
#include "plan.h"
#include "tqd_internal.h"

namespace tqd {
// kernels.cu
cudaError_t launch_sweep(bool dbl, bool bwd, const DevStage *d_stage, const void *d_kops, const int32_t *d_slots,
                         void *psi, void *lam, double *grad, uint64_t rank_hi, const ScatterInfo &sc, int k, int W,
                         int n_ops, int n_slots, int nseg, int n_cvals, int grid, cudaStream_t s);
int sweep_max_ctas_per_sm(bool dbl, bool bwd, int k, int W, int n_ops, int n_slots, int nseg, int n_cvals);
cudaError_t launch_small(bool dbl, bool bwd, const DevOp *d_ops, int n_ops, void *psi, void *lam, double *grad, int n_loc,
                         uint64_t rank_hi, int batch, cudaStream_t s);
cudaError_t launch_lambda_init(bool dbl, const void *psi, void *lam, uint64_t n, uint64_t rank_hi, const ZTerms &t,
                               double *eout, cudaStream_t s);
cudaError_t launch_expval_z(bool dbl, const void *psi, uint64_t n, uint64_t rank_hi, const uint64_t *d_z, int T,
                            double *out, cudaStream_t s);
cudaError_t launch_expval_xy(bool dbl, const void *psi, const void *peer, uint64_t n, uint64_t rank_hi, uint64_t xloc,
                             const uint64_t *d_z, const int *d_ny, int T, double *out, cudaStream_t s);
cudaError_t launch_lambda_add_xy(bool dbl, const void *psi, const void *peer, void *lam, uint64_t n, uint64_t rank_hi,
                                 uint64_t xloc, uint64_t xfull, const uint64_t *d_z, const int *d_ny, const double *d_c,
                                 int T, double *eout, cudaStream_t s);
cudaError_t launch_gather(bool dbl, const void *psi, void *out, uint64_t first, uint64_t count, const GatherMap &gm,
                          cudaStream_t s);
cudaError_t launch_chunk_mass(bool dbl, const void *psi, uint64_t n_chunks, int csz, double *out, cudaStream_t s);
cudaError_t launch_chunk_sample(bool dbl, const void *psi, int n_active, const uint64_t *chunk_id, const uint32_t *off,
                                const double *r, const uint64_t *shot_idx, uint64_t rank_hi, const GatherMap &gm,
                                int csz, double *out, cudaStream_t s);
int sample_chunk_amps();
cudaError_t launch_gauss_sums(bool dbl, const void *psi, uint64_t n, uint64_t rank_hi, const GatherMap &gm, uint64_t seed,
                              const int *qpos, int nq, double *out, cudaStream_t s);
cudaError_t launch_lambda_gauss(bool dbl, const void *psi, void *lam, uint64_t n, uint64_t rank_hi, const GatherMap &gm,
                                uint64_t seed, const ZTerms &t, double alpha, double fc, double k2, double kc,
                                cudaStream_t s);
cudaError_t launch_set_one(bool dbl, void *psi, cudaStream_t s);
cudaError_t launch_remap_block(bool dbl, void *shard, void *stage, uint64_t e0, uint64_t cnt, uint64_t bdep, uint64_t rest,
                              bool unpack, cudaStream_t s);
cudaError_t launch_debug_delay(uint32_t us, cudaStream_t s);
cudaError_t launch_prefix_init(bool dbl, void *psi, uint64_t n, int ng, const void *tab, double cre, double cim,
                               cudaStream_t s);
cudaError_t launch_prefix_contract(bool dbl, const void *lam, uint64_t n, int ng, const void *tab, double *M, int sms,
                                   cudaStream_t s);
cudaError_t dense_tc_upload(const double *U, int m, void **bsplit, cudaStream_t s);
cudaError_t dense_tc_launch(float *x, uint64_t n_amps, const void *bsplit, int prec, int sms, cudaStream_t s);
cudaError_t launch_circuit(bool dbl, const DevOp *fops, int n_f, const DevOp *bops, int n_b, const void *psi,
                           const ZTerms *zts, double *eval, double *grad, int n_loc, uint64_t rank_hi, int batch,
                           cudaStream_t s);
size_t circuit_l3_smem(bool dbl, int n_loc, int nops, int n_rows, int n_gt, int n_acc);
cudaError_t launch_circuit_l3(bool dbl, const L3Op *ops, int n_f, int n_b, const uint32_t *xtab, const uint16_t *xreg,
                              int n_rows, const uint16_t *accp, int n_acc, const double *gtab, int n_gt, const void *psi,
                              const ZTerms *zts, double *eval, double *grad, int n_loc, int batch, cudaStream_t s);
}  // namespace tqd

using namespace tqd;

static thread_local std::string g_err;

static int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

struct tqd_ctx {
    int world = 1, rank = 0, device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    Comm *comm = nullptr;  // world > 1: NCCL, or the in-process loopback (comm.h)
    bool poisoned = false;
    int sms = 148;
};

enum Cat { CAT_FWD = 0, CAT_BWD = 1, CAT_OTHER = 2, CAT_A2A = 3 };

// product-state prefix: one gate of the prefix as a 1-qubit op on product factor `slot`
struct PfOp {
    int gate, slot;
    cd M[4];
};

struct tqd_state {
    tqd_ctx *ctx = nullptr;
    int n = 0, n_loc = 0, g = 0;
    bool dbl = false;
    size_t esz = 8;
    void *psi = nullptr, *lam = nullptr;
    // bounded exchange staging (world > 1): [send half | receive half], stg_bytes in all
    void *stg = nullptr;
    size_t stg_bytes = 0;
    bool own_psi = false, own_lam = false, own_stg = false;
    void *user_buf = nullptr;
    size_t user_bytes = 0;
    std::vector<GateRec> gates;
    int batch = 1;                              // states in the batch (one tape, B shards)
    std::vector<std::vector<GateRec>> brec;     // per gate: B per-state records (batched gates) or empty
    int n_params = 0;
    size_t executed = 0;
    std::vector<Stage> history;
    std::vector<int> pos;
    bool consumed = false;
    // options
    int opt_k = 12, opt_small = 8, opt_profile = 0, opt_grid = 0, opt_graph = 0, opt_fused = 1, opt_absorb = 1;
    size_t opt_stage = 0;  // TQD_OPT_STAGING_BYTES (0 = default)
    int opt_circuit = 10;  // TQD_OPT_CIRCUIT_MAX: single-launch fwd+grad up to this many local qubits
    // single-launch circuit path: forward + backward op lists and Z terms on the device
    void *circ_dev = nullptr;
    size_t circ_cap = 0;
    uint64_t circ_key = 0;
    int circ_nf = 0, circ_nb = 0;
    size_t circ_off_b = 0, circ_off_z = 0;
    std::vector<int> circ_pos;  // qubit map after the cached circuit
    // layout-circuit variant (circuit_l3_kernel) of the cached circuit
    bool circ_l3 = false;
    int l3_nf = 0, l3_nb = 0, l3_rows = 0, l3_nacc = 0, l3_ngt = 0;
    size_t l3_off_x = 0, l3_off_r = 0, l3_off_a = 0, l3_off_g = 0;
    // product-state prefix of the current execution (prefix_build)
    int opt_prefix = 2;            // TQD_OPT_PRODUCT_PREFIX: 0 off, 1 on, 2 auto (on from 22 local qubits)
    int opt_layout = 0;            // TQD_OPT_CIRCUIT_LAYOUT (experiment, measured slower)
    uint64_t pf_dec_sig = 0;       // auto prefix: circuit structure of the cached decision
    bool pf_dec = false;           // auto prefix: keep it (cheaper plan)
    bool pf_on = false;
    std::vector<char> pf_in;       // per gate: in the prefix
    std::vector<std::vector<cd>> pf_s;    // per batch element, per qubit: s_q (2 entries) at the boundary
    std::vector<std::vector<PfOp>> pf_ops; // per batch element: the prefix as 1-qubit ops on product
                                           // factors, in gate order (same structure for every element)
    std::vector<int> pf_slot_of;   // per qubit: its product factor at the boundary
    int pf_ng = 0;
    void *pf_dev = nullptr;        // group tables (device, state dtype) + M environments (fp64)
    size_t pf_cap = 0;
    // fused forward sweep -> remap (peer memory): every rank's two shard allocations
    // (first psi, first lambda), shared once; the forward stores into the owners'
    // lambda-role buffer (idle until the adjoint seed) and the roles swap.  The
    // current role of a buffer is looked up by pointer identity.
    std::vector<void *> peer_pl;  // [rank * 2 + i], i = 0: first psi, 1: first lambda
    void *psi_first = nullptr, *lam_first = nullptr;
    tqd_metrics met;
    double *d_red = nullptr;  // reductions: values / grads
    uint64_t *d_xy = nullptr;  // X/Y adjoint-seed term scratch: z masks, coefficients, #Y
    size_t red_count = 0;
    // plan / descriptor caches (tqd_state_rewind replays the same tape)
    uint64_t tape_version = 1;
    uint64_t fwd_cache_version = 0, bwd_cache_version = ~0ull;
    bool history_cached = false;
    std::vector<Stage> cached_stages, rev_stages;
    std::vector<int> cached_pos;
    uint64_t plan_sig = 0;  // plan_signature of cached_stages
    uint64_t fwd_vhash = 0, bwd_vhash = 0;  // tape_values_hash of the resident descriptors
    uint64_t cached_tmix = 0;  // absorbed-tail length mix of the cached plan (execute_pending)
    struct Encoded *enc_fwd = nullptr, *enc_bwd = nullptr, *enc_tmp = nullptr;
    // TQD_OPT_USE_GRAPH: the cached forward / reverse launch sequences as CUDA graphs
    cudaGraphExec_t g_fwd = nullptr, g_bwd = nullptr;
    uint64_t g_fwd_key = 0, g_bwd_key = 0;
    tqd_metrics g_fwd_delta, g_bwd_delta;
    // profiling
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<int, int>> ev_used;  // (start index, category); stop = start+1
    size_t ev_next = 0;
};

#define CUDA_TRY(st, call)                                                                            \
    do {                                                                                              \
        cudaError_t e_ = (call);                                                                      \
        if (e_ != cudaSuccess) {                                                                      \
            (st)->ctx->poisoned = true;                                                               \
            return fail(TQD_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));            \
        }                                                                                             \
    } while (0)

#define COMM_TRY(st, call)                                                                            \
    do {                                                                                              \
        if ((call) != 0) {                                                                            \
            (st)->ctx->poisoned = true;                                                               \
            return fail(TQD_ERR_NCCL, (st)->ctx->comm->err);                                          \
        }                                                                                             \
    } while (0)

static int check_live(const tqd_state *st) {
    if (!st) return fail(TQD_ERR_ARG, "state is NULL");
    if (st->ctx->poisoned) return fail(TQD_ERR_STATE, "context poisoned by an earlier CUDA/NCCL error");
    return TQD_OK;
}

// ---- profiling events ------------------------------------------------------
static int ev_begin(tqd_state *st, int cat) {
    if (!st->opt_profile) return -1;
    if (st->ev_next + 2 > st->ev_pool.size()) {
        for (int i = 0; i < 64; i++) {
            cudaEvent_t e;
            if (cudaEventCreate(&e) != cudaSuccess) return -1;
            st->ev_pool.push_back(e);
        }
    }
    const int idx = (int)st->ev_next;
    st->ev_next += 2;
    cudaEventRecord(st->ev_pool[idx], st->ctx->stream);
    st->ev_used.push_back({idx, cat});
    return idx;
}
static void ev_end(tqd_state *st, int idx) {
    if (idx < 0) return;
    cudaEventRecord(st->ev_pool[idx + 1], st->ctx->stream);
}
static int ev_collect(tqd_state *st) {
    if (st->ev_used.empty()) return TQD_OK;
    CUDA_TRY(st, cudaEventSynchronize(st->ev_pool[st->ev_used.back().first + 1]));
    for (auto &u : st->ev_used) {
        float ms = 0;
        cudaEventElapsedTime(&ms, st->ev_pool[u.first], st->ev_pool[u.first + 1]);
        switch (u.second) {
        case CAT_FWD: st->met.fwd_sweep_ms += ms; break;
        case CAT_BWD: st->met.bwd_sweep_ms += ms; break;
        case CAT_A2A: st->met.a2a_ms += ms; break;
        default: st->met.other_ms += ms; break;
        }
    }
    st->ev_used.clear();
    st->ev_next = 0;
    return TQD_OK;
}

static PlanConfig make_plan_cfg(int n, int n_loc, int k, int small_max, bool dbl) {
    PlanConfig c;
    const size_t esz = dbl ? 16 : 8;
    c.n = n;
    c.n_loc = n_loc;
    c.k = k;
    c.R = TQD_SWEEP_R;
    c.small_max = small_max;
    c.c128 = dbl;
    c.swz_bits = dbl ? 3 : 4;
    {
        // pinned low bits: 2^c amplitudes per contiguous run = one 128 B line (c64: 4, c128: 3)
        const char *e = getenv("TQD_C_LOW");
        c.c_low = e ? std::max(1, std::min(5, atoi(e))) : (dbl ? 3 : 4);
    }
    // shared-memory budget of the adjoint sweep kernel (the larger of the two):
    // psi + lambda exchange tiles, the stage's kernel ops, per-thread gradient
    // accumulators and per-thread layout constants, within ~200 KB per CTA
    if (dbl && c.k > 11) c.k = 11;
    if (c.k > c.n_loc) c.k = c.n_loc;
    if (c.k - LANE_BITS - c.R > WMAX) c.k = LANE_BITS + c.R + WMAX;
    const size_t threads = (size_t)32 << std::max(0, c.k - LANE_BITS - c.R);
    const size_t exch = ((size_t)2 << c.k) * esz;
    // layout constants + prefetch offsets; the diagonal-block C rows / U values
    // (<= 16.5 KB) live in the headroom between this 200 KB budget and the 227 KB opt-in
    const size_t tables = (size_t)3 * MAXSEG * threads * 4 + (size_t)3 * threads * 8;
    const size_t kop = dbl ? sizeof(KOp<double>) : sizeof(KOp<float>);
    const size_t real = esz / 2;
    static const char *bkb = getenv("TQD_EXPERIMENT_SMEM_KB");  // timing experiments only
    const size_t cap = (size_t)(bkb ? atoi(bkb) : 200) * 1024;
    const size_t budget = cap - std::min(cap - 32 * 1024, exch + tables);
    c.max_slots = (int)std::min<size_t>(MAX_STAGE_SLOTS, (budget / 3) / (threads * real));
    c.max_slots = std::max(c.max_slots, 3);
    c.max_ops = (int)std::min<size_t>(MAX_STAGE_OPS, (budget - (size_t)c.max_slots * threads * real) / kop);
    c.max_ops = std::max(c.max_ops, 8);
    return c;
}

static PlanConfig plan_cfg(const tqd_state *st) {
    return make_plan_cfg(st->n, st->n_loc, st->opt_k, st->opt_small, st->dbl);
}

static int ensure_red(tqd_state *st, size_t count) {
    if (count <= st->red_count) return TQD_OK;
    if (st->d_red) {
        CUDA_TRY(st, cudaStreamSynchronize(st->ctx->stream));
        cudaFree(st->d_red);
        st->d_red = nullptr;
    }
    size_t nc = std::max(count, (size_t)4096);
    if (cudaMalloc(&st->d_red, nc * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        st->red_count = 0;
        return fail(TQD_ERR_OOM, "cannot allocate reduction buffer");
    }
    st->red_count = nc;
    return TQD_OK;
}

static uint64_t shard_bytes(const tqd_state *st) { return ((uint64_t)1 << st->n_loc) * st->esz; }
// every buffer holds the shards of all batch elements back to back
static uint64_t all_bytes(const tqd_state *st) { return shard_bytes(st) * (uint64_t)st->batch; }

// Exchange staging (world > 1): bounded, independent of the shard size -- the
// remap and the partner-shard exchange of X / Y strings move their blocks through
// it chunk by chunk (SURVEY.md §8(e) memory: at 36 qubits on 8 GPUs psi + lambda are
// 2 x 64 GiB per GPU; two shard-sized staging buffers would not fit).
static constexpr size_t kDefaultStagingBytes = (size_t)1 << 30;  // send half + receive half
static size_t staging_bytes_for(size_t shard, size_t esz, size_t opt) {
    size_t b = opt ? opt : kDefaultStagingBytes;
    b = std::min(b, 2 * shard);
    b = std::max(b, 2 * esz);  // at least one amplitude per half
    return b & ~(2 * esz - 1);
}

static int ensure_staging(tqd_state *st) {
    const size_t want = staging_bytes_for(shard_bytes(st), st->esz, st->opt_stage);
    if (st->stg && st->stg_bytes >= want) return TQD_OK;
    if (st->stg && st->own_stg) {
        CUDA_TRY(st, cudaStreamSynchronize(st->ctx->stream));
        cudaFree(st->stg);
        st->met.peak_device_bytes -= st->stg_bytes;
    }
    st->stg = nullptr;
    if (cudaMalloc(&st->stg, want) != cudaSuccess) {
        cudaGetLastError();
        st->stg_bytes = 0;
        return fail(TQD_ERR_OOM, "cannot allocate the exchange staging buffer");
    }
    st->own_stg = true;
    st->stg_bytes = want;
    st->met.peak_device_bytes += want;
    return TQD_OK;
}

static int ensure_xy_scratch(tqd_state *st) {
    if (st->d_xy) return TQD_OK;
    if (cudaMalloc(&st->d_xy, 48 * sizeof(uint64_t)) != cudaSuccess) {
        cudaGetLastError();
        return fail(TQD_ERR_OOM, "cannot allocate the X/Y term scratch");
    }
    return TQD_OK;
}

static int ensure_lambda(tqd_state *st) {
    if (st->lam) return TQD_OK;
    const size_t b = all_bytes(st);
    if (cudaMalloc(&st->lam, b) != cudaSuccess) {
        cudaGetLastError();
        return fail(TQD_ERR_OOM, "cannot allocate the adjoint state lambda");
    }
    st->own_lam = true;
    st->lam_first = st->lam;
    st->met.peak_device_bytes += b;
    return TQD_OK;
}

static uint64_t rank_hi(const tqd_state *st) { return (uint64_t)st->ctx->rank << st->n_loc; }

// ---- remap exchange -------------------------------------
// Swapping global positions gpos[i] with local positions lpos[i]: rank r sends
// its block b (= the values of its lpos-bits) to the peer whose gpos-bits equal
// b; the block received from a peer lands at block index u = that peer's
// gpos-bits (the values the lpos-bits take after the swap).  Pure integer
// schedule, shared by the device path and tqd_debug_remap_schedule.
static void remap_schedule(int rank, int n_loc, const RemapPlan &rp, std::vector<int> &peer, std::vector<int> &recv_block) {
    const int nb = 1 << rp.m;
    peer.assign(nb, 0);
    recv_block.assign(nb, 0);
    for (int b = 0; b < nb; b++) {
        int pr = rank;
        for (int i = 0; i < rp.m; i++) {
            const int gb = rp.gpos[i] - n_loc;
            pr = (pr & ~(1 << gb)) | (((b >> i) & 1) << gb);
        }
        int u = 0;
        for (int i = 0; i < rp.m; i++) u |= ((pr >> (rp.gpos[i] - n_loc)) & 1) << i;
        peer[b] = pr;
        recv_block[b] = u;
    }
}

// One remap of one shard through the bounded staging: with every partner of the
// rank group (XOR schedule s = 1 .. 2^m - 1; the partner's gpos-bits are
// b = mine ^ s) this rank swaps its block b -- send block b, receive the partner's
// block (its lpos-bits = my gpos-bits) into the same place -- chunk by chunk:
// pack -> grouped send/recv (NCCL over NVLink) -> unpack.  Block b = mine stays.
static int exec_remap_one(tqd_state *st, const RemapPlan &rp, void *buf) {
    int rc = ensure_staging(st);
    if (rc) return rc;
    tqd_ctx *c = st->ctx;
    uint64_t lmask = 0;
    for (int i = 0; i < rp.m; i++) lmask |= 1ull << rp.lpos[i];
    const uint64_t rest = ((st->n_loc >= 64 ? 0 : (1ull << st->n_loc)) - 1) & ~lmask;
    const uint64_t blk = (uint64_t)1 << (st->n_loc - rp.m);
    const uint64_t chunk = std::min<uint64_t>(blk, (st->stg_bytes / 2) / st->esz);
    char *sb = (char *)st->stg, *rb = (char *)st->stg + st->stg_bytes / 2;
    int mine = 0;
    for (int i = 0; i < rp.m; i++) mine |= ((c->rank >> (rp.gpos[i] - st->n_loc)) & 1) << i;
    const char *dly = getenv("TQD_DEBUG_REMAP_DELAY_US");  // race tests: odd ranks lag before unpacking
    const uint32_t delay_us = (dly && (c->rank & 1)) ? (uint32_t)atoi(dly) : 0;
    const int ev = ev_begin(st, CAT_A2A);
    for (int sx = 1; sx < (1 << rp.m); sx++) {
        const int b = mine ^ sx;
        int peer = c->rank;
        uint64_t bdep = 0;
        for (int i = 0; i < rp.m; i++) {
            const int gb = rp.gpos[i] - st->n_loc;
            peer = (peer & ~(1 << gb)) | (((b >> i) & 1) << gb);
            if ((b >> i) & 1) bdep |= 1ull << rp.lpos[i];
        }
        for (uint64_t e0 = 0; e0 < blk; e0 += chunk) {
            const uint64_t cnt = std::min(chunk, blk - e0);
            const size_t bytes = cnt * st->esz;
            CUDA_TRY(st, launch_remap_block(st->dbl, buf, sb, e0, cnt, bdep, rest, false, c->stream));
            COMM_TRY(st, c->comm->group_start());
            COMM_TRY(st, c->comm->send(sb, bytes, peer, c->stream));
            COMM_TRY(st, c->comm->recv(rb, bytes, peer, c->stream));
            COMM_TRY(st, c->comm->group_end(c->stream));
            if (delay_us) CUDA_TRY(st, launch_debug_delay(delay_us, c->stream));
            CUDA_TRY(st, launch_remap_block(st->dbl, buf, rb, e0, cnt, bdep, rest, true, c->stream));
            st->met.a2a_bytes += bytes;
            st->met.hbm_bytes += 4 * bytes;
            st->met.kernel_launches += 2;
        }
    }
    ev_end(st, ev);
    return TQD_OK;
}

// a remap of every batch element's shard
static int exec_remap(tqd_state *st, const RemapPlan &rp, void *buf) {
    for (int b = 0; b < st->batch; b++) {
        const int rc = exec_remap_one(st, rp, (char *)buf + (size_t)b * shard_bytes(st));
        if (rc) return rc;
    }
    return TQD_OK;
}

// X / Y strings acting on rank bits pair this shard with the partner rank's
// (rank ^ gx): local index i meets the partner's i ^ xl.  Chunk by chunk through
// the staging receive half: in step j both ranks send their chunk j ^ (xl's bits
// above the chunk) and run `fn` on their own chunk j against the received one
// (fn(psi_off, peer_chunk, count, xl within the chunk); the kernels see the chunk's
// full index through rank_hi | psi_off).
template <typename F>
static int xy_partner_chunks(tqd_state *st, const void *psi_b, int gx, uint64_t xl, F &&fn) {
    int rc = ensure_staging(st);
    if (rc) return rc;
    tqd_ctx *c = st->ctx;
    const uint64_t N = 1ull << st->n_loc;
    uint64_t C = 1;  // power of two <= the receive half
    while (C * 2 * st->esz <= st->stg_bytes / 2 && C * 2 <= N) C *= 2;
    const uint64_t hi = xl & ~(C - 1), lo = xl & (C - 1);
    void *rb = (char *)st->stg + st->stg_bytes / 2;
    const int partner = c->rank ^ gx;
    for (uint64_t j0 = 0; j0 < N; j0 += C) {
        COMM_TRY(st, c->comm->group_start());
        COMM_TRY(st, c->comm->send((const char *)psi_b + (j0 ^ hi) * st->esz, C * st->esz, partner, c->stream));
        COMM_TRY(st, c->comm->recv(rb, C * st->esz, partner, c->stream));
        COMM_TRY(st, c->comm->group_end(c->stream));
        st->met.a2a_bytes += C * st->esz;
        rc = fn(j0, (const void *)rb, C, lo);
        if (rc) return rc;
    }
    return TQD_OK;
}

// ---- forward execution ------------------------------------------------------
static int sweep_grid(tqd_state *st, const SweepPlan &sp, bool bwd, int n_ops, int n_slots, int n_cvals) {
    if (st->opt_grid > 0) return std::max(1, st->opt_grid / st->batch) * st->batch;
    int per = sweep_max_ctas_per_sm(st->dbl, bwd, sp.k, sp.W, n_ops, n_slots, (int)sp.lays.size(), n_cvals);
    if (per < 1) per = 1;
    int64_t g = (int64_t)per * st->ctx->sms;
    const int64_t tiles = (int64_t)1 << (st->n_loc - sp.k);
    // a batch of B states: the grid is a multiple of B (CTA i serves state i % B)
    int64_t per_state = std::max<int64_t>(1, g / st->batch);
    if (per_state > tiles) per_state = tiles;
    return (int)(per_state * st->batch);
}

// the tape as seen by batch element b (batched gates replaced by element b's record)
static const std::vector<GateRec> &gates_for(tqd_state *st, int b, std::vector<GateRec> &tmp) {
    bool any = false;
    for (const auto &v : st->brec) if (!v.empty()) { any = true; break; }
    if (!any || b == 0) return st->gates;
    tmp = st->gates;
    for (size_t i = 0; i < tmp.size() && i < st->brec.size(); i++)
        if (!st->brec[i].empty()) tmp[i] = st->brec[i][b];
    return tmp;
}

// gate i as seen by batch element b (no copy of the tape)
static const GateRec &gate_of(const tqd_state *st, size_t i, int b) {
    if (b > 0 && i < st->brec.size() && !st->brec[i].empty()) return st->brec[i][b];
    return st->gates[i];
}

// Encoded launch list: descriptors of a stage list, uploaded once to the device.
struct Encoded {
    void *dev = nullptr;
    size_t cap = 0;
    size_t off_ops = 0, off_sl = 0;
    size_t off_kops = 0;
    struct L { int type; int idx; int op_base; int n_ops; int stage; int grid; int n_slots; int no_store = 0; int n_cvals = 0; };
    std::vector<L> launches;
    bool valid = false;
    // pinned host staging of the descriptors (async copy); the event guards its reuse
    void *host = nullptr;
    size_t host_cap = 0;
    cudaEvent_t copied = nullptr;
};

static int encode_upload(tqd_state *st, const std::vector<Stage> &stages, bool bwd, Encoded &E);

// Launch an encoded stage list (forward or backward) on the context stream.
// The remap right after a sweep is fused into it: the sweep stores every amplitude
// straight into its post-remap owner's receive buffer (peer memory over NVLink; the
// loopback world: the same device), then one barrier and a pointer swap replace the
// pack -> all-to-all -> unpack of exec_remap.
// Forward only: the stores go into the owners' lambda-role buffer, which holds
// nothing until the adjoint seed (no extra memory).  In the adjoint psi and lambda
// are both live, so its remaps run through the bounded staging.
static bool fusable_remap(const tqd_state *st, bool bwd) {
    return !bwd && st->opt_fused && st->ctx->world > 1 && st->ctx->world <= SCATTER_MAX_RANKS && st->own_psi &&
           (!st->lam || st->own_lam);
}

// 1 = peer memory unavailable on some rank (same on every rank): fusion is turned
// off for this state and the remap runs as pack -> all-to-all -> unpack
static int share_pair(tqd_state *st, void *a, void *b, std::vector<void *> &table) {
    if (!table.empty()) return TQD_OK;
    void *loc[2] = {a, b};
    const int rc = st->ctx->comm->share_buffers(loc, 2, table, st->ctx->stream);
    if (rc == 2) {
        st->opt_fused = 0;
        return 1;
    }
    COMM_TRY(st, rc);
    return TQD_OK;
}

static uint64_t peer_of(const std::vector<void *> &table, void *psi_first, void *cur, int r) {
    // the role of a buffer is symmetric over the ranks: same slot on every rank
    return (uint64_t)table[r * 2 + (cur == psi_first ? 0 : 1)];
}

static int launch_encoded(tqd_state *st, const std::vector<Stage> &stages, bool bwd, const Encoded &E, double *d_grad) {
    tqd_ctx *c = st->ctx;
    const DevStage *d_st = (const DevStage *)E.dev;
    const DevOp *d_ops = (const DevOp *)((char *)E.dev + E.off_ops);
    const char *d_kops = (const char *)E.dev + E.off_kops;
    const int32_t *d_sl = (const int32_t *)((char *)E.dev + E.off_sl);
    const uint64_t sb = all_bytes(st);
    for (size_t li = 0; li < E.launches.size(); li++) {
        const Encoded::L &l = E.launches[li];
        const Stage &s = stages[l.stage];
        if (l.type == ST_SWEEP) {
            const SweepPlan &sp = s.sw;
            ScatterInfo sc;
            memset(&sc, 0, sizeof(sc));
            bool fuse = li + 1 < E.launches.size() && E.launches[li + 1].type == ST_REMAP && fusable_remap(st, bwd);
            if (fuse && !st->lam) {  // the lambda buffer (the fwd+grad budget) receives the remap
                const int rc = ensure_lambda(st);
                if (rc) return rc;
            }
            if (fuse) {
                const int rc = share_pair(st, st->psi_first, st->lam_first, st->peer_pl);
                if (rc < 0) return rc;
                fuse = rc == 0;  // 1: no peer memory, the remap launch below runs unfused
            }
            if (fuse) {
                const RemapPlan &rp = stages[E.launches[li + 1].stage].rm;
                sc.m = rp.m;
                sc.n_loc = st->n_loc;
                for (int i = 0; i < rp.m && i < 8; i++) { sc.gbit[i] = (uint8_t)rp.gpos[i]; sc.lbit[i] = (uint8_t)rp.lpos[i]; }
                for (int r = 0; r < c->world; r++) sc.dst_psi[r] = peer_of(st->peer_pl, st->psi_first, st->lam, r);
            }
            const int ev = ev_begin(st, bwd ? CAT_BWD : CAT_FWD);
            CUDA_TRY(st, launch_sweep(st->dbl, bwd, d_st + l.idx, d_kops, d_sl, st->psi, st->lam, d_grad, rank_hi(st),
                                      sc, sp.k, sp.W, l.n_ops, l.n_slots, (int)sp.lays.size(), l.n_cvals, l.grid,
                                      c->stream));
            ev_end(st, ev);
            if (fuse) {
                // every rank's stores into its peers' lambda-role buffers are complete
                // (and every rank finished reading its psi, the next target)
                COMM_TRY(st, c->comm->barrier(c->stream));
                std::swap(st->psi, st->lam);
                const uint64_t moved = sb - (sb >> sc.m);
                st->met.a2a_bytes += moved;
                st->met.remaps++;
                st->met.fused_remaps++;
                li++;  // the remap is done
            }
            const uint64_t bb = (l.no_store == 1 ? 2 : l.no_store == 2 ? 3 : 4) * sb;  // the last reverse sweep stores less
            if (bwd) { st->met.bwd_sweeps++; st->met.bwd_sweep_bytes += bb; st->met.hbm_bytes += bb; st->met.gates_unapplied += sp.n_gates; }
            else { st->met.fwd_sweeps++; st->met.fwd_sweep_bytes += 2 * sb; st->met.hbm_bytes += 2 * sb; st->met.gates_applied += sp.n_gates; }
            st->met.kernel_launches++;
        } else if (l.type == ST_SMALL) {
            const int ev = ev_begin(st, bwd ? CAT_BWD : CAT_FWD);
            CUDA_TRY(st, launch_small(st->dbl, bwd, d_ops + l.op_base, l.n_ops, st->psi, st->lam, d_grad, st->n_loc,
                                      rank_hi(st), st->batch, c->stream));
            ev_end(st, ev);
            if (bwd) { st->met.bwd_sweeps++; st->met.bwd_sweep_bytes += 4 * sb; st->met.hbm_bytes += 4 * sb; st->met.gates_unapplied += s.sm.n_gates; }
            else { st->met.fwd_sweeps++; st->met.fwd_sweep_bytes += 2 * sb; st->met.hbm_bytes += 2 * sb; st->met.gates_applied += s.sm.n_gates; }
            st->met.kernel_launches++;
        } else {
            int rc = exec_remap(st, s.rm, st->psi);
            if (rc) return rc;
            if (bwd) { rc = exec_remap(st, s.rm, st->lam); if (rc) return rc; }
            st->met.remaps++;
        }
    }
    return TQD_OK;
}

// Replays of a cached launch sequence as one CUDA graph (TQD_OPT_USE_GRAPH; one
// rank, no profiling events): captured on first use, relaunched while the key
// (plan structure, descriptor / state / gradient buffers) is unchanged.  The
// descriptors are read from device memory at run time, so new parameter values
// uploaded into the same buffer need no re-capture.  Host-side metrics of the
// captured launches are re-added on every replay.
static void add_counts(tqd_metrics &m, const tqd_metrics &d, int sign) {
    auto f = [&](uint64_t &x, uint64_t y) { x = sign > 0 ? x + y : x - y; };
    f(m.fwd_sweeps, d.fwd_sweeps); f(m.bwd_sweeps, d.bwd_sweeps); f(m.remaps, d.remaps);
    f(m.gates_applied, d.gates_applied); f(m.gates_unapplied, d.gates_unapplied); f(m.hbm_bytes, d.hbm_bytes);
    f(m.a2a_bytes, d.a2a_bytes); f(m.fwd_sweep_bytes, d.fwd_sweep_bytes); f(m.bwd_sweep_bytes, d.bwd_sweep_bytes);
    f(m.kernel_launches, d.kernel_launches); f(m.fused_remaps, d.fused_remaps);
}

static int launch_graphed(tqd_state *st, const std::vector<Stage> &stages, bool bwd, const Encoded &E, double *d_grad,
                          cudaGraphExec_t &ge, uint64_t &gkey, tqd_metrics &delta) {
    if (!st->opt_graph || st->ctx->world != 1 || st->opt_profile) return launch_encoded(st, stages, bwd, E, d_grad);
    uint64_t key = st->plan_sig ^ (st->cached_tmix * 3) ^ 0x51ED27ull;
    for (uint64_t v : {(uint64_t)E.dev, (uint64_t)st->psi, (uint64_t)st->lam, (uint64_t)d_grad, (uint64_t)E.launches.size(),
                       (uint64_t)stages.size(), (uint64_t)E.off_ops, (uint64_t)E.off_kops, (uint64_t)E.off_sl})
        key = (key ^ v) * 1099511628211ull;
    for (const Encoded::L &l : E.launches)  // every captured launch parameter
        for (uint64_t v : {(uint64_t)l.type, (uint64_t)l.idx, (uint64_t)l.op_base, (uint64_t)l.n_ops, (uint64_t)l.stage,
                           (uint64_t)l.grid, (uint64_t)l.n_slots, (uint64_t)l.no_store, (uint64_t)(int64_t)l.n_cvals})
            key = (key ^ v) * 1099511628211ull;
    cudaStream_t s = st->ctx->stream;
    if (ge && gkey == key) {
        CUDA_TRY(st, cudaGraphLaunch(ge, s));
        add_counts(st->met, delta, +1);
        return TQD_OK;
    }
    const tqd_metrics before = st->met;
    CUDA_TRY(st, cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    const int rc = launch_encoded(st, stages, bwd, E, d_grad);
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(s, &g);
    if (rc) {
        if (e == cudaSuccess && g) cudaGraphDestroy(g);
        return rc;
    }
    CUDA_TRY(st, e);
    if (ge) cudaGraphExecDestroy(ge);
    ge = nullptr;
    const cudaError_t ei = cudaGraphInstantiate(&ge, g, 0);
    cudaGraphDestroy(g);
    CUDA_TRY(st, ei);
    delta = st->met;
    add_counts(delta, before, -1);
    gkey = key;
    CUDA_TRY(st, cudaGraphLaunch(ge, s));
    return TQD_OK;
}

// the product prefix holds trainable gates (the adjoint then runs down to its boundary)
static bool prefix_has_grads(const tqd_state *st) {
    if (!st->pf_on) return false;
    for (size_t i = 0; i < st->pf_in.size(); i++)
        if (st->pf_in[i] && st->gates[i].ngen) return true;
    return false;
}

template <typename Real>
static void encode_all(tqd_state *st, const std::vector<Stage> &stages, bool bwd, Encoded &E,
                       std::vector<DevStage> &dstages, std::vector<DevOp> &ops, std::vector<KOp<Real>> &kops,
                       std::vector<int32_t> &slots) {
    std::vector<GateRec> tmp;
    // reverse sweep: nothing before the earliest trainable gate is un-applied, and
    // the last reverse sweep stores neither psi nor lambda (only gradients remain)
    int skip_below = 0, last_sweep = -1;
    if (bwd) {
        // (prefix gradients need lambda at the prefix boundary: every gate un-applied)
        skip_below = prefix_has_grads(st) ? 0 : (int)st->gates.size();
        for (size_t i = 0; i < (size_t)skip_below; i++)
            if (st->gates[i].ngen) { skip_below = (int)i; break; }
        for (size_t ii = 0; ii < stages.size(); ii++)
            if (stages[ii].type != ST_REMAP) last_sweep = (int)ii;
    }
    for (size_t ii = 0; ii < stages.size(); ii++) {
        const Stage &s = stages[ii];
        if (s.type == ST_SWEEP) {
            if (s.sw.ops.empty()) continue;
            // one copy of the op stream / slot table per batch element (same structure)
            DevStage ds;
            encode_sweep_k<Real>(s.sw, gates_for(st, 0, tmp), bwd, st->n_loc, ds, kops, slots, skip_below);
            for (int b = 1; b < st->batch; b++) {
                DevStage dsb;
                encode_sweep_k<Real>(s.sw, gates_for(st, b, tmp), bwd, st->n_loc, dsb, kops, slots, skip_below);
            }
            ds.batch = st->batch;
            // (with a product prefix the last reverse sweep stores lambda: its environments
            // give the prefix gates' gradients)
            ds.no_store = (bwd && (int)ii == last_sweep) ? (prefix_has_grads(st) ? 2 : 1) : 0;
            const int ncv = ds.n_dblk ? ds.n_cvals : -1;  // -1: no diagonal blocks (plain kernel)
            E.launches.push_back({ST_SWEEP, (int)dstages.size(), 0, ds.n_ops, (int)ii,
                                  sweep_grid(st, s.sw, bwd, ds.n_ops, ds.n_slots, ncv), ds.n_slots, ds.no_store, ncv});
            dstages.push_back(ds);
        } else if (s.type == ST_SMALL) {
            if (s.sm.ops.empty()) continue;
            const int b = (int)ops.size();
            for (int bb = 0; bb < st->batch; bb++) encode_small(s.sm, gates_for(st, bb, tmp), bwd, ops, skip_below);
            E.launches.push_back({ST_SMALL, -1, b, ((int)ops.size() - b) / st->batch, (int)ii, 1, 0});
        } else {
            E.launches.push_back({ST_REMAP, -1, 0, 0, (int)ii, 0, 0});
        }
    }
}

static int encode_upload(tqd_state *st, const std::vector<Stage> &stages, bool bwd, Encoded &E) {
    // a captured graph carries the launch parameters (op counts, shared-memory sizes,
    // kernel instantiations, descriptor offsets) of the encoding it was captured
    // from: re-encoding into the same buffer invalidates it (values can change the
    // kernel-op structure, e.g. diagonal runs with zero or cancelling terms)
    if (&E == st->enc_fwd && st->g_fwd) { cudaGraphExecDestroy(st->g_fwd); st->g_fwd = nullptr; st->g_fwd_key = 0; }
    if (&E == st->enc_bwd && st->g_bwd) { cudaGraphExecDestroy(st->g_bwd); st->g_bwd = nullptr; st->g_bwd_key = 0; }
    std::vector<DevStage> dstages;
    std::vector<DevOp> ops;
    std::vector<KOp<float>> kf;
    std::vector<KOp<double>> kd;
    std::vector<int32_t> slots;
    E.launches.clear();
    E.valid = false;
    if (st->dbl) encode_all<double>(st, stages, bwd, E, dstages, ops, kd, slots);
    else encode_all<float>(st, stages, bwd, E, dstages, ops, kf, slots);
    const size_t b_st = dstages.size() * sizeof(DevStage);
    const size_t b_ops = ops.size() * sizeof(DevOp);
    const size_t b_k = st->dbl ? kd.size() * sizeof(KOp<double>) : kf.size() * sizeof(KOp<float>);
    const size_t b_sl = slots.size() * sizeof(int32_t);
    E.off_ops = (b_st + 255) & ~(size_t)255;
    E.off_kops = (E.off_ops + b_ops + 255) & ~(size_t)255;
    E.off_sl = (E.off_kops + b_k + 255) & ~(size_t)255;
    const size_t total = E.off_sl + b_sl + 256;
    if (total > E.cap) {
        if (E.dev) {
            CUDA_TRY(st, cudaStreamSynchronize(st->ctx->stream));
            cudaFree(E.dev);
            E.dev = nullptr;
        }
        const size_t nb = std::max(total, (size_t)1 << 20);
        if (cudaMalloc(&E.dev, nb) != cudaSuccess) {
            cudaGetLastError();
            E.cap = 0;
            return fail(TQD_ERR_OOM, "cannot allocate descriptor buffer");
        }
        E.cap = nb;
    }
    // pinned staging: wait until the previous upload from it has been copied
    if (E.copied) CUDA_TRY(st, cudaEventSynchronize(E.copied));
    else CUDA_TRY(st, cudaEventCreateWithFlags(&E.copied, cudaEventDisableTiming));
    if (total > E.host_cap) {
        if (E.host) cudaFreeHost(E.host);
        E.host = nullptr;
        const size_t nb = std::max(total, (size_t)1 << 20);
        if (cudaMallocHost(&E.host, nb) != cudaSuccess) {
            cudaGetLastError();
            E.host_cap = 0;
            return fail(TQD_ERR_OOM, "cannot allocate pinned descriptor staging");
        }
        E.host_cap = nb;
    }
    char *host = (char *)E.host;
    memset(host, 0, total);
    if (b_st) memcpy(host, dstages.data(), b_st);
    if (b_ops) memcpy(host + E.off_ops, ops.data(), b_ops);
    if (b_k) memcpy(host + E.off_kops, st->dbl ? (const void *)kd.data() : (const void *)kf.data(), b_k);
    if (b_sl) memcpy(host + E.off_sl, slots.data(), b_sl);
    // stream-ordered after earlier launches that may still read the device buffer
    CUDA_TRY(st, cudaMemcpyAsync(E.dev, host, total, cudaMemcpyHostToDevice, st->ctx->stream));
    CUDA_TRY(st, cudaEventRecord(E.copied, st->ctx->stream));
    st->met.h2d_bytes += total;
    E.valid = true;
    return TQD_OK;
}

static void free_encoded(Encoded &E) {
    if (E.dev) cudaFree(E.dev);
    if (E.host) cudaFreeHost(E.host);
    if (E.copied) cudaEventDestroy(E.copied);
    E.dev = nullptr;
    E.host = nullptr;
    E.copied = nullptr;
    E.cap = E.host_cap = 0;
    E.valid = false;
}

// structure + every value of the tape: an identical re-recording (reset + the same
// gates) replays the resident descriptors like tqd_state_rewind
static uint64_t tape_values_hash(const tqd_state *st) {
    uint64_t h = plan_signature(st->gates, plan_cfg(st));
    auto mix = [&](double v) {
        uint64_t b;
        memcpy(&b, &v, 8);
        h = (h ^ b) * 1099511628211ull;
    };
    auto rec = [&](const GateRec &g) {
        for (int i = 0; i < 16; i++) { mix(g.M[i].real()); mix(g.M[i].imag()); }
        for (int i = 0; i < 4; i++) { mix(g.sub[i].real()); mix(g.sub[i].imag()); }
        for (int j = 0; j < g.ngen; j++)
            for (int i = 0; i < 4; i++) { mix(g.G[j][i].real()); mix(g.G[j][i].imag()); }
        mix((double)g.slot0);
    };
    for (size_t i = 0; i < st->gates.size(); i++) {
        if (i < st->brec.size() && !st->brec[i].empty())
            for (const GateRec &g : st->brec[i]) rec(g);
        else
            rec(st->gates[i]);
    }
    return h;
}

// ---- product-state prefix (exact) -------------------------------------------
// Every qubit's leading run of 1-qubit gates acts on |0> before the qubit meets any
// multi-qubit gate (the gates of other qubits commute with them), so after those
// gates the state is the product psi_P = (x)_q s_q with s_q = (its gates) |0>
// (e.g. the HEA's first RY + RZ layer, Listing 2's encoder).  A
// fixed 2-qubit gate on two such qubits keeps the product when it only relabels
// (SWAP) or when one of its qubits is in a parameter-independent computational basis
// state |v>: a diagonal gate then acts on the other qubit as diag(d[v,0], d[v,1]), a
// controlled gate with that control as U (v = 1) or I (v = 0).  (A QFT of a basis
// state is a product state this way: each CP meets a still-unrotated control.)  The
// forward writes psi_P directly (prefix_init_kernel, the same HBM pass as the |0..0>
// reset) instead of sweeping those gates; the adjoint stops at the prefix boundary
// and finishes their gradients from the environments of lambda (prefix_contract_kernel,
// one read of lambda): dE/dtheta_j = 2 Re sum_v T_q(v) (d s_q / d theta_j)(v).
// Single state, from |0..0>, local qubits >= 11; with world > 1 the sharded qubits'
// factors are one scalar per rank (c_r), their gradients come from every rank's total
// contraction Z_r (one small all-reduce).
constexpr int PF_BITS_H = 10;
static bool prefix_build(tqd_state *st, size_t end) {
    st->pf_on = false;
    if (!st->opt_prefix || st->executed != 0 || st->n_loc < 11 || st->n_loc > 40) return false;
    // auto: below ~4 M amplitudes per state the host work of the tables and of the
    // environments' contraction costs more than the sweeps it saves (tools/bench_batch.py:
    // batch 16 at 20 q 9.2 -> 10.7 ms per step with it, at 24 q 161 -> 143 ms)
    if (st->opt_prefix == 2 && st->n_loc < 22) return false;
    const int n = st->n;
    st->pf_in.assign(st->gates.size(), 0);
    std::vector<PfOp> ops0;  // element 0 (the structure; batched gates' values per element below)
    // product factors ("slots"): slot f starts as qubit f in |0>; a SWAP of two
    // untouched qubits exchanges their slots
    std::vector<cd> sv(2 * n, cd(0.0));
    std::vector<int> slot_of(n), fixed(n, 1);  // fixed: no trainable gate in the slot's chain yet
    for (int q = 0; q < n; q++) { sv[2 * q] = cd(1.0); slot_of[q] = q; }
    auto zero = [](cd v) { return v.real() == 0.0 && v.imag() == 0.0; };
    // basis bit of a slot whose state is exactly |0> or |1> (up to a phase) and
    // independent of the parameters, else -1
    auto basis = [&](int f) -> int {
        if (!fixed[f]) return -1;
        if (zero(sv[2 * f + 1])) return 0;
        if (zero(sv[2 * f])) return 1;
        return -1;
    };
    auto apply = [&](size_t i, int f, const cd *M) {
        PfOp o;
        o.gate = (int)i;
        o.slot = f;
        for (int j = 0; j < 4; j++) o.M[j] = M[j];
        ops0.push_back(o);
        const cd a = sv[2 * f], b = sv[2 * f + 1];
        sv[2 * f] = M[0] * a + M[1] * b;
        sv[2 * f + 1] = M[2] * a + M[3] * b;
    };
    std::vector<char> touched(n, 0);
    bool any = false;
    for (size_t i = 0; i < end; i++) {
        const GateRec &g = st->gates[i];
        bool free_ = !(g.batched && g.nw != 1);
        for (int j = 0; j < g.nw; j++) free_ = free_ && !touched[g.w[j]];
        bool take = false;
        if (free_ && g.nw == 1) {
            // (a batched gate: per-element values, element 0's here; never a basis control)
            const int f = slot_of[g.w[0]];
            apply(i, f, g.M);
            if (g.ngen || g.batched) fixed[f] = 0;
            take = true;
        } else if (free_ && g.nw == 2) {
            // a fixed 2-qubit gate keeps the product when it is a relabeling or one of
            // its qubits is in a parameter-independent basis state: it then acts on
            // the other factor as the 1-qubit gate selected by that bit (exact)
            const int a = g.w[0], b = g.w[1], fa = slot_of[a], fb = slot_of[b];
            const int va = basis(fa), vb = basis(fb);
            if (g.cls == CL_IDENT) {
                take = true;
            } else if (g.cls == CL_SWAP) {
                std::swap(slot_of[a], slot_of[b]);
                take = true;
            } else if (g.cls == CL_DIAG2 && (va >= 0 || vb >= 0)) {
                // M index = 2 bit(w0) + bit(w1)
                if (va >= 0) {
                    const cd D[4] = {g.M[5 * (2 * va)], cd(0.0), cd(0.0), g.M[5 * (2 * va + 1)]};
                    apply(i, fb, D);
                } else {
                    const cd D[4] = {g.M[5 * vb], cd(0.0), cd(0.0), g.M[5 * (2 + vb)]};
                    apply(i, fa, D);
                }
                take = true;
            } else if (g.cls == CL_CTRL1 && va >= 0) {  // [control, target]
                if (va == 1) apply(i, fb, g.sub);
                take = true;
            }
        }
        if (take) {
            st->pf_in[i] = 1;
            any = true;
        } else {
            for (int j = 0; j < g.nw; j++) touched[g.w[j]] = 1;
        }
    }
    // per batch element: its ops (1-qubit gates with the element's values; the 2-qubit
    // rules only ever read parameter-independent, hence common, factors) and factors
    st->pf_slot_of = slot_of;
    st->pf_ops.assign(st->batch, ops0);
    st->pf_s.assign(st->batch, std::vector<cd>(2 * n, cd(0.0)));
    for (int b = 0; b < st->batch; b++) {
        std::vector<cd> fv(2 * n, cd(0.0));
        for (int f = 0; f < n; f++) fv[2 * f] = cd(1.0);
        for (PfOp &o : st->pf_ops[b]) {
            const GateRec &gr = gate_of(st, o.gate, b);
            if (gr.nw == 1)
                for (int j = 0; j < 4; j++) o.M[j] = gr.M[j];
            const cd a = fv[2 * o.slot], c1 = fv[2 * o.slot + 1];
            fv[2 * o.slot] = o.M[0] * a + o.M[1] * c1;
            fv[2 * o.slot + 1] = o.M[2] * a + o.M[3] * c1;
        }
        for (int q = 0; q < n; q++) {
            st->pf_s[b][2 * q] = fv[2 * slot_of[q]];
            st->pf_s[b][2 * q + 1] = fv[2 * slot_of[q] + 1];
        }
    }
    (void)sv;
    st->pf_on = any;
    return any;
}

// the global (sharded) qubits' factor of rank r: prod over the rank bits of s_q(bit)
// (physical position n_loc + i = qubit n-1-n_loc-i at the start), skipping qubit `skip`
static cd prefix_rank_factor(const tqd_state *st, const std::vector<cd> &S, int r, int skip) {
    cd v(1.0);
    for (int i = 0; i < st->g; i++) {
        const int q = st->n - 1 - (st->n_loc + i);
        if (q == skip) continue;
        v *= S[2 * q + ((r >> i) & 1)];
    }
    return v;
}

// the group tables tab_g[i] = prod over the group's physical bits of s_q(bit), q the
// qubit at that bit (pi = identity at the start: physical bit p = qubit n-1-p)
static int prefix_init(tqd_state *st) {
    const int nl = st->n_loc, n = st->n, B = st->batch;
    const int ng = (nl + PF_BITS_H - 1) / PF_BITS_H;
    st->pf_ng = ng;
    const size_t tab_elems = (size_t)ng << PF_BITS_H;
    // device: [B element tables (state dtype)][B M environments (fp64)]
    const size_t tab_bytes = tab_elems * st->esz, m_bytes = tab_elems * 2 * sizeof(double);
    const size_t need = (size_t)B * (tab_bytes + m_bytes);
    if (need > st->pf_cap) {
        if (st->pf_dev) { CUDA_TRY(st, cudaStreamSynchronize(st->ctx->stream)); cudaFree(st->pf_dev); }
        st->pf_dev = nullptr;
        st->pf_cap = 0;
        if (cudaMalloc(&st->pf_dev, need) != cudaSuccess) {
            cudaGetLastError();
            return fail(TQD_ERR_OOM, "cannot allocate the product-prefix tables");
        }
        st->pf_cap = need;
    }
    tqd_ctx *c = st->ctx;
    std::vector<double> h((size_t)B * tab_elems * 2, 0.0);
    for (int b = 0; b < B; b++) {
        const std::vector<cd> &S = st->pf_s[b];
        double *hb = h.data() + (size_t)b * tab_elems * 2;
        for (int g = 0; g < ng; g++) {
            // tab[i] = prod_j s_{q_j}(bit j of i), built bit by bit (tab[i | 2^j] = tab[i] s(1) / ... )
            const int bits = std::min(PF_BITS_H, nl - PF_BITS_H * g);
            std::vector<cd> t(1, cd(1.0));
            for (int j = 0; j < bits; j++) {
                const int q = n - 1 - (PF_BITS_H * g + j);
                const size_t half = t.size();
                t.resize(2 * half);
                for (size_t i = 0; i < half; i++) {
                    t[half + i] = t[i] * S[2 * q + 1];
                    t[i] = t[i] * S[2 * q];
                }
            }
            for (size_t i = 0; i < t.size(); i++) {
                hb[2 * (((size_t)g << PF_BITS_H) + i)] = t[i].real();
                hb[2 * (((size_t)g << PF_BITS_H) + i) + 1] = t[i].imag();
            }
        }
    }
    std::vector<float> hf;
    const void *src = h.data();
    if (!st->dbl) {
        hf.assign(h.begin(), h.end());
        src = hf.data();
    }
    CUDA_TRY(st, cudaMemcpyAsync(st->pf_dev, src, (size_t)B * tab_bytes, cudaMemcpyHostToDevice, c->stream));
    st->met.h2d_bytes += (size_t)B * tab_bytes;
    const int ev = ev_begin(st, CAT_OTHER);
    for (int b = 0; b < B; b++) {
        const cd cr = prefix_rank_factor(st, st->pf_s[b], c->rank, -1);
        CUDA_TRY(st, launch_prefix_init(st->dbl, (char *)st->psi + (size_t)b * shard_bytes(st), 1ull << nl, ng,
                                        (const char *)st->pf_dev + (size_t)b * tab_bytes, cr.real(), cr.imag(),
                                        c->stream));
        st->met.kernel_launches++;
    }
    ev_end(st, ev);
    CUDA_TRY(st, cudaStreamSynchronize(c->stream));  // host tables go out of scope
    st->met.hbm_bytes += (uint64_t)B * shard_bytes(st);
    for (char in : st->pf_in) {
        st->met.gates_applied += in ? (uint64_t)B : 0;
        st->met.gates_prefix += in ? (uint64_t)B : 0;
    }
    return TQD_OK;
}

// gradients of the prefix gates from lambda at the prefix boundary (st->lam)
static int allreduce_sum(tqd_state *st, double *d, size_t count);

static int prefix_grads(tqd_state *st, std::vector<double> &grad) {
    tqd_ctx *c = st->ctx;
    const int nl = st->n_loc, n = st->n, ng = st->pf_ng, B = st->batch;
    const size_t tab_elems = (size_t)ng << PF_BITS_H;
    const size_t tab_bytes = tab_elems * st->esz;
    // every element's environments M_g in one pass each, one readback
    double *dM = (double *)((char *)st->pf_dev + (size_t)B * tab_bytes);
    CUDA_TRY(st, cudaMemsetAsync(dM, 0, (size_t)B * tab_elems * 2 * sizeof(double), c->stream));
    {
        const int ev = ev_begin(st, CAT_OTHER);
        for (int be = 0; be < B; be++) {
            CUDA_TRY(st, launch_prefix_contract(st->dbl, (const char *)st->lam + (size_t)be * shard_bytes(st),
                                                1ull << nl, ng, (const char *)st->pf_dev + (size_t)be * tab_bytes,
                                                dM + (size_t)be * tab_elems * 2, c->sms, c->stream));
            st->met.kernel_launches++;
        }
        ev_end(st, ev);
    }
    std::vector<double> Mall((size_t)B * tab_elems * 2);
    CUDA_TRY(st, cudaMemcpyAsync(Mall.data(), dM, Mall.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(st, cudaStreamSynchronize(c->stream));
    st->met.hbm_bytes += (uint64_t)B * shard_bytes(st);
    st->met.d2h_bytes += Mall.size() * sizeof(double);
    std::vector<int> q_of_slot(n);
    for (int q = 0; q < n; q++) q_of_slot[st->pf_slot_of[q]] = q;
    for (int be = 0; be < B; be++) {
        const std::vector<cd> &S = st->pf_s[be];
        const std::vector<PfOp> &ops = st->pf_ops[be];
        std::vector<double> M(Mall.begin() + (size_t)be * tab_elems * 2, Mall.begin() + (size_t)(be + 1) * tab_elems * 2);
        // world > 1: this rank's total contraction Z_r (M_0 . tab_0), then M scaled by the
        // rank factor c_r and summed over the ranks together with every rank's Z_r
        std::vector<cd> Zr(c->world, cd(0.0));
        if (c->world > 1) {
            std::vector<cd> t0(1 << PF_BITS_H, cd(0.0));
            {
                const int bits = std::min(PF_BITS_H, nl);
                for (int i = 0; i < (1 << bits); i++) {
                    cd v(1.0);
                    for (int j = 0; j < bits; j++) v *= S[2 * (n - 1 - j) + ((i >> j) & 1)];
                    t0[i] = v;
                }
            }
            cd z(0.0);
            for (int i = 0; i < (1 << PF_BITS_H); i++) z += cd(M[2 * i], M[2 * i + 1]) * t0[i];
            const cd cr = prefix_rank_factor(st, S, c->rank, -1);
            for (size_t i = 0; i < tab_elems; i++) {
                const cd v = cd(M[2 * i], M[2 * i + 1]) * cr;
                M[2 * i] = v.real();
                M[2 * i + 1] = v.imag();
            }
            std::vector<double> buf(M);
            buf.resize(M.size() + 2 * c->world, 0.0);
            buf[M.size() + 2 * c->rank] = z.real();
            buf[M.size() + 2 * c->rank + 1] = z.imag();
            const size_t bytes = buf.size() * sizeof(double);
            int rc = ensure_red(st, buf.size());  // (the gradients are already on the host)
            if (rc) return rc;
            double *dr = st->d_red;
            CUDA_TRY(st, cudaMemcpyAsync(dr, buf.data(), bytes, cudaMemcpyHostToDevice, c->stream));
            rc = allreduce_sum(st, dr, buf.size());
            if (rc) return rc;
            CUDA_TRY(st, cudaMemcpyAsync(buf.data(), dr, bytes, cudaMemcpyDeviceToHost, c->stream));
            CUDA_TRY(st, cudaStreamSynchronize(c->stream));
            for (size_t i = 0; i < M.size(); i++) M[i] = buf[i];
            for (int r = 0; r < c->world; r++) Zr[r] = cd(buf[M.size() + 2 * r], buf[M.size() + 2 * r + 1]);
        }
        // T_q(v) = sum_{i: bit j of i = v} M_g[i] prod_{j' != j in group g} s_{q'}(bit j'):
        // contract M_g with every factor of the group but j (top bits by halving, then
        // the bits below j by pairing), O(bits 2^bits) per group
        std::vector<cd> T(2 * n, cd(0.0));
        for (int g = 0; g < ng; g++) {
            const int bits = std::min(PF_BITS_H, nl - PF_BITS_H * g);
            auto sf = [&](int jj, int v) { return S[2 * (n - 1 - (PF_BITS_H * g + jj)) + v]; };
            for (int j = 0; j < bits; j++) {
                std::vector<cd> W(1u << bits);
                for (size_t i = 0; i < W.size(); i++)
                    W[i] = cd(M[2 * (((size_t)g << PF_BITS_H) + i)], M[2 * (((size_t)g << PF_BITS_H) + i) + 1]);
                for (int jj = bits - 1; jj > j; jj--) {  // top bit jj: W'[i] = W[i] s(0) + W[i + half] s(1)
                    const size_t half = W.size() / 2;
                    for (size_t i = 0; i < half; i++) W[i] = W[i] * sf(jj, 0) + W[i + half] * sf(jj, 1);
                    W.resize(half);
                }
                for (int jj = 0; jj < j; jj++) {  // lowest remaining bit: W'[i] = W[2i] s(0) + W[2i+1] s(1)
                    const size_t half = W.size() / 2;
                    for (size_t i = 0; i < half; i++) W[i] = W[2 * i] * sf(jj, 0) + W[2 * i + 1] * sf(jj, 1);
                    W.resize(half);
                }
                const int q = n - 1 - (PF_BITS_H * g + j);
                T[2 * q] += W[0];
                T[2 * q + 1] += W[1];
            }
        }
        // sharded qubits: T_q(v) = sum over the ranks whose bit of q is v of Z_r times the
        // other sharded qubits' factors
        for (int i = 0; i < st->g && c->world > 1; i++) {
            const int q = n - 1 - (nl + i);
            for (int r = 0; r < c->world; r++) T[2 * q + ((r >> i) & 1)] += Zr[r] * prefix_rank_factor(st, S, r, q);
        }
        // d s_f / d theta for every generator of every prefix gate: replay the gate's
        // slot chain from |0> with dU = G U inserted at that gate; T of the qubit holding
        // the slot at the boundary; the element's own gradient slots (batched gates)
        for (size_t oi = 0; oi < ops.size(); oi++) {
            const PfOp &oi_ = ops[oi];
            const GateRec &gi = gate_of(st, oi_.gate, be);
            if (!gi.ngen) continue;
            const int f = oi_.slot, q = q_of_slot[f];
            for (int p = 0; p < gi.ngen; p++) {
                cd a(1.0), bb(0.0);
                for (size_t k = 0; k < ops.size(); k++) {
                    const PfOp &o = ops[k];
                    if (o.slot != f) continue;
                    cd na = o.M[0] * a + o.M[1] * bb, nb = o.M[2] * a + o.M[3] * bb;
                    if (k == oi) {
                        const cd ga = gi.G[p][0] * na + gi.G[p][1] * nb, gb2 = gi.G[p][2] * na + gi.G[p][3] * nb;
                        na = ga;
                        nb = gb2;
                    }
                    a = na;
                    bb = nb;
                }
                grad[gi.slot0 + p] += 2.0 * (T[2 * q] * a + T[2 * q + 1] * bb).real();
            }
        }
    }
    return TQD_OK;
}

// Execute the recorded gates [executed, end).  end < gates.size() only from
// tqd_adjoint_grad: the gates [end, size) were absorbed into the observable
// (absorb_tail) and are never applied; the plan caches are keyed by that split.
// keep_tail (tqd_expval): the absorbed gates stay pending (executed = end), so a
// later readback or non-Z observable applies them; else they count as executed.
static int execute_pending(tqd_state *st, size_t end = SIZE_MAX, bool keep_tail = false) {
    if (end > st->gates.size()) end = st->gates.size();
    const size_t done_to = keep_tail ? end : st->gates.size();
    if (st->executed >= end) {
        if (!keep_tail) st->executed = st->gates.size();
        return TQD_OK;
    }
    uint64_t tmix = (uint64_t)(st->gates.size() - end) * 0x9E3779B97F4A7C15ull;
    if (prefix_build(st, end) && st->opt_prefix == 2) {
        // auto: keep the prefix only if the plan without its gates is cheaper by more
        // than the extra read pass of the environments (~0.17 of a sweep pair); the
        // decision is cached per circuit structure
        const uint64_t dsig = plan_signature(st->gates, plan_cfg(st)) ^ tmix;
        if (st->pf_dec_sig != dsig) {
            std::vector<int> pa, pb;
            for (size_t i = 0; i < end; i++) {
                pb.push_back((int)i);
                if (!st->pf_in[i]) pa.push_back((int)i);
            }
            std::vector<int> posa = st->pos, posb = st->pos;
            std::vector<Stage> sa, sb;
            std::string e2;
            const bool ok = plan_circuit(st->gates, pa, posa, plan_cfg(st), sa, e2) == TQD_OK &&
                            plan_circuit(st->gates, pb, posb, plan_cfg(st), sb, e2) == TQD_OK;
            st->pf_dec = ok && plan_cost(sa) + 0.17 < plan_cost(sb);
            st->pf_dec_sig = dsig;
        }
        if (!st->pf_dec) st->pf_on = false;
    }
    if (st->pf_on) {
        // the prefix replaces |0..0> + its gates' sweeps; it is part of the plan's structure
        for (size_t i = 0; i < st->pf_in.size(); i++)
            if (st->pf_in[i]) tmix = (tmix ^ (i + 1)) * 1099511628211ull;
        int rc = prefix_init(st);
        if (rc) return rc;
    }
    if (st->executed == 0 && st->fwd_cache_version != st->tape_version && st->enc_fwd->valid &&
        !st->cached_stages.empty() && st->cached_tmix == tmix) {
        const uint64_t vh = tape_values_hash(st);
        if (vh == st->fwd_vhash) {
            st->fwd_cache_version = st->tape_version;
            if (vh == st->bwd_vhash) st->bwd_cache_version = st->tape_version;
            st->met.plans_reused++;
        }
    }
    if (st->executed == 0 && st->fwd_cache_version == st->tape_version && st->enc_fwd->valid &&
        st->cached_tmix == tmix) {
        // replay of the same tape from |0..0> (tqd_state_rewind): plan + descriptors are resident
        st->history = st->cached_stages;
        int rc = launch_graphed(st, st->history, false, *st->enc_fwd, nullptr, st->g_fwd, st->g_fwd_key, st->g_fwd_delta);
        if (rc) return rc;
        st->pos = st->cached_pos;
        st->executed = done_to;
        st->history_cached = true;
        return TQD_OK;
    }
    std::vector<int> pending;
    for (size_t i = st->executed; i < end; i++)
        if (!st->pf_on || !st->pf_in[i]) pending.push_back((int)i);
    std::vector<Stage> stages;
    std::string err;
    const bool from_zero = st->executed == 0;
    const uint64_t sig = from_zero ? plan_signature(st->gates, plan_cfg(st)) ^ tmix : 0;
    if (from_zero && !st->cached_stages.empty() && sig == st->plan_sig) {
        // same circuit structure, new parameter values: reuse the plan
        stages = st->cached_stages;
        refresh_plan_values(stages, st->gates);
        st->pos = st->cached_pos;
        st->met.plans_reused++;
    } else {
        int rc = plan_circuit(st->gates, pending, st->pos, plan_cfg(st), stages, err);
        if (rc) return fail(rc, err);
    }
    int rc;
    Encoded &E = from_zero ? *st->enc_fwd : *st->enc_tmp;
    rc = encode_upload(st, stages, false, E);
    if (rc) return rc;
    rc = launch_encoded(st, stages, false, E, nullptr);
    if (rc) return rc;
    if (from_zero) {
        st->cached_stages = stages;
        st->cached_pos = st->pos;
        st->plan_sig = sig;
        st->cached_tmix = tmix;
        st->fwd_cache_version = st->tape_version;
        st->fwd_vhash = tape_values_hash(st);
        st->bwd_cache_version = ~0ull;
        st->bwd_vhash = 0;
        st->history_cached = true;
    } else {
        st->history_cached = false;
    }
    for (auto &s : stages) st->history.push_back(std::move(s));
    st->executed = done_to;
    return TQD_OK;
}

static int allreduce_sum(tqd_state *st, double *d, size_t count) {
    if (st->ctx->world == 1 || count == 0) return TQD_OK;
    COMM_TRY(st, st->ctx->comm->allreduce_sum(d, count, CE_F64, st->ctx->stream));
    return TQD_OK;
}

static uint64_t phys_mask(const tqd_state *st, uint64_t logical_mask) {
    uint64_t m = 0;
    for (int q = 0; q < st->n; q++)
        if ((logical_mask >> q) & 1) m |= 1ull << st->pos[q];
    return m;
}

static int check_terms(const tqd_state *st, int T, const uint64_t *x, const uint64_t *z) {
    if (T < 0) return fail(TQD_ERR_ARG, "n_terms < 0");
    if (T > 0 && (!x || !z)) return fail(TQD_ERR_ARG, "x_mask / z_mask is NULL");
    const uint64_t lim = st->n >= 64 ? ~0ull : ((1ull << st->n) - 1);
    for (int t = 0; t < T; t++)
        if ((x[t] & ~lim) || (z[t] & ~lim)) return fail(TQD_ERR_ARG, "Pauli mask names a qubit >= n");
    return TQD_OK;
}

// ============================================================================
extern "C" {

const char *tqd_last_error(void) { return g_err.c_str(); }

const char *tqd_version(void) {
    static std::string v;
    if (v.empty()) {
        char b[160];
        snprintf(b, sizeof(b), "tqd-b200 sm_100a CUDA %d NCCL %d.%d.%d", CUDART_VERSION, NCCL_MAJOR, NCCL_MINOR, NCCL_PATCH);
        v = b;
    }
    return v.c_str();
}

int tqd_nccl_unique_id(void *out128) {
    if (!out128) return fail(TQD_ERR_ARG, "out128 is NULL");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return fail(TQD_ERR_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    static_assert(sizeof(id) == 128, "NCCL unique id is 128 bytes");
    memcpy(out128, &id, 128);
    return TQD_OK;
}

int tqd_loopback_id(void *out128) {
    if (!out128) return fail(TQD_ERR_ARG, "out128 is NULL");
    comm_make_loopback_id(out128);
    return TQD_OK;
}

int tqd_ctx_create(int world, int rank, int cuda_device, const void *nccl_id, void *cuda_stream, tqd_ctx **out) {
    if (!out) return fail(TQD_ERR_ARG, "out is NULL");
    *out = nullptr;
    if (world < 1 || (world & (world - 1)) != 0) return fail(TQD_ERR_WORLD, "world size must be a power of two");
    if (rank < 0 || rank >= world) return fail(TQD_ERR_WORLD, "rank out of range");
    if (world > 1 && !nccl_id) return fail(TQD_ERR_ARG, "nccl_id is NULL for world > 1");
    cudaError_t e = cudaSetDevice(cuda_device);
    if (e != cudaSuccess) return fail(TQD_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    tqd_ctx *c = new tqd_ctx();
    c->world = world;
    c->rank = rank;
    c->device = cuda_device;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, cuda_device) == cudaSuccess) c->sms = prop.multiProcessorCount;
    if (cuda_stream) {
        c->stream = (cudaStream_t)cuda_stream;
    } else {
        e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) { delete c; return fail(TQD_ERR_CUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e)); }
        c->own_stream = true;
    }
    if (world > 1) {
        std::string err;
        c->comm = comm_create(nccl_id, world, rank, err);
        if (!c->comm) {
            if (c->own_stream) cudaStreamDestroy(c->stream);
            delete c;
            return fail(TQD_ERR_NCCL, err);
        }
    }
    *out = c;
    return TQD_OK;
}

int tqd_ctx_destroy(tqd_ctx *c) {
    if (!c) return fail(TQD_ERR_ARG, "ctx is NULL");
    delete c->comm;
    if (c->own_stream) cudaStreamDestroy(c->stream);
    delete c;
    return TQD_OK;
}

int tqd_state_bytes(int n, tqd_dtype dt, int world, int with_adjoint, size_t *out) {
    if (!out) return fail(TQD_ERR_ARG, "out is NULL");
    if (world < 1 || (world & (world - 1))) return fail(TQD_ERR_WORLD, "world size must be a power of two");
    int g = 0;
    while ((1 << g) < world) g++;
    if (n < (g ? g + 2 : 1) || n > 62) return fail(TQD_ERR_QUBITS, "need g + 2 <= n <= 62");
    const size_t esz = dt == TQD_C128 ? 16 : 8;
    const size_t shard = ((size_t)1 << (n - g)) * esz;
    *out = shard * (with_adjoint ? 2 : 1) + (world > 1 ? staging_bytes_for(shard, esz, 0) : 0);
    return TQD_OK;
}

static int state_init(tqd_ctx *c, int n, tqd_dtype dt, int batch, void *dev_buf, size_t buf_bytes, tqd_state **out);

int tqd_state_init(tqd_ctx *c, int n, tqd_dtype dt, void *dev_buf, size_t buf_bytes, tqd_state **out) {
    return state_init(c, n, dt, 1, dev_buf, buf_bytes, out);
}

int tqd_state_init_batch(tqd_ctx *c, int n, tqd_dtype dt, int batch, tqd_state **out) {
    if (batch < 1 || batch > (1 << 20)) return fail(TQD_ERR_ARG, "batch must be in [1, 2^20]");
    return state_init(c, n, dt, batch, nullptr, 0, out);
}

static int state_init(tqd_ctx *c, int n, tqd_dtype dt, int batch, void *dev_buf, size_t buf_bytes, tqd_state **out) {
    if (!c || !out) return fail(TQD_ERR_ARG, "ctx/out is NULL");
    *out = nullptr;
    if (c->poisoned) return fail(TQD_ERR_STATE, "context poisoned");
    if (dt != TQD_C64 && dt != TQD_C128) return fail(TQD_ERR_ARG, "bad dtype");
    int g = 0;
    while ((1 << g) < c->world) g++;
    if (n < (g ? g + 2 : 1) || n > 62)
        return fail(TQD_ERR_QUBITS, "n must satisfy log2(world) + 2 <= n <= 62 (PAPER.md:162: at least two unsharded qubits)");
    tqd_state *st = new tqd_state();
    st->ctx = c;
    st->n = n;
    st->g = g;
    st->n_loc = n - g;
    st->dbl = dt == TQD_C128;
    st->esz = st->dbl ? 16 : 8;
    st->batch = batch;
    memset(&st->met, 0, sizeof(st->met));
    st->enc_fwd = new Encoded();
    st->enc_bwd = new Encoded();
    st->enc_tmp = new Encoded();
    const size_t sb = shard_bytes(st);
    if (dev_buf) {
        if (buf_bytes < sb) { delete st; return fail(TQD_ERR_OOM, "dev_buf smaller than one shard"); }
        // carve: psi, then lambda (when two shards fit), then the staging (world > 1)
        st->psi = dev_buf;
        size_t used = sb;
        if (buf_bytes >= 2 * sb) { st->lam = (char *)dev_buf + sb; used = 2 * sb; }
        const size_t sg = staging_bytes_for(sb, st->esz, 0);
        if (c->world > 1 && buf_bytes >= used + sg) { st->stg = (char *)dev_buf + used; st->stg_bytes = sg; }
        st->met.peak_device_bytes = buf_bytes;
    } else {
        if (cudaMalloc(&st->psi, sb * batch) != cudaSuccess) {
            cudaGetLastError();
            delete st;
            return fail(TQD_ERR_OOM, "cannot allocate the state shard");
        }
        st->own_psi = true;
        st->psi_first = st->psi;
        st->met.peak_device_bytes = sb * batch;
    }
    int rc = tqd_state_reset(st);
    if (rc) { tqd_state_free(st); return rc; }
    *out = st;
    return TQD_OK;
}

int tqd_state_reset(tqd_state *st) {
    int rc = check_live(st);
    if (rc) return rc;
    st->pf_on = false;
    st->gates.clear();
    st->brec.clear();
    st->history.clear();
    st->tape_version++;
    st->history_cached = false;
    st->n_params = 0;
    st->executed = 0;
    st->consumed = false;
    st->pos.assign(st->n, 0);
    for (int q = 0; q < st->n; q++) st->pos[q] = st->n - 1 - q;  // MSB-first identity (R1)
    const int ev = ev_begin(st, CAT_OTHER);
    CUDA_TRY(st, cudaMemsetAsync(st->psi, 0, all_bytes(st), st->ctx->stream));
    if (st->ctx->rank == 0)
        for (int b = 0; b < st->batch; b++)
            CUDA_TRY(st, launch_set_one(st->dbl, (char *)st->psi + (size_t)b * shard_bytes(st), st->ctx->stream));
    ev_end(st, ev);
    st->met.hbm_bytes += all_bytes(st);
    st->met.kernel_launches += 1;
    return ev_collect(st);
}

int tqd_state_rewind(tqd_state *st) {
    int rc = check_live(st);
    if (rc) return rc;
    st->pf_on = false;
    st->history.clear();
    st->history_cached = false;
    st->executed = 0;
    st->consumed = false;
    st->pos.assign(st->n, 0);
    for (int q = 0; q < st->n; q++) st->pos[q] = st->n - 1 - q;
    const int ev = ev_begin(st, CAT_OTHER);
    CUDA_TRY(st, cudaMemsetAsync(st->psi, 0, all_bytes(st), st->ctx->stream));
    if (st->ctx->rank == 0)
        for (int b = 0; b < st->batch; b++)
            CUDA_TRY(st, launch_set_one(st->dbl, (char *)st->psi + (size_t)b * shard_bytes(st), st->ctx->stream));
    ev_end(st, ev);
    st->met.hbm_bytes += all_bytes(st);
    st->met.kernel_launches += 1;
    return TQD_OK;
}

int tqd_state_free(tqd_state *st) {
    if (!st) return fail(TQD_ERR_ARG, "state is NULL");
    if (st->ctx && st->ctx->stream) cudaStreamSynchronize(st->ctx->stream);
    if (st->ctx && st->ctx->comm) {
        st->ctx->comm->release_buffers(st->peer_pl, 2);
    }
    if (st->own_psi) cudaFree(st->psi);
    if (st->own_lam) cudaFree(st->lam);
    if (st->own_stg) cudaFree(st->stg);
    for (Encoded *E : {st->enc_fwd, st->enc_bwd, st->enc_tmp}) {
        if (E) { free_encoded(*E); delete E; }
    }
    if (st->g_fwd) cudaGraphExecDestroy(st->g_fwd);
    if (st->g_bwd) cudaGraphExecDestroy(st->g_bwd);
    if (st->d_red) cudaFree(st->d_red);
    if (st->d_xy) cudaFree(st->d_xy);
    if (st->circ_dev) cudaFree(st->circ_dev);
    if (st->pf_dev) cudaFree(st->pf_dev);
    for (auto e : st->ev_pool) cudaEventDestroy(e);
    delete st;
    return TQD_OK;
}

int tqd_state_set_option(tqd_state *st, int option, int64_t v) {
    if (!st) return fail(TQD_ERR_ARG, "state is NULL");
    switch (option) {
    case TQD_OPT_TILE_QUBITS: {
        // the sweep kernels are built for <= 256 threads per CTA (launch bounds):
        // 2^k = 32 lanes x 2^R registers x <= 8 warps
        const int kmax = LANE_BITS + TQD_SWEEP_R + 3;
        if (v < 9 || v > kmax) return fail(TQD_ERR_ARG, "tile qubits must be in [9, " + std::to_string(kmax) + "]");
        st->opt_k = (int)v; return TQD_OK;
    }
    case TQD_OPT_SMALL_MAX:
        if (v < 0 || v > 12) return fail(TQD_ERR_ARG, "small_max must be in [0, 12]");
        if (st->dbl && v > 11) return fail(TQD_ERR_ARG, "small_max must be <= 11 for complex128");
        st->opt_small = (int)v; return TQD_OK;
    case TQD_OPT_PROFILE: st->opt_profile = v ? 1 : 0; return TQD_OK;
    case TQD_OPT_GRID_CTAS:
        if (v < 0) return fail(TQD_ERR_ARG, "grid must be >= 0");
        st->opt_grid = (int)v; return TQD_OK;
    case TQD_OPT_USE_GRAPH: st->opt_graph = v ? 1 : 0; return TQD_OK;
    case TQD_OPT_FUSED_REMAP: st->opt_fused = v ? 1 : 0; return TQD_OK;
    case TQD_OPT_ABSORB_TAIL: st->opt_absorb = v ? 1 : 0; return TQD_OK;
    case TQD_OPT_PRODUCT_PREFIX:
        if (v < 0 || v > 2) return fail(TQD_ERR_ARG, "TQD_OPT_PRODUCT_PREFIX: 0, 1 or 2");
        st->opt_prefix = (int)v;
        return TQD_OK;
    case TQD_OPT_CIRCUIT_LAYOUT:
        if (st->opt_layout != (v ? 1 : 0)) st->circ_key = 0;  // re-encode the cached circuit
        st->opt_layout = v ? 1 : 0;
        return TQD_OK;
    case TQD_OPT_CIRCUIT_MAX:
        if (v < 0 || v > 12) return fail(TQD_ERR_ARG, "circuit_max must be in [0, 12]");
        st->opt_circuit = (int)v; return TQD_OK;
    case TQD_OPT_STAGING_BYTES:
        if (v < 0) return fail(TQD_ERR_ARG, "staging bytes must be >= 0");
        st->opt_stage = (size_t)v; return TQD_OK;
    default: return fail(TQD_ERR_ARG, "unknown option");
    }
}

int tqd_apply_gate(tqd_state *st, tqd_gate g, const int *wires, int n_wires, const double *params,
                   const double *matrix, int trainable) {
    if (!st) return fail(TQD_ERR_ARG, "state is NULL");
    if (st->consumed) return fail(TQD_ERR_STATE, "state consumed by tqd_adjoint_grad; call tqd_state_reset");
    if (!wires) return fail(TQD_ERR_ARG, "wires is NULL");
    if (n_wires < 1 || n_wires > 2) return fail(TQD_ERR_ARG, "n_wires must be 1 or 2");
    for (int i = 0; i < n_wires; i++)
        if (wires[i] < 0 || wires[i] >= st->n) return fail(TQD_ERR_ARG, "wire out of range");
    if (n_wires == 2 && wires[0] == wires[1]) return fail(TQD_ERR_ARG, "duplicate wires");
    GateRec rec;
    std::string err;
    int rc = make_gate((int)g, wires, n_wires, params, matrix, trainable, st->dbl, rec, err);
    if (rc) return fail(rc, err);
    if (rec.trainable) {
        rec.slot0 = st->n_params;
        st->n_params += gate_num_params((int)g);
    }
    st->gates.push_back(rec);
    st->tape_version++;
    return TQD_OK;
}

int tqd_apply_circuit(tqd_state *st, int G, const int *kinds, const int *wires, const double *params,
                      const double *mats, const int *trainable) {
    if (!st) return fail(TQD_ERR_ARG, "state is NULL");
    if (st->consumed) return fail(TQD_ERR_STATE, "state consumed by tqd_adjoint_grad; call tqd_state_reset");
    if (G < 0) return fail(TQD_ERR_ARG, "G < 0");
    if (G == 0) return TQD_OK;
    if (!kinds || !wires || !params || !mats || !trainable) return fail(TQD_ERR_ARG, "NULL argument");
    std::vector<GateRec> recs;
    recs.reserve(G);
    int np_ = st->n_params;
    for (int i = 0; i < G; i++) {
        const int nw = gate_arity(kinds[i]);
        if (nw < 1 || nw > 2) return fail(TQD_ERR_ARG, "unknown gate kind");
        for (int j = 0; j < nw; j++)
            if (wires[2 * i + j] < 0 || wires[2 * i + j] >= st->n) return fail(TQD_ERR_ARG, "wire out of range");
        if (nw == 2 && wires[2 * i] == wires[2 * i + 1]) return fail(TQD_ERR_ARG, "duplicate wires");
        GateRec rec;
        std::string err;
        int rc = make_gate(kinds[i], wires + 2 * i, nw, params + 3 * i, mats + 32 * i, trainable[i], st->dbl, rec, err);
        if (rc) return fail(rc, err);
        if (rec.trainable) { rec.slot0 = np_; np_ += gate_num_params(kinds[i]); }
        recs.push_back(rec);
    }
    st->gates.insert(st->gates.end(), recs.begin(), recs.end());
    st->n_params = np_;
    st->tape_version++;
    return TQD_OK;
}

int tqd_apply_gate_batch(tqd_state *st, tqd_gate g, const int *wires, int n_wires, const double *params, int trainable) {
    if (!st) return fail(TQD_ERR_ARG, "state is NULL");
    if (st->consumed) return fail(TQD_ERR_STATE, "state consumed by tqd_adjoint_grad; call tqd_state_reset");
    if (g != TQD_RX && g != TQD_RY && g != TQD_RZ && g != TQD_U3)
        return fail(TQD_ERR_ARG, "batched parameters: RX, RY, RZ or U3 only");
    if (!wires || n_wires != 1) return fail(TQD_ERR_ARG, "batched gates act on one wire");
    if (wires[0] < 0 || wires[0] >= st->n) return fail(TQD_ERR_ARG, "wire out of range");
    if (!params) return fail(TQD_ERR_ARG, "params is NULL");
    const int np_ = gate_num_params((int)g);
    std::vector<GateRec> recs(st->batch);
    std::string err;
    for (int b = 0; b < st->batch; b++) {
        int rc = make_gate((int)g, wires, 1, params + (size_t)b * np_, nullptr, trainable, st->dbl, recs[b], err);
        if (rc) return fail(rc, err);
        recs[b].batched = 1;
        recs[b].cls = g == TQD_RZ ? CL_DIAG1 : CL_U1;  // by kind: the same kernel ops for every element
        if (recs[b].trainable) recs[b].slot0 = st->n_params + b * np_;
    }
    if (recs[0].trainable) st->n_params += st->batch * np_;
    st->gates.push_back(recs[0]);
    st->brec.resize(st->gates.size());
    st->brec.back() = std::move(recs);
    st->tape_version++;
    return TQD_OK;
}

int tqd_state_info(const tqd_state *st, int *n_qubits, int *batch, int *dtype) {
    if (!st) return fail(TQD_ERR_ARG, "state is NULL");
    if (n_qubits) *n_qubits = st->n;
    if (batch) *batch = st->batch;
    if (dtype) *dtype = st->dbl ? TQD_C128 : TQD_C64;
    return TQD_OK;
}

int tqd_num_params(const tqd_state *st, int *out) {
    if (!st || !out) return fail(TQD_ERR_ARG, "NULL argument");
    *out = st->n_params;
    return TQD_OK;
}

static size_t absorb_tail(const std::vector<GateRec> &gates, size_t executed, std::vector<uint64_t> &z,
                          std::vector<double> &sgn);

int tqd_expval(tqd_state *st, int T, const uint64_t *x, const uint64_t *z, const double *coeff, double *out) {
    int rc = check_live(st);
    if (rc) return rc;
    if (st->consumed) return fail(TQD_ERR_STATE, "state consumed by tqd_adjoint_grad; call tqd_state_reset");
    if (T > 0 && !out) return fail(TQD_ERR_ARG, "out is NULL");
    rc = check_terms(st, T, x, z);
    if (rc) return rc;
    // Z-only observables: the trailing diagonal / permutation gates are folded into
    // the terms (absorb_tail) and stay pending for later calls
    std::vector<uint64_t> zabs(z, z + T);
    std::vector<double> sabs(T, 1.0);
    size_t end = st->gates.size();
    bool z_only = T > 0;
    for (int t = 0; t < T; t++)
        if (x[t]) z_only = false;
    if (st->opt_absorb && z_only) {
        end = absorb_tail(st->gates, st->executed, zabs, sabs);
        z = zabs.data();
        if (end < st->gates.size()) st->met.gates_absorbed += st->gates.size() - end;
    }
    rc = execute_pending(st, end, true);
    if (rc) return rc;
    if (T == 0) return ev_collect(st);
    const int BT = st->batch * T;  // outputs: batch element b, term t at b * T + t
    rc = ensure_red(st, (size_t)BT + 2 * 64 + 64 + 16);
    if (rc) return rc;
    tqd_ctx *c = st->ctx;
    double *d_all = st->d_red;
    uint64_t *d_masks = (uint64_t *)(st->d_red + BT);
    int *d_ny = (int *)(st->d_red + BT + 64);
    const uint64_t N = 1ull << st->n_loc;
    CUDA_TRY(st, cudaMemsetAsync(d_all, 0, BT * sizeof(double), c->stream));
    const int ev = ev_begin(st, CAT_OTHER);
    // Z-only terms, 16 per launch; X/Y terms grouped by x mask
    std::vector<int> zt;
    for (int t = 0; t < T; t++) if (x[t] == 0) zt.push_back(t);
    for (int bi = 0; bi < st->batch; bi++) {
    void *psi_b = (char *)st->psi + (size_t)bi * shard_bytes(st);
    double *d_out = d_all + (size_t)bi * T;
    std::vector<char> done(T, 0);
    for (size_t b = 0; b < zt.size();) {
        // terms contiguous in the output? use a staging vector + scatter by index below
        const int cnt = (int)std::min<size_t>(16, zt.size() - b);
        uint64_t hm[16];
        for (int i = 0; i < cnt; i++) hm[i] = phys_mask(st, z[zt[b + i]]);
        CUDA_TRY(st, cudaMemcpyAsync(d_masks, hm, cnt * sizeof(uint64_t), cudaMemcpyHostToDevice, c->stream));
        // results go to d_out[T..] scratch? simpler: accumulate into d_out at the term positions via a temp
        double *tmp = st->d_red + BT + 128;
        CUDA_TRY(st, cudaMemsetAsync(tmp, 0, 16 * sizeof(double), c->stream));
        CUDA_TRY(st, launch_expval_z(st->dbl, psi_b, N, rank_hi(st), d_masks, cnt, tmp, c->stream));
        for (int i = 0; i < cnt; i++)
            CUDA_TRY(st, cudaMemcpyAsync(d_out + zt[b + i], tmp + i, sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
        CUDA_TRY(st, cudaStreamSynchronize(c->stream));  // hm lives on the host stack
        st->met.hbm_bytes += N * st->esz;
        st->met.kernel_launches++;
        for (int i = 0; i < cnt; i++) done[zt[b + i]] = 1;
        b += cnt;
    }
    for (int t0 = 0; t0 < T; t0++) {
        if (done[t0]) continue;
        std::vector<int> grp;
        for (int t = t0; t < T; t++)
            if (!done[t] && x[t] == x[t0] && grp.size() < 16) grp.push_back(t);
        const uint64_t xp = phys_mask(st, x[t0]);
        const uint64_t xl = xp & ((1ull << st->n_loc) - 1);
        const int gx = (int)(xp >> st->n_loc);
        uint64_t hm[16];
        int hn[16];
        for (size_t i = 0; i < grp.size(); i++) {
            hm[i] = phys_mask(st, z[grp[i]]);
            hn[i] = __builtin_popcountll(x[grp[i]] & z[grp[i]]) & 3;
        }
        CUDA_TRY(st, cudaMemcpyAsync(d_masks, hm, grp.size() * sizeof(uint64_t), cudaMemcpyHostToDevice, c->stream));
        CUDA_TRY(st, cudaMemcpyAsync(d_ny, hn, grp.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream));
        double *tmp = st->d_red + BT + 128;
        CUDA_TRY(st, cudaMemsetAsync(tmp, 0, 16 * sizeof(double), c->stream));
        if (gx) {
            // X / Y on rank bits: <psi|P|psi> pairs this shard with rank ^ gx's shard
            // (PAPER.md:164), exchanged chunk by chunk through the bounded staging
            rc = xy_partner_chunks(st, psi_b, gx, xl, [&](uint64_t off, const void *pc, uint64_t cnt, uint64_t lo) {
                CUDA_TRY(st, launch_expval_xy(st->dbl, (const char *)psi_b + off * st->esz, pc, cnt, rank_hi(st) | off, lo,
                                              d_masks, d_ny, (int)grp.size(), tmp, c->stream));
                return (int)TQD_OK;
            });
            if (rc) return rc;
        } else {
            CUDA_TRY(st, launch_expval_xy(st->dbl, psi_b, psi_b, N, rank_hi(st), xl, d_masks, d_ny, (int)grp.size(), tmp,
                                          c->stream));
        }
        for (size_t i = 0; i < grp.size(); i++)
            CUDA_TRY(st, cudaMemcpyAsync(d_out + grp[i], tmp + i, sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
        CUDA_TRY(st, cudaStreamSynchronize(c->stream));
        st->met.hbm_bytes += 2 * N * st->esz;
        st->met.kernel_launches++;
        for (int t : grp) done[t] = 1;
    }
    }  // batch elements
    ev_end(st, ev);
    rc = allreduce_sum(st, d_all, BT);
    if (rc) return rc;
    std::vector<double> h(BT);
    CUDA_TRY(st, cudaMemcpyAsync(h.data(), d_all, BT * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(st, cudaStreamSynchronize(c->stream));
    st->met.d2h_bytes += BT * sizeof(double);
    for (int i = 0; i < BT; i++) out[i] = (coeff ? coeff[i % T] : 1.0) * sabs[i % T] * h[i];
    return ev_collect(st);
}

// The adjoint reverse sweep (lambda already seeded) and the
// gradient / value readback; value_host is added to the device-accumulated value.
static int reverse_and_collect(tqd_state *st, double *d_grad, int n_grad, double value_host, double *out_value,
                               double *out_grad) {
    tqd_ctx *c = st->ctx;
    int rc;
    // reverse sweep down to (and including) the earliest stage holding a trainable gate
    int first = -1;
    for (size_t i = 0; i < st->history.size() && first < 0; i++) {
        const Stage &s = st->history[i];
        const std::vector<POp> *ops = s.type == ST_SWEEP ? &s.sw.ops : s.type == ST_SMALL ? &s.sm.ops : nullptr;
        if (!ops) continue;
        for (const POp &o : *ops)
            if (st->gates[o.gate].ngen) { first = (int)i; break; }
    }
    const bool pf_grads = prefix_has_grads(st);  // lambda down to the prefix boundary
    if (pf_grads && !st->history.empty()) first = 0;
    if (first >= 0) {
        // backward stage list = the forward history reversed; its descriptors are
        // cached with the forward plan when the history is the cached one
        const bool cacheable = st->history_cached && st->fwd_cache_version == st->tape_version;
        if (!(cacheable && st->bwd_cache_version == st->tape_version && st->enc_bwd->valid)) {
            st->rev_stages.clear();
            for (int i = (int)st->history.size() - 1; i >= first; i--) st->rev_stages.push_back(st->history[i]);
            Encoded &E = cacheable ? *st->enc_bwd : *st->enc_tmp;
            rc = encode_upload(st, st->rev_stages, true, E);
            if (rc) return rc;
            st->bwd_cache_version = cacheable ? st->tape_version : ~0ull;
            st->bwd_vhash = cacheable ? st->fwd_vhash : 0;
            rc = launch_encoded(st, st->rev_stages, true, E, d_grad);
        } else {
            rc = launch_graphed(st, st->rev_stages, true, *st->enc_bwd, d_grad, st->g_bwd, st->g_bwd_key, st->g_bwd_delta);
        }
        if (rc) return rc;
    }
    rc = allreduce_sum(st, st->d_red, (size_t)n_grad + 1);
    if (rc) return rc;
    std::vector<double> h(n_grad + 1);
    CUDA_TRY(st, cudaMemcpyAsync(h.data(), st->d_red, (n_grad + 1) * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(st, cudaStreamSynchronize(c->stream));
    st->met.d2h_bytes += (n_grad + 1) * sizeof(double);
    *out_value = h[0] + value_host;
    for (int p = 0; p < n_grad; p++) out_grad[p] = h[p + 1];
    if (pf_grads) {
        std::vector<double> pg(n_grad, 0.0);
        rc = prefix_grads(st, pg);
        if (rc) return rc;
        for (int p = 0; p < n_grad; p++) out_grad[p] += pg[p];
    }
    st->consumed = true;
    return ev_collect(st);
}

// Observable absorption (Heisenberg picture): E = <psi_K|H|psi_K> with
// psi_K = U_tail psi_p equals <psi_p|U_tail^dag H U_tail|psi_p>.  For a Z-string
// H (PAPER.md:308 measure_allZ; the adjoint seed of PAPER.md:226-231) a trailing
// run of gates that are diagonal or permutations-with-phase maps H to Z strings
// again, gate by gate from the last one:
//   diagonal (RZ, Z, S, T, CZ, CP, diagonal MAT1/MAT2): commutes, dropped;
//   anti-diagonal 1q (X, Y) on q: Z_q -> -Z_q;
//   controlled anti-diagonal (CNOT) [c, t]: Z_t -> Z_c Z_t, Z_c unchanged;
//   SWAP(a, b): exchanges bits a and b of the mask.
// Those gates are never applied (the state is consumed by the adjoint anyway);
// trainable gates in the run are diagonal (RZ) and their gradient is exactly 0
// (d/dtheta of a diagonal commuting with H).  Returns the first absorbed gate;
// z / sgn are updated in place.  Stops at anything else, at batched non-diagonal
// gates and at already executed gates.
static size_t absorb_tail(const std::vector<GateRec> &gates, size_t executed, std::vector<uint64_t> &z,
                          std::vector<double> &sgn) {
    auto zero = [](cd v) { return v.real() == 0.0 && v.imag() == 0.0; };
    size_t i = gates.size();
    while (i > executed) {
        const GateRec &g = gates[i - 1];
        const bool diag = g.cls == CL_IDENT || g.cls == CL_DIAG1 || g.cls == CL_DIAG2;
        if (!diag && (g.batched || g.trainable)) break;
        if (diag) {
            // commutes with every Z string
        } else if (g.cls == CL_SWAP) {
            const int a = g.w[0], b = g.w[1];
            for (auto &m : z) {
                const uint64_t ba = (m >> a) & 1ull, bb = (m >> b) & 1ull;
                if (ba != bb) m ^= (1ull << a) | (1ull << b);
            }
        } else if (g.cls == CL_U1 && zero(g.M[0]) && zero(g.M[3])) {
            for (size_t t = 0; t < z.size(); t++)
                if ((z[t] >> g.w[0]) & 1ull) sgn[t] = -sgn[t];
        } else if (g.cls == CL_CTRL1 && zero(g.sub[0]) && zero(g.sub[3])) {
            for (auto &m : z)
                if ((m >> g.w[1]) & 1ull) m ^= 1ull << g.w[0];
        } else {
            break;
        }
        i--;
    }
    return i;
}

// Z-string seed of one batch element in physical masks (lambda-init form, ZTerms)
static void build_zterms(const tqd_state *st, int T, const uint64_t *x, const uint64_t *z, const double *coeff,
                         const std::vector<double> &sabs, size_t cb, ZTerms &zt) {
    memset(&zt, 0, sizeof(zt));
    for (int t = 0; t < T; t++) {
        if (x && x[t]) continue;  // X / Y strings: lambda_add_xy
        const uint64_t zp = phys_mask(st, z[t]);
        const double ct = (coeff ? coeff[cb + t] : 1.0) * sabs[t];
        if (zp == 0) {  // identity (e.g. Z_q Z_q after absorption)
            zt.cst += ct;
        } else if (__builtin_popcountll(zp) == 1) {  // c (1 - 2 b_p)
            zt.cst += ct;
            zt.w[__builtin_ctzll(zp)] += ct;
        } else {
            zt.z[zt.T] = zp;
            zt.c[zt.T] = ct;
            zt.T++;
        }
    }
}

// ---- layout-circuit encoder (circuit_l3_kernel; tqd_internal.h L3Op) -----------
struct L3Enc {
    std::vector<L3Op> ops;       // batch x (nf + nb)
    std::vector<uint32_t> xtab;  // rows x threads
    std::vector<uint16_t> xreg;  // rows x 16
    std::vector<uint16_t> accp;  // batch x nacc: parameter index of each gradient accumulator
    std::vector<double> gtab;    // batch x ngt x 8: general generators
    int nf = 0, nb = 0, rows = 0, nacc = 0, ngt = 0;
    std::vector<int> pos;        // qubit map after the forward (the seed's Z masks)
};

static int gf2_rank(std::vector<uint32_t> v, int nbits) {
    int rank = 0;
    for (int bit = 0; bit < nbits; bit++) {
        int piv = -1;
        for (int i = rank; i < (int)v.size(); i++)
            if ((v[i] >> bit) & 1u) { piv = i; break; }
        if (piv < 0) continue;
        std::swap(v[rank], v[piv]);
        for (int i = 0; i < (int)v.size(); i++)
            if (i != rank && ((v[i] >> bit) & 1u)) v[i] ^= v[rank];
        rank++;
    }
    return rank;
}

// Plan + encode the whole circuit for circuit_l3_kernel: gates [0, end) forward,
// [skip_below, end) reversed with gradients.  Layouts: a gate whose target is not in
// a register slot triggers an exchange that brings in the next (up to) three
// register targets of the sequence (Belady: evict register bits not needed next);
// SWAP is a relabeling of the qubit map.  false: a gate this kernel does not take
// (general 2-qubit), or the state is out of range.
static bool encode_l3(tqd_state *st, size_t end, int skip_below, L3Enc &E) {
    const int n = st->n_loc;
    if (n < 8 || n > 10 || st->n_params > 65535) return false;
    const int T = 1 << (n - 3);
    const int LB = st->dbl ? 3 : 4;  // lane bits of one bank phase (16-B / 8-B elements)
    struct Item { int gate; bool bwd; int b0, b1, need; };
    std::vector<Item> seq;
    std::vector<int> pos = st->pos;
    auto add = [&](int i, bool bwd) -> bool {
        const GateRec &g = st->gates[i];
        if (g.cls == CL_U2) return false;
        if (g.cls == CL_IDENT) return true;
        if (g.cls == CL_SWAP) {
            std::swap(pos[g.w[0]], pos[g.w[1]]);
            return true;
        }
        Item it{i, bwd, pos[g.w[0]], g.nw > 1 ? pos[g.w[1]] : -1, -1};
        if (g.cls == CL_U1) it.need = it.b0;
        else if (g.cls == CL_CTRL1) it.need = it.b1;
        seq.push_back(it);
        return true;
    };
    for (size_t i = 0; i < end; i++)
        if (!add((int)i, false)) return false;
    E.pos = pos;
    E.nf = (int)seq.size();
    for (int i = (int)end - 1; i >= skip_below; i--)
        if (!add(i, true)) return false;
    // layouts (slot -> physical bit) and the op order (exchanges before items)
    std::vector<int> lay(n), where(n);
    {
        std::vector<int> first;
        for (const Item &it : seq)
            if (it.need >= 0 && std::find(first.begin(), first.end(), it.need) == first.end()) {
                first.push_back(it.need);
                if (first.size() == 3) break;
            }
        std::vector<char> used(n, 0);
        for (int b : first) used[b] = 1;
        int s = 0;
        for (int b : first) lay[s++] = b;
        for (int b = 0; b < n; b++)
            if (!used[b]) lay[s++] = b;
        for (int q = 0; q < n; q++) where[lay[q]] = q;
    }
    struct Ent { int item; int xrow; std::vector<int> wh; };  // item >= 0: gate item, else exchange row
    std::vector<Ent> order;
    std::vector<std::vector<int>> lays;  // per row: rows 0, 1 plain layouts; exchanges: old, new
    std::vector<std::vector<int>> xnew;
    lays.push_back(lay);                 // row 0
    lays.push_back(lay);                 // row 1 (seed layout, set below)
    xnew.push_back(lay);
    xnew.push_back(lay);
    int nf_ops = -1;
    for (size_t k = 0; k <= seq.size(); k++) {
        if ((int)k == E.nf) {
            lays[1] = lay;
            nf_ops = (int)order.size();
        }
        if (k == seq.size()) break;
        const Item &it = seq[k];
        if (it.need >= 0 && where[it.need] >= 3) {
            std::vector<int> want;
            for (size_t kk = k; kk < seq.size() && want.size() < 3; kk++) {
                const int nd = seq[kk].need;
                if (nd >= 0 && std::find(want.begin(), want.end(), nd) == want.end()) want.push_back(nd);
            }
            std::vector<int> nl = lay;
            std::vector<int> evict;
            for (int s = 0; s < 3; s++)
                if (std::find(want.begin(), want.end(), lay[s]) == want.end()) evict.push_back(s);
            size_t ei = 0;
            for (int b : want) {
                if (where[b] < 3) continue;
                const int s = evict[ei++];
                nl[where[b]] = lay[s];
                nl[s] = b;
            }
            lays.push_back(lay);
            xnew.push_back(nl);
            order.push_back(Ent{-1, (int)lays.size() - 1, {}});
            lay = nl;
            for (int q = 0; q < n; q++) where[lay[q]] = q;
        }
        order.push_back(Ent{(int)k, -1, where});
    }
    E.rows = (int)lays.size();
    if (E.rows > 65535) return false;
    E.xtab.assign((size_t)E.rows * T, 0);
    E.xreg.assign((size_t)E.rows * 16, 0);
    auto thr = [&](const std::vector<int> &L, int t) {
        uint32_t v = 0;
        for (int i = 0; i < n - 3; i++) v |= (uint32_t)((t >> i) & 1) << L[3 + i];
        return v;
    };
    auto roff = [&](const std::vector<int> &L, int r) {
        uint32_t v = 0;
        for (int j = 0; j < 3; j++) v |= (uint32_t)((r >> j) & 1) << L[j];
        return v;
    };
    for (int e = 0; e < 2; e++) {
        for (int t = 0; t < T; t++) E.xtab[(size_t)e * T + t] = thr(lays[e], t);
        for (int r = 0; r < 8; r++) E.xreg[(size_t)e * 16 + r] = (uint16_t)roff(lays[e], r);
    }
    const uint32_t lowm = (1u << LB) - 1;
    uint64_t rs = 0x2545F4914F6CDD1Dull;
    for (int e = 2; e < E.rows; e++) {
        const std::vector<int> &Lo = lays[e], &Ln = xnew[e];
        // F: column per physical bit (LB bits), identity on the low bits; conflict-free
        // when both layouts' first LB lane bits map to independent columns
        std::vector<uint32_t> col(n);
        for (int p = 0; p < n; p++) col[p] = p < LB ? (1u << p) : 0u;
        auto ok = [&]() {
            std::vector<uint32_t> a(LB), b(LB);
            for (int i = 0; i < LB; i++) {
                a[i] = col[Lo[3 + i]];
                b[i] = col[Ln[3 + i]];
            }
            return gf2_rank(a, LB) == LB && gf2_rank(b, LB) == LB;
        };
        bool good = ok();
        for (int tries = 0; tries < 4000 && !good; tries++) {
            for (int p = LB; p < n; p++) {
                rs ^= rs << 13; rs ^= rs >> 7; rs ^= rs << 17;
                col[p] = (uint32_t)(rs & lowm);
            }
            good = ok();
        }
        if (!good)
            for (int p = 0; p < n; p++) col[p] = p < LB ? (1u << p) : 0u;
        auto S = [&](uint32_t x) {
            uint32_t f = 0;
            for (int p = 0; p < n; p++)
                if ((x >> p) & 1u) f ^= col[p];
            return (x & ~lowm) | f;
        };
        for (int t = 0; t < T; t++) E.xtab[(size_t)e * T + t] = S(thr(Lo, t)) | (S(thr(Ln, t)) << 16);
        for (int r = 0; r < 8; r++) {
            E.xreg[(size_t)e * 16 + r] = (uint16_t)S(roff(Lo, r));
            E.xreg[(size_t)e * 16 + 8 + r] = (uint16_t)S(roff(Ln, r));
        }
    }
    // accumulators / general generators (structure: the same for every batch element)
    std::vector<int> acc0(seq.size(), -1), gi0(seq.size(), -1);
    for (size_t k = E.nf; k < seq.size(); k++) {
        const GateRec &g = st->gates[seq[k].gate];
        if (!g.ngen) continue;
        acc0[k] = E.nacc;
        E.nacc += g.ngen;
        bool full = false;
        for (int p = 0; p < g.ngen; p++) full = full || (g.gkind[p] != GEN_X && g.gkind[p] != GEN_Y);
        if (full && g.cls == CL_U1) {
            gi0[k] = E.ngt;
            E.ngt += g.ngen;
        }
    }
    const int nops = (int)order.size();
    E.nb = nops - nf_ops;
    E.nf = nf_ops;
    E.ops.assign((size_t)st->batch * nops, L3Op());
    E.accp.assign((size_t)st->batch * E.nacc, 0);
    E.gtab.assign((size_t)st->batch * E.ngt * 8, 0.0);
    std::vector<GateRec> tmp;
    for (int b = 0; b < st->batch; b++) {
        const std::vector<GateRec> &gb = gates_for(st, b, tmp);
        for (int oi = 0; oi < nops; oi++) {
            L3Op &o = E.ops[(size_t)b * nops + oi];
            memset(&o, 0, sizeof(o));
            const Ent &en = order[oi];
            if (en.item < 0) {
                o.type = L3_X;
                o.xi = (uint16_t)en.xrow;
                continue;
            }
            const Item &it = seq[en.item];
            const GateRec &g = gb[it.gate];
            const bool bwd = it.bwd;
            auto bk = [&](int bit, uint8_t &kind, uint8_t &idx) {
                const int sl = en.wh[bit];
                kind = sl < 3 ? 1 : 2;
                idx = (uint8_t)(sl < 3 ? sl : sl - 3);
            };
            auto put = [&](int i, cd v) {
                if (bwd) v = std::conj(v);
                o.m[2 * i] = v.real();
                o.m[2 * i + 1] = v.imag();
            };
            if (g.cls == CL_U1 || g.cls == CL_CTRL1) {
                const cd *M = g.cls == CL_U1 ? g.M : g.sub;
                o.type = L3_U1;
                o.j = (uint8_t)en.wh[it.need];
                if (g.cls == CL_CTRL1) bk(it.b0, o.ck, o.ci);
                // forward M, adjoint M^dag (conj of the transpose)
                put(0, M[0]);
                put(1, bwd ? M[2] : M[1]);
                put(2, bwd ? M[1] : M[2]);
                put(3, M[3]);
                bool real = true;
                for (int i = 0; i < 4; i++) real = real && o.m[2 * i + 1] == 0.0;
                const bool swp = o.m[0] == 0.0 && o.m[1] == 0.0 && o.m[6] == 0.0 && o.m[7] == 0.0 && o.m[2] == 1.0 &&
                                 o.m[3] == 0.0 && o.m[4] == 1.0 && o.m[5] == 0.0;
                o.form = swp ? L3F_SWAP : real ? L3F_REAL : L3F_GEN;
            } else if (g.cls == CL_DIAG1) {
                o.type = L3_D1;
                bk(it.b0, o.d0k, o.d0i);
                put(0, g.M[0]);
                put(1, g.M[3]);
            } else {  // CL_DIAG2: index 2 bit(w0) + bit(w1)
                o.type = L3_D2;
                bk(it.b0, o.d0k, o.d0i);
                bk(it.b1, o.d1k, o.d1i);
                for (int i = 0; i < 4; i++) put(i, g.M[5 * i]);
            }
            if (bwd && g.ngen) {
                o.ngen = (uint8_t)g.ngen;
                for (int p = 0; p < g.ngen; p++) {
                    o.gk[p] = g.gkind[p];
                    o.acc[p] = (uint16_t)(acc0[en.item] + p);
                    E.accp[(size_t)b * E.nacc + acc0[en.item] + p] = (uint16_t)(g.slot0 + p);
                }
                if (gi0[en.item] >= 0) {
                    o.gi = (uint16_t)gi0[en.item];
                    for (int p = 0; p < g.ngen; p++)
                        for (int i = 0; i < 4; i++) {
                            E.gtab[((size_t)b * E.ngt + gi0[en.item] + p) * 8 + 2 * i] = g.G[p][i].real();
                            E.gtab[((size_t)b * E.ngt + gi0[en.item] + p) * 8 + 2 * i + 1] = g.G[p][i].imag();
                        }
                }
            }
        }
    }
    return true;
}

// The whole circuit in ONE launch (circuit_kernel): forward gates, lambda = H psi and
// the reverse sweep with gradients, one CTA per batch element, for single-GPU states
// of <= opt_circuit qubits (BASELINE.json configs[0]: 10 qubits complex128).  The op
// lists are cached by tape version (tqd_state_rewind replays upload nothing).
// Returns 1 when the state does not qualify (the caller runs the staged path).
static int adjoint_circuit(tqd_state *st, int T, const uint64_t *x, const uint64_t *z, const double *coeff,
                           const std::vector<double> &sabs, size_t end, double *out_value, double *out_grad, int n_grad) {
    tqd_ctx *c = st->ctx;
    if (c->world != 1 || st->executed != 0 || st->n_loc > st->opt_circuit) return 1;
    for (int t = 0; t < T && x; t++)
        if (x[t]) return 1;
    const size_t smem = (size_t)2 * shard_bytes(st);
    if (smem > 200 * 1024) return 1;
    const uint64_t key = (st->tape_version * 0x9E3779B97F4A7C15ull) ^ (uint64_t)(st->gates.size() - end) ^
                         ((uint64_t)T << 40);
    std::vector<ZTerms> zts(st->batch);
    auto dev_alloc = [&](size_t total) -> int {
        if (total > st->circ_cap) {
            if (st->circ_dev) { CUDA_TRY(st, cudaStreamSynchronize(c->stream)); cudaFree(st->circ_dev); }
            st->circ_dev = nullptr;
            st->circ_cap = 0;
            if (cudaMalloc(&st->circ_dev, total) != cudaSuccess) {
                cudaGetLastError();
                return fail(TQD_ERR_OOM, "cannot allocate the circuit op lists");
            }
            st->circ_cap = total;
        }
        return TQD_OK;
    };
    if (st->circ_key != key || !st->circ_dev) {
        int skip_below = (int)st->gates.size();
        for (size_t i = 0; i < st->gates.size(); i++)
            if (st->gates[i].ngen) { skip_below = (int)i; break; }
        L3Enc E;
        st->circ_l3 = st->opt_layout && encode_l3(st, end, skip_below, E) &&
                      circuit_l3_smem(st->dbl, st->n_loc, E.nf + E.nb, E.rows, E.ngt, E.nacc) <= 220 * 1024;
        if (st->circ_l3) {
            // device: [ops][xtab][xreg][accp][gtab][Z terms]
            auto al = [](size_t v) { return (v + 255) & ~(size_t)255; };
            st->l3_nf = E.nf;
            st->l3_nb = E.nb;
            st->l3_rows = E.rows;
            st->l3_nacc = E.nacc;
            st->l3_ngt = E.ngt;
            st->l3_off_x = al(E.ops.size() * sizeof(L3Op));
            st->l3_off_r = al(st->l3_off_x + E.xtab.size() * sizeof(uint32_t));
            st->l3_off_a = al(st->l3_off_r + E.xreg.size() * sizeof(uint16_t));
            st->l3_off_g = al(st->l3_off_a + E.accp.size() * sizeof(uint16_t));
            st->circ_off_z = al(st->l3_off_g + E.gtab.size() * sizeof(double));
            int rc = dev_alloc(st->circ_off_z + zts.size() * sizeof(ZTerms));
            if (rc) return rc;
            char *d = (char *)st->circ_dev;
            CUDA_TRY(st, cudaMemcpyAsync(d, E.ops.data(), E.ops.size() * sizeof(L3Op), cudaMemcpyHostToDevice, c->stream));
            CUDA_TRY(st, cudaMemcpyAsync(d + st->l3_off_x, E.xtab.data(), E.xtab.size() * sizeof(uint32_t),
                                         cudaMemcpyHostToDevice, c->stream));
            CUDA_TRY(st, cudaMemcpyAsync(d + st->l3_off_r, E.xreg.data(), E.xreg.size() * sizeof(uint16_t),
                                         cudaMemcpyHostToDevice, c->stream));
            if (!E.accp.empty())
                CUDA_TRY(st, cudaMemcpyAsync(d + st->l3_off_a, E.accp.data(), E.accp.size() * sizeof(uint16_t),
                                             cudaMemcpyHostToDevice, c->stream));
            if (!E.gtab.empty())
                CUDA_TRY(st, cudaMemcpyAsync(d + st->l3_off_g, E.gtab.data(), E.gtab.size() * sizeof(double),
                                             cudaMemcpyHostToDevice, c->stream));
            st->met.h2d_bytes += E.ops.size() * sizeof(L3Op) + E.xtab.size() * 4 + E.xreg.size() * 2 +
                                 E.accp.size() * 2 + E.gtab.size() * 8;
            CUDA_TRY(st, cudaStreamSynchronize(c->stream));  // host vectors go out of scope
            st->pos = E.pos;  // lambda-init sees the final qubit map
            st->circ_key = key;
            st->circ_pos = E.pos;
        } else {
        std::vector<int> pending;
        for (size_t i = 0; i < end; i++) pending.push_back((int)i);
        PlanConfig cfg = plan_cfg(st);
        cfg.small_max = st->n_loc;
        std::vector<int> pos = st->pos;
        std::vector<Stage> stages;
        std::string err;
        int rc = plan_circuit(st->gates, pending, pos, cfg, stages, err);
        if (rc) return fail(rc, err);
        for (const Stage &s : stages)
            if (s.type != ST_SMALL) return 1;
        std::vector<DevOp> fops, bops;
        std::vector<GateRec> tmp;
        for (int b = 0; b < st->batch; b++) {
            const std::vector<GateRec> &gb = gates_for(st, b, tmp);
            for (const Stage &s : stages) encode_small(s.sm, gb, false, fops, 0);
            for (int i = (int)stages.size() - 1; i >= 0; i--) encode_small(stages[i].sm, gb, true, bops, skip_below);
        }
        st->pos = pos;  // lambda-init sees the final qubit map
        st->circ_nf = (int)fops.size() / st->batch;
        st->circ_nb = (int)bops.size() / st->batch;
        st->circ_off_b = ((fops.size() * sizeof(DevOp)) + 255) & ~(size_t)255;
        st->circ_off_z = (st->circ_off_b + bops.size() * sizeof(DevOp) + 255) & ~(size_t)255;
        rc = dev_alloc(st->circ_off_z + zts.size() * sizeof(ZTerms));
        if (rc) return rc;
        CUDA_TRY(st, cudaMemcpyAsync(st->circ_dev, fops.data(), fops.size() * sizeof(DevOp), cudaMemcpyHostToDevice, c->stream));
        CUDA_TRY(st, cudaMemcpyAsync((char *)st->circ_dev + st->circ_off_b, bops.data(), bops.size() * sizeof(DevOp),
                                     cudaMemcpyHostToDevice, c->stream));
        st->met.h2d_bytes += (fops.size() + bops.size()) * sizeof(DevOp);
        CUDA_TRY(st, cudaStreamSynchronize(c->stream));  // host vectors go out of scope
        st->circ_key = key;
        st->circ_pos = pos;
        }
    } else {
        st->pos = st->circ_pos;
    }
    for (int b = 0; b < st->batch; b++) build_zterms(st, T, x, z, coeff, sabs, (size_t)b * T, zts[b]);
    ZTerms *d_z = (ZTerms *)((char *)st->circ_dev + st->circ_off_z);
    CUDA_TRY(st, cudaMemcpyAsync(d_z, zts.data(), zts.size() * sizeof(ZTerms), cudaMemcpyHostToDevice, c->stream));
    st->met.h2d_bytes += zts.size() * sizeof(ZTerms);
    int rc = ensure_red(st, (size_t)n_grad + 1);
    if (rc) return rc;
    CUDA_TRY(st, cudaMemsetAsync(st->d_red, 0, (n_grad + 1) * sizeof(double), c->stream));
    const int ev = ev_begin(st, CAT_BWD);
    if (st->circ_l3) {
        const char *d = (const char *)st->circ_dev;
        CUDA_TRY(st, launch_circuit_l3(st->dbl, (const L3Op *)d, st->l3_nf, st->l3_nb, (const uint32_t *)(d + st->l3_off_x),
                                       (const uint16_t *)(d + st->l3_off_r), st->l3_rows,
                                       (const uint16_t *)(d + st->l3_off_a), st->l3_nacc,
                                       (const double *)(d + st->l3_off_g), st->l3_ngt, st->psi, d_z, st->d_red,
                                       st->d_red + 1, st->n_loc, st->batch, c->stream));
        st->met.circuit_layout_launches++;
    } else {
        const DevOp *d_f = (const DevOp *)st->circ_dev;
        const DevOp *d_b = (const DevOp *)((char *)st->circ_dev + st->circ_off_b);
        CUDA_TRY(st, launch_circuit(st->dbl, d_f, st->circ_nf, d_b, st->circ_nb, st->psi, d_z, st->d_red, st->d_red + 1,
                                    st->n_loc, rank_hi(st), st->batch, c->stream));
    }
    ev_end(st, ev);
    st->met.kernel_launches++;
    st->met.fwd_sweeps++;
    st->met.bwd_sweeps++;
    st->met.gates_applied += end * st->batch;
    st->met.gates_unapplied += end * st->batch;
    st->met.hbm_bytes += all_bytes(st);
    std::vector<double> h(n_grad + 1);
    CUDA_TRY(st, cudaMemcpyAsync(h.data(), st->d_red, (n_grad + 1) * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(st, cudaStreamSynchronize(c->stream));
    st->met.d2h_bytes += (n_grad + 1) * sizeof(double);
    *out_value = h[0];
    for (int p = 0; p < n_grad; p++) out_grad[p] = h[p + 1];
    st->executed = st->gates.size();
    st->consumed = true;
    return ev_collect(st);
}

int tqd_adjoint_grad(tqd_state *st, int T, const uint64_t *x, const uint64_t *z, const double *coeff, double *out_value,
                     double *out_grad, int n_grad) {
    int rc = check_live(st);
    if (rc) return rc;
    if (st->consumed) return fail(TQD_ERR_STATE, "state consumed by tqd_adjoint_grad; call tqd_state_reset");
    if (!out_value) return fail(TQD_ERR_ARG, "out_value is NULL");
    if (n_grad != st->n_params) return fail(TQD_ERR_ARG, "n_grad != tqd_num_params");
    if (n_grad > 0 && !out_grad) return fail(TQD_ERR_ARG, "out_grad is NULL");
    rc = check_terms(st, T, x, z);
    if (rc) return rc;
    if (T > 64) return fail(TQD_ERR_UNSUPPORTED, "at most 64 observable terms in tqd_adjoint_grad");
    // Z-only observables absorb the circuit's trailing diagonal / permutation gates
    std::vector<uint64_t> zabs(z, z + T);
    std::vector<double> sabs(T, 1.0);
    size_t end = st->gates.size();
    bool z_only = true;
    for (int t = 0; t < T && x; t++)
        if (x[t]) z_only = false;
    if (st->opt_absorb && z_only) {
        end = absorb_tail(st->gates, st->executed, zabs, sabs);
        z = zabs.data();
    }
    st->met.gates_absorbed += st->gates.size() - end;
    {
        const int crc = adjoint_circuit(st, T, x, z, coeff, sabs, end, out_value, out_grad, n_grad);
        if (crc <= 0) return crc;  // 1: the staged path below
    }
    // lambda first: the forward's remaps can then be fused into its sweeps (they
    // store into the owners' still idle lambda buffers)
    rc = ensure_lambda(st);
    if (rc) return rc;
    rc = execute_pending(st, end);
    if (rc) return rc;
    rc = ensure_red(st, (size_t)n_grad + 1);
    if (rc) return rc;
    tqd_ctx *c = st->ctx;
    double *d_val = st->d_red;
    double *d_grad = st->d_red + 1;
    CUDA_TRY(st, cudaMemsetAsync(st->d_red, 0, (n_grad + 1) * sizeof(double), c->stream));
    // the seed lambda = H psi per batch element; coefficients c[b * T + t] for a batch
    // (the VJP weights of every state), c[t] for a single state
    for (int bi = 0; bi < st->batch; bi++) {
        void *psi_b = (char *)st->psi + (size_t)bi * shard_bytes(st);
        void *lam_b = (char *)st->lam + (size_t)bi * shard_bytes(st);
        const size_t cb = (size_t)bi * T;
        ZTerms zt;
        memset(&zt, 0, sizeof(zt));
        for (int t = 0; t < T; t++) {
            if (x && x[t]) continue;  // X / Y strings: lambda_add_xy below
            const uint64_t zp = phys_mask(st, z[t]);
            const double ct = (coeff ? coeff[cb + t] : 1.0) * sabs[t];
            if (zp == 0) {  // identity (e.g. Z_q Z_q after absorption)
                zt.cst += ct;
            } else if (__builtin_popcountll(zp) == 1) {  // c (1 - 2 b_p)
                zt.cst += ct;
                zt.w[__builtin_ctzll(zp)] += ct;
            } else {
                zt.z[zt.T] = zp;
                zt.c[zt.T] = ct;
                zt.T++;
            }
        }
        const uint64_t N = 1ull << st->n_loc;
        {
            const int ev = ev_begin(st, CAT_OTHER);
            CUDA_TRY(st, launch_lambda_init(st->dbl, psi_b, lam_b, N, rank_hi(st), zt, d_val, c->stream));
            ev_end(st, ev);
            st->met.hbm_bytes += 2 * N * st->esz;
            st->met.kernel_launches++;
        }
        // X / Y strings: lambda += c_t P_t psi, grouped by x mask (<= 16 terms per launch);
        // x masks with rank bits pair the shard with the partner rank's (as in tqd_expval)
        if (x) {
            std::vector<char> done(T, 0);
            std::vector<uint64_t> hz;
            std::vector<int> hn;
            std::vector<double> hc;
            for (int t0 = 0; t0 < T; t0++) {
                if (done[t0] || !x[t0]) continue;
                std::vector<int> grp;
                for (int t = t0; t < T; t++)
                    if (!done[t] && x[t] == x[t0] && grp.size() < 16) grp.push_back(t);
                const uint64_t xp = phys_mask(st, x[t0]);
                const uint64_t xl = xp & (N - 1);
                const int gx = (int)(xp >> st->n_loc);
                hz.assign(16, 0);
                hn.assign(16, 0);
                hc.assign(16, 0.0);
                for (size_t i = 0; i < grp.size(); i++) {
                    hz[i] = phys_mask(st, z[grp[i]]);
                    hn[i] = __builtin_popcountll(x[grp[i]] & z[grp[i]]) & 3;
                    hc[i] = coeff ? coeff[cb + grp[i]] : 1.0;
                }
                rc = ensure_xy_scratch(st);
                if (rc) return rc;
                CUDA_TRY(st, cudaMemcpyAsync(st->d_xy, hz.data(), 16 * sizeof(uint64_t), cudaMemcpyHostToDevice, c->stream));
                CUDA_TRY(st, cudaMemcpyAsync(st->d_xy + 16, hc.data(), 16 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
                CUDA_TRY(st, cudaMemcpyAsync(st->d_xy + 32, hn.data(), 16 * sizeof(int), cudaMemcpyHostToDevice, c->stream));
                const int ev = ev_begin(st, CAT_OTHER);
                if (gx) {  // partner rank's shard, chunk by chunk (as in tqd_expval)
                    rc = xy_partner_chunks(st, psi_b, gx, xl, [&](uint64_t off, const void *pc, uint64_t cnt, uint64_t lo) {
                        CUDA_TRY(st, launch_lambda_add_xy(st->dbl, (const char *)psi_b + off * st->esz, pc,
                                                          (char *)lam_b + off * st->esz, cnt, rank_hi(st) | off, lo, xp,
                                                          st->d_xy, (const int *)(st->d_xy + 32),
                                                          (const double *)(st->d_xy + 16), (int)grp.size(), d_val,
                                                          c->stream));
                        return (int)TQD_OK;
                    });
                    if (rc) return rc;
                } else {
                    CUDA_TRY(st, launch_lambda_add_xy(st->dbl, psi_b, psi_b, lam_b, N, rank_hi(st), xl, xp, st->d_xy,
                                                      (const int *)(st->d_xy + 32), (const double *)(st->d_xy + 16),
                                                      (int)grp.size(), d_val, c->stream));
                }
                ev_end(st, ev);
                CUDA_TRY(st, cudaStreamSynchronize(c->stream));  // host staging vectors are reused
                st->met.h2d_bytes += 16 * (8 + 8 + 4);
                st->met.hbm_bytes += 4 * N * st->esz;
                st->met.kernel_launches++;
                for (int t : grp) done[t] = 1;
            }
        }
    }
    return reverse_and_collect(st, d_grad, n_grad, 0.0, out_value, out_grad);
}

// ---- shot noise: approximate (Gaussian) sampler, PAPER.md:200-218 -----------
// For batch element b (seed + b): the global sums of the sample's closed form
// (DESIGN.md §8c): m_q = <Z_q>, A_q = sum_i u_i z_i s_q(i), B = sum_i u_i z_i and
// psi at the last canonical outcome K; one reduction pass per 16 qubits.
struct GaussStats {
    std::vector<double> m, A;
    double B = 0, uK = 0, pKr = 0, pKi = 0;
};

static GatherMap canon_map(const tqd_state *st) {
    GatherMap gm;
    memset(&gm, 0, sizeof(gm));
    gm.n = st->n;
    gm.n_loc = st->n_loc;
    gm.rank = (uint64_t)st->ctx->rank;
    for (int b = 0; b < st->n; b++) gm.phys_of_canon_bit[b] = (uint8_t)st->pos[st->n - 1 - b];
    return gm;
}

static int gauss_stats(tqd_state *st, int b, uint64_t seed, GaussStats &gs) {
    tqd_ctx *c = st->ctx;
    const uint64_t N = 1ull << st->n_loc;
    const GatherMap gm = canon_map(st);
    const void *psi_b = (char *)st->psi + (size_t)b * shard_bytes(st);
    int rc = ensure_red(st, 40);
    if (rc) return rc;
    gs.m.assign(st->n, 0.0);
    gs.A.assign(st->n, 0.0);
    for (int q0 = 0; q0 < st->n; q0 += 16) {
        const int nq = std::min(16, st->n - q0);
        int qpos[16];
        for (int i = 0; i < nq; i++) qpos[i] = st->pos[q0 + i];
        CUDA_TRY(st, cudaMemsetAsync(st->d_red, 0, 35 * sizeof(double), c->stream));
        const int ev = ev_begin(st, CAT_OTHER);
        CUDA_TRY(st, launch_gauss_sums(st->dbl, psi_b, N, rank_hi(st), gm, seed, qpos, nq, st->d_red, c->stream));
        ev_end(st, ev);
        rc = allreduce_sum(st, st->d_red, 35);
        if (rc) return rc;
        double h[35];
        CUDA_TRY(st, cudaMemcpyAsync(h, st->d_red, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(st, cudaStreamSynchronize(c->stream));
        st->met.hbm_bytes += N * st->esz;
        st->met.kernel_launches++;
        st->met.d2h_bytes += sizeof(h);
        for (int i = 0; i < nq; i++) { gs.m[q0 + i] = h[i]; gs.A[q0 + i] = h[16 + i]; }
        gs.B = h[32];
        gs.pKr = h[33];
        gs.pKi = h[34];
    }
    gs.uK = std::sqrt(gs.pKr * gs.pKr + gs.pKi * gs.pKi);
    return TQD_OK;
}

// Zhat_q = m_q + (A_q + B F_q) / sqrt(shots),  F_q = (u_K s_q(K) - m_q) / (1 - u_K),
// s_q(K) = -1 (K = 1...1); the degenerate state u_K = 1 has no noise (v = 0).
static double gauss_F(const GaussStats &gs, int q) {
    const double D = 1.0 - gs.uK;
    return D > 1e-14 ? (-gs.uK - gs.m[q]) / D : 0.0;
}

int tqd_sample_gaussian_z(tqd_state *st, double shots, uint64_t seed, double *out) {
    int rc = check_live(st);
    if (rc) return rc;
    if (st->consumed) return fail(TQD_ERR_STATE, "state consumed by tqd_adjoint_grad; call tqd_state_reset");
    if (!out) return fail(TQD_ERR_ARG, "out is NULL");
    if (!(shots > 0)) return fail(TQD_ERR_ARG, "shots must be > 0");
    rc = execute_pending(st);
    if (rc) return rc;
    for (int b = 0; b < st->batch; b++) {
        GaussStats gs;
        rc = gauss_stats(st, b, seed + (uint64_t)b, gs);
        if (rc) return rc;
        for (int q = 0; q < st->n; q++)
            out[(size_t)b * st->n + q] = gs.m[q] + (gs.A[q] + gs.B * gauss_F(gs, q)) / std::sqrt(shots);
    }
    return ev_collect(st);
}

int tqd_adjoint_grad_gaussian(tqd_state *st, double shots, uint64_t seed, const double *coeff, double *out_value,
                              double *out_grad, int n_grad) {
    int rc = check_live(st);
    if (rc) return rc;
    if (st->consumed) return fail(TQD_ERR_STATE, "state consumed by tqd_adjoint_grad; call tqd_state_reset");
    if (!out_value) return fail(TQD_ERR_ARG, "out_value is NULL");
    if (!(shots > 0)) return fail(TQD_ERR_ARG, "shots must be > 0");
    if (n_grad != st->n_params) return fail(TQD_ERR_ARG, "n_grad != tqd_num_params");
    if (n_grad > 0 && !out_grad) return fail(TQD_ERR_ARG, "out_grad is NULL");
    rc = execute_pending(st);
    if (rc) return rc;
    rc = ensure_lambda(st);
    if (rc) return rc;
    // statistics of every element first (their reduction scratch is reused below)
    std::vector<GaussStats> all(st->batch);
    for (int b = 0; b < st->batch; b++) {
        rc = gauss_stats(st, b, seed + (uint64_t)b, all[b]);
        if (rc) return rc;
    }
    rc = ensure_red(st, (size_t)n_grad + 1);
    if (rc) return rc;
    tqd_ctx *c = st->ctx;
    CUDA_TRY(st, cudaMemsetAsync(st->d_red, 0, (n_grad + 1) * sizeof(double), c->stream));
    const GatherMap gm = canon_map(st);
    const uint64_t N = 1ull << st->n_loc;
    const double rs = std::sqrt(shots);
    double value = 0.0;
    for (int b = 0; b < st->batch; b++) {
        const GaussStats &gs = all[b];
        const double *cb = coeff ? coeff + (size_t)b * st->n : nullptr;
        // lambda = dL/dpsi* of L = sum_q c_q Zhat_q
        ZTerms zt;
        memset(&zt, 0, sizeof(zt));
        double fc = 0.0, sK = 0.0;
        for (int q = 0; q < st->n; q++) {
            const double cq = cb ? cb[q] : 1.0;
            zt.cst += cq;
            zt.w[st->pos[q]] += cq;
            fc += cq * gauss_F(gs, q);
            sK -= cq;
            value += cq * (gs.m[q] + (gs.A[q] + gs.B * gauss_F(gs, q)) / rs);
        }
        const double D = 1.0 - gs.uK;
        const double alpha = D > 1e-14 ? 1.0 - gs.B / (rs * D) : 1.0;
        const double kc = D > 1e-14 ? gs.B / (2.0 * rs * D) * (sK + fc) : 0.0;
        const int ev = ev_begin(st, CAT_OTHER);
        CUDA_TRY(st, launch_lambda_gauss(st->dbl, (char *)st->psi + (size_t)b * shard_bytes(st),
                                         (char *)st->lam + (size_t)b * shard_bytes(st), N, rank_hi(st), gm,
                                         seed + (uint64_t)b, zt, alpha, fc, 0.5 / rs, kc, c->stream));
        ev_end(st, ev);
        st->met.hbm_bytes += 2 * N * st->esz;
        st->met.kernel_launches++;
    }
    return reverse_and_collect(st, st->d_red + 1, n_grad, value, out_value, out_grad);
}

// ---- shot noise: exact hierarchical multinomial sampler, PAPER.md:184-198 ------
// counter-based uniforms, the library's own implementation of the definition in
// DESIGN.md R22 (splitmix64)
static uint64_t sm64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
static double uniform01(uint64_t seed, uint64_t k) {
    return (double)(sm64(seed ^ (k * 0xD1B54A32D192ED03ull)) >> 11) * 0x1.0p-53;
}

static int upload_bytes(tqd_state *st, void *&buf, size_t &cap, const void *src, size_t bytes) {
    const size_t need = std::max<size_t>(bytes, 1);
    if (cap < need) {
        if (buf) cudaFree(buf);
        buf = nullptr;
        cap = 0;
        if (cudaMalloc(&buf, need) != cudaSuccess) { cudaGetLastError(); return fail(TQD_ERR_OOM, "sampler scratch"); }
        cap = need;
    }
    if (bytes) CUDA_TRY(st, cudaMemcpyAsync(buf, src, bytes, cudaMemcpyHostToDevice, st->ctx->stream));
    st->met.h2d_bytes += bytes;
    return TQD_OK;
}
#define UPLOAD(st, buf, cap, vec) upload_bytes(st, buf, cap, (vec).data(), (vec).size() * sizeof((vec)[0]))

int tqd_sample(tqd_state *st, uint64_t shots, uint64_t seed, uint64_t *out) {
    int rc = check_live(st);
    if (rc) return rc;
    if (st->consumed) return fail(TQD_ERR_STATE, "state consumed by tqd_adjoint_grad; call tqd_state_reset");
    if (shots > 0 && !out) return fail(TQD_ERR_ARG, "out is NULL");
    if (shots > (1ull << 32)) return fail(TQD_ERR_ARG, "at most 2^32 shots per call");
    rc = execute_pending(st);
    if (rc) return rc;
    if (shots == 0) return ev_collect(st);
    tqd_ctx *c = st->ctx;
    const uint64_t N = 1ull << st->n_loc;
    const int csz = (int)std::min<uint64_t>((uint64_t)sample_chunk_amps(), N);
    const uint64_t n_chunks = N / (uint64_t)csz;
    const GatherMap gm = canon_map(st);
    void *d_mass = nullptr, *d_cid = nullptr, *d_off = nullptr, *d_r = nullptr, *d_idx = nullptr, *d_out = nullptr;
    size_t c_mass = 0, c_cid = 0, c_off = 0, c_r = 0, c_idx = 0;
    auto cleanup = [&]() {
        for (void *p : {d_mass, d_cid, d_off, d_r, d_idx, d_out}) if (p) cudaFree(p);
    };
    if (cudaMalloc(&d_out, shots * sizeof(double)) != cudaSuccess || cudaMalloc(&d_mass, n_chunks * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        cleanup();
        return fail(TQD_ERR_OOM, "sampler buffers");
    }
    rc = ensure_red(st, (size_t)c->world);
    if (rc) { cleanup(); return rc; }
    std::vector<double> host(shots);
    for (int b = 0; b < st->batch && rc == TQD_OK; b++) {
        const void *psi_b = (char *)st->psi + (size_t)b * shard_bytes(st);
        const uint64_t sb = seed + (uint64_t)b;
        // 1. probability mass of every chunk of the local shard
        std::vector<double> mass(n_chunks);
        if (launch_chunk_mass(st->dbl, psi_b, n_chunks, csz, (double *)d_mass, c->stream) != cudaSuccess ||
            cudaMemcpyAsync(mass.data(), d_mass, n_chunks * sizeof(double), cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
            cudaStreamSynchronize(c->stream) != cudaSuccess) {
            cleanup();
            c->poisoned = true;
            return fail(TQD_ERR_CUDA, cudaGetErrorString(cudaGetLastError()));
        }
        st->met.hbm_bytes += N * st->esz;
        st->met.kernel_launches++;
        double qloc = 0;
        for (double m : mass) qloc += m;
        // 2. the groups' masses q_j (one per rank) on every rank
        std::vector<double> q(c->world, 0.0);
        q[c->rank] = qloc;
        CUDA_TRY(st, cudaMemcpyAsync(st->d_red, q.data(), c->world * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        rc = allreduce_sum(st, st->d_red, c->world);
        if (rc) { cleanup(); return rc; }
        CUDA_TRY(st, cudaMemcpyAsync(q.data(), st->d_red, c->world * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(st, cudaStreamSynchronize(c->stream));
        std::vector<double> Q(c->world + 1, 0.0);
        for (int j = 0; j < c->world; j++) Q[j + 1] = Q[j] + q[j];
        int last_pos = 0;  // rank of the last positive mass (rounding guard)
        for (int j = 0; j < c->world; j++) if (q[j] > 0) last_pos = j;
        // 3. shared seed: every rank draws the same uniforms; shot k goes to group j with
        //    Q_j <= u_k Q_W < Q_{j+1} (y ~ Multinomial(shots, q)); the residual is uniform
        //    on the group's mass, i.e. the conditional sample of PAPER.md:194-196
        std::vector<std::pair<double, uint64_t>> mine;
        for (uint64_t kk = 0; kk < shots; kk++) {
            const double u = uniform01(sb, kk) * Q[c->world];
            int j = (int)(std::upper_bound(Q.begin() + 1, Q.end(), u) - (Q.begin() + 1));
            if (j >= c->world || q[j] <= 0) j = std::min(j, last_pos);
            while (q[j] <= 0 && j > 0) j--;
            if (j == c->rank) mine.push_back({std::min(u - Q[j], q[j]), kk});
        }
        std::sort(mine.begin(), mine.end());
        // 4. local: chunk of every shot from the chunks' prefix masses, residual inside it
        std::vector<uint64_t> cid, sidx;
        std::vector<uint32_t> off;
        std::vector<double> rr;
        double pre = 0;
        uint64_t ch = 0;
        uint64_t last_nz = 0;
        for (uint64_t i = 0; i < n_chunks; i++) if (mass[i] > 0) last_nz = i;
        for (size_t s = 0; s < mine.size(); s++) {
            const double u = mine[s].first;
            while (ch < last_nz && (pre + mass[ch] <= u || mass[ch] <= 0)) { pre += mass[ch]; ch++; }
            if (cid.empty() || cid.back() != ch) { cid.push_back(ch); off.push_back((uint32_t)rr.size()); }
            rr.push_back(u - pre);
            sidx.push_back(mine[s].second);
        }
        off.push_back((uint32_t)rr.size());
        CUDA_TRY(st, cudaMemsetAsync(d_out, 0, shots * sizeof(double), c->stream));
        if ((rc = UPLOAD(st, d_cid, c_cid, cid)) || (rc = UPLOAD(st, d_off, c_off, off)) ||
            (rc = UPLOAD(st, d_r, c_r, rr)) || (rc = UPLOAD(st, d_idx, c_idx, sidx))) {
            cleanup();
            return rc;
        }
        const int ev = ev_begin(st, CAT_OTHER);
        CUDA_TRY(st, launch_chunk_sample(st->dbl, psi_b, (int)cid.size(), (const uint64_t *)d_cid, (const uint32_t *)d_off,
                                         (const double *)d_r, (const uint64_t *)d_idx, rank_hi(st), gm, csz,
                                         (double *)d_out, c->stream));
        ev_end(st, ev);
        st->met.kernel_launches++;
        // 5. every rank wrote its own shots; the sum assembles all of them everywhere
        rc = allreduce_sum(st, (double *)d_out, shots);
        if (rc) { cleanup(); return rc; }
        CUDA_TRY(st, cudaMemcpyAsync(host.data(), d_out, shots * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(st, cudaStreamSynchronize(c->stream));
        st->met.d2h_bytes += shots * sizeof(double);
        for (uint64_t kk = 0; kk < shots; kk++) out[(size_t)b * shots + kk] = (uint64_t)host[kk];
    }
    cleanup();
    return ev_collect(st);
}

int tqd_get_amplitudes(tqd_state *st, uint64_t first, uint64_t count, void *host_out) {
    int rc = check_live(st);
    if (rc) return rc;
    if (st->consumed) return fail(TQD_ERR_STATE, "state consumed by tqd_adjoint_grad; call tqd_state_reset");
    if (count && !host_out) return fail(TQD_ERR_ARG, "host_out is NULL");
    const uint64_t per = 1ull << st->n;  // amplitudes per batch element; index b * 2^n + i
    const uint64_t total = per * (uint64_t)st->batch;
    if (first > total || count > total - first) return fail(TQD_ERR_ARG, "amplitude range out of bounds");
    rc = execute_pending(st);
    if (rc) return rc;
    if (count == 0) return ev_collect(st);
    GatherMap gm;
    memset(&gm, 0, sizeof(gm));
    gm.n = st->n;
    gm.n_loc = st->n_loc;
    gm.rank = (uint64_t)st->ctx->rank;
    for (int b = 0; b < st->n; b++) gm.phys_of_canon_bit[b] = (uint8_t)st->pos[st->n - 1 - b];
    const uint64_t chunk = std::min<uint64_t>(count, 1ull << 24);
    void *tmp = nullptr;
    if (cudaMalloc(&tmp, chunk * st->esz) != cudaSuccess) { cudaGetLastError(); return fail(TQD_ERR_OOM, "gather buffer"); }
    tqd_ctx *c = st->ctx;
    for (uint64_t o = 0; o < count;) {
        const uint64_t idx = first + o, bi = idx / per, in = idx % per;
        const uint64_t cnt = std::min(std::min(chunk, count - o), per - in);  // within one batch element
        cudaError_t e = launch_gather(st->dbl, (char *)st->psi + bi * shard_bytes(st), tmp, in, cnt, gm, c->stream);
        if (e == cudaSuccess && c->world > 1) {
            if (c->comm->allreduce_sum(tmp, cnt * 2, st->dbl ? CE_F64 : CE_F32, c->stream) != 0) {
                cudaFree(tmp);
                c->poisoned = true;
                return fail(TQD_ERR_NCCL, c->comm->err);
            }
        }
        if (e == cudaSuccess) e = cudaMemcpyAsync((char *)host_out + o * st->esz, tmp, cnt * st->esz, cudaMemcpyDeviceToHost, c->stream);
        st->met.d2h_bytes += cnt * st->esz;
        if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
        if (e != cudaSuccess) { cudaFree(tmp); c->poisoned = true; return fail(TQD_ERR_CUDA, cudaGetErrorString(e)); }
        st->met.kernel_launches++;
        o += cnt;
    }
    cudaFree(tmp);
    return ev_collect(st);
}

int tqd_get_metrics(const tqd_state *st, tqd_metrics *out) {
    if (!st || !out) return fail(TQD_ERR_ARG, "NULL argument");
    *out = st->met;
    return TQD_OK;
}

int tqd_reset_metrics(tqd_state *st) {
    if (!st) return fail(TQD_ERR_ARG, "state is NULL");
    const uint64_t peak = st->met.peak_device_bytes;
    memset(&st->met, 0, sizeof(st->met));
    st->met.peak_device_bytes = peak;
    return TQD_OK;
}

// Diagnostic (no GPU needed): plan a circuit and return the stages as JSON.
// gates: parallel arrays as in tqd_apply_gate (kinds[G], wires[2G], params[3G],
// mats[32G], trainable[G]).  Returns the needed size if cap is too small.
// circuit as parallel arrays (tqd_debug_plan / tqd_debug_absorb) -> gate records
static int parse_debug_gates(int n, int c128, int G, const int *kinds, const int *wires, const double *params,
                             const double *mats, const int *trainable, std::vector<GateRec> &gates) {
    int np = 0;
    for (int i = 0; i < G; i++) {
        GateRec r;
        std::string err;
        const int nw = gate_arity(kinds[i]);
        for (int j = 0; j < nw; j++)
            if (wires[2 * i + j] < 0 || wires[2 * i + j] >= n) return fail(TQD_ERR_ARG, "wire out of range");
        if (nw == 2 && wires[2 * i] == wires[2 * i + 1]) return fail(TQD_ERR_ARG, "duplicate wires");
        int rc = make_gate(kinds[i], wires + 2 * i, nw, params + 3 * i, mats + 32 * i, trainable[i], c128 != 0, r, err);
        if (rc) return fail(rc, err);
        if (r.trainable) { r.slot0 = np; np += gate_num_params(kinds[i]); }
        gates.push_back(r);
    }
    return TQD_OK;
}

int tqd_debug_absorb(int n, int G, const int *kinds, const int *wires, const double *params, const double *mats,
                     const int *trainable, int T, const uint64_t *z_in, uint64_t *z_out, double *sign_out,
                     int *tail_begin) {
    if (n < 1 || n > 63 || G < 0 || T < 0 || T > 64) return fail(TQD_ERR_ARG, "bad n, G or T");
    if ((G && (!kinds || !wires || !params || !mats || !trainable)) || (T && (!z_in || !z_out || !sign_out)) ||
        !tail_begin)
        return fail(TQD_ERR_ARG, "NULL argument");
    std::vector<GateRec> gates;
    int rc = parse_debug_gates(n, 1, G, kinds, wires, params, mats, trainable, gates);
    if (rc) return rc;
    std::vector<uint64_t> z(z_in, z_in + T);
    std::vector<double> sg(T, 1.0);
    *tail_begin = (int)absorb_tail(gates, 0, z, sg);
    for (int t = 0; t < T; t++) { z_out[t] = z[t]; sign_out[t] = sg[t]; }
    return TQD_OK;
}

int tqd_debug_plan(int n, int world, int k, int small_max, int c128, int G, const int *kinds, const int *wires,
                   const double *params, const double *mats, const int *trainable, char *json_out, size_t cap,
                   size_t *needed) {
    if (world < 1 || (world & (world - 1))) return fail(TQD_ERR_WORLD, "world size must be a power of two");
    int g = 0;
    while ((1 << g) < world) g++;
    if (n < g + 2 || n > 62) return fail(TQD_ERR_QUBITS, "bad n");
    std::vector<GateRec> gates;
    {
        int rc = parse_debug_gates(n, c128, G, kinds, wires, params, mats, trainable, gates);
        if (rc) return rc;
    }
    PlanConfig cfg = make_plan_cfg(n, n - g, k, small_max, c128 != 0);
    std::vector<int> pos(n);
    for (int q = 0; q < n; q++) pos[q] = n - 1 - q;
    std::vector<int> pending;
    for (int i = 0; i < G; i++) pending.push_back(i);
    std::vector<Stage> stages;
    std::string err;
    int rc = plan_circuit(gates, pending, pos, cfg, stages, err);
    if (rc) return fail(rc, err);
    if (getenv("TQD_DEBUG_KOPS")) {  // diagnostic: kernel-op counts per sweep stage (forward encoding)
        for (size_t si = 0; si < stages.size(); si++) {
            if (stages[si].type != ST_SWEEP) continue;
            DevStage ds;
            std::vector<KOp<float>> kops;
            std::vector<int32_t> slots;
            encode_sweep_k<float>(stages[si].sw, gates, false, n - g, ds, kops, slots);
            int cnt[KC_COUNT + 1] = {0};
            for (const auto &k : kops) cnt[std::min<int>(k.code, KC_COUNT)]++;
            fprintf(stderr, "stage %zu: %d kops:", si, (int)kops.size());
            for (int c = 0; c <= KC_COUNT; c++)
                if (cnt[c]) fprintf(stderr, " %d:%d", c, cnt[c]);
            fprintf(stderr, "  (C rows %d, U values %d)\n", ds.n_cvals, ds.n_uvals);
        }
    }
    std::string js = plan_to_json(stages, cfg);
    if (needed) *needed = js.size() + 1;
    if (!json_out || cap < js.size() + 1) return fail(TQD_ERR_ARG, "json buffer too small");
    memcpy(json_out, js.c_str(), js.size() + 1);
    return TQD_OK;
}

// Experiment (tensor cores): a dense m-qubit block on the
// m lowest bits of a 2^n complex64 state by tcgen05.mma (dense_tc.cu), on `device`.
int tqd_debug_dense_block(int device, int n, int m, int precision, const double *U, const void *psi_in, void *psi_out,
                          int iters, double *ms_out) {
    if (m != 6 || n < 13 || n > 33 || (precision != 1 && precision != 3) || !U || iters < 0)
        return fail(TQD_ERR_ARG, "dense block: m = 6, 13 <= n <= 33, precision 1 or 3");
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return fail(TQD_ERR_CUDA, cudaGetErrorString(e));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const uint64_t N = 1ull << n;
    float *x = nullptr;
    void *bs = nullptr;
    cudaStream_t s = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    auto done = [&](int rc, const char *msg) {
        if (s) cudaStreamSynchronize(s);
        if (x) cudaFree(x);
        if (bs) cudaFree(bs);
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
        if (s) cudaStreamDestroy(s);
        return rc ? fail(rc, msg) : TQD_OK;
    };
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess || cudaMalloc(&x, N * 8) != cudaSuccess ||
        cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
        cudaGetLastError();
        return done(TQD_ERR_OOM, "dense block buffers");
    }
    if ((e = dense_tc_upload(U, m, &bs, s)) != cudaSuccess) return done(TQD_ERR_CUDA, cudaGetErrorString(e));
    if (psi_in) e = cudaMemcpyAsync(x, psi_in, N * 8, cudaMemcpyHostToDevice, s);
    else e = cudaMemsetAsync(x, 0, N * 8, s);
    if (e == cudaSuccess) e = dense_tc_launch(x, N, bs, precision, sms, s);
    if (e == cudaSuccess && psi_out) e = cudaMemcpyAsync(psi_out, x, N * 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess && iters > 0) {
        e = cudaEventRecord(e0, s);
        for (int i = 0; i < iters && e == cudaSuccess; i++) e = dense_tc_launch(x, N, bs, precision, sms, s);
        if (e == cudaSuccess) e = cudaEventRecord(e1, s);
        if (e == cudaSuccess) e = cudaEventSynchronize(e1);
        float ms = 0;
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
        if (ms_out) *ms_out = ms / iters;
    }
    if (e != cudaSuccess) return done(TQD_ERR_CUDA, cudaGetErrorString(e));
    return done(TQD_OK, "");
}

// Diagnostic, host only: the remap exchange schedule of one rank.  For each
// send block b in [0, 2^m): peer_out[b] = destination rank, recv_block_out[b] =
// block index where the data received from that peer is placed.
int tqd_debug_remap_schedule(int rank, int n_loc, int m, const int *gpos, const int *lpos, int *peer_out,
                             int *recv_block_out) {
    if (m < 0 || m > 8 || !gpos || !lpos || !peer_out || !recv_block_out) return fail(TQD_ERR_ARG, "bad arguments");
    RemapPlan rp;
    rp.m = m;
    for (int i = 0; i < m; i++) {
        if (gpos[i] < n_loc || lpos[i] < 0 || lpos[i] >= n_loc) return fail(TQD_ERR_ARG, "bad positions");
        rp.gpos[i] = gpos[i];
        rp.lpos[i] = lpos[i];
    }
    std::vector<int> pr, ub;
    remap_schedule(rank, n_loc, rp, pr, ub);
    for (int b = 0; b < (1 << m); b++) {
        peer_out[b] = pr[b];
        recv_block_out[b] = ub[b];
    }
    return TQD_OK;
}

}  // extern "C"
