"""Multi-rank DEVICE path on one GPU: W ranks emulated in one process (one host
thread + one stream + one shard per rank) through the loopback transport
(include/tqd.h tqd_loopback_id).  Everything the ranks run on the device is the
product path for world > 1 -- rank-bit conditioned sweeps (diagonal gates and
controls on global qubits), remap pack / unpack around the
block exchange, sharded expval / lambda-init / adjoint partials and their sums,
the sharded readback -- only the transport between the shards is host-driven
copies instead of NCCL (no kernel waits on another rank's kernel).

Every rank's result is compared with the float64 oracle of the whole circuit.
"""
import threading
import traceback

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

TOL = {"c64": dict(amp=1e-5, val=1e-4), "c128": dict(amp=1e-12, val=1e-10)}


@pytest.fixture(scope="module")
def tqd():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need CUDA (run with -m 'not gpu' on CPU)")
    import paper_2511_19291_b200 as t
    return t


def run_world(tqd, world, fn, timeout=600):
    """fn(rank, ctx) on `world` threads sharing one loopback id; returns per-rank results."""
    lid = tqd.tqd_loopback_id()
    res, err = [None] * world, [None] * world

    def worker(r):
        try:
            ctx = tqd.Context(world, r, 0, lid)
            try:
                res[r] = fn(r, ctx)
            finally:
                ctx.close()
        except Exception:
            err[r] = traceback.format_exc()

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout)
    assert not any(t.is_alive() for t in th), "emulated world hung"
    bad = [f"rank {r}:\n{e}" for r, e in enumerate(err) if e is not None]
    assert not bad, "\n".join(bad)
    return res


def mixed_circuit(n, seed):
    return W.random_circuit(n, 120, seed) + W.hea(n, 2, seed) + W.qft(n)[:30]


@pytest.mark.parametrize("grid", [0, 3])
@pytest.mark.parametrize("fused", [1, 0])
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("world,n,k", [(2, 12, 9), (4, 13, 9), (8, 14, 9), (2, 16, 12), (4, 17, 12)])
def test_world_amplitudes(tqd, orc, world, n, k, dtype, fused, grid):
    """fused = 1: remaps fused into the preceding sweep (stores into the owners'
    peer memory); fused = 0: pack -> all-to-all -> unpack."""
    gates = mixed_circuit(n, world + n)

    def fn(r, ctx):
        st = tqd.State(ctx, n, dtype)
        st.set_option(tqd.OPT_TILE_QUBITS, k)
        st.set_option(tqd.OPT_SMALL_MAX, 0)
        st.set_option(tqd.OPT_FUSED_REMAP, fused)
        st.set_option(tqd.OPT_GRID_CTAS, grid)
        st.apply_circuit(gates)
        amp = st.amplitudes()
        m = st.metrics()
        st.free()
        return amp, m
    out = run_world(tqd, world, fn)
    ref = orc.run(n, gates)
    for amp, m in out:
        assert np.max(np.abs(amp - ref)) < TOL[dtype]["amp"]
        assert m["remaps"] > 0 and m["a2a_bytes"] > 0  # the exchange really ran
        assert (m["fused_remaps"] > 0) == bool(fused)


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("world,n", [(2, 12), (4, 14), (8, 15)])
def test_world_expval_pauli(tqd, orc, world, n, dtype):
    """Z strings and X/Y strings, including strings acting on the global qubits."""
    gates = mixed_circuit(n, 3 * world)
    terms = W.random_pauli_terms(n, 16, n) + W.random_z_terms(n, 16, n) + W.sum_z(n)
    # logical qubits 0..log2(world)-1 start on the rank bits (MSB-first)
    terms += [(1, 0, 0.7), (0, 1, -0.4), (3, 4, 1.1), (2, 1 | (1 << (n - 1)), 0.3)]

    def fn(r, ctx):
        st = tqd.State(ctx, n, dtype)
        st.set_option(tqd.OPT_TILE_QUBITS, 9)
        st.set_option(tqd.OPT_SMALL_MAX, 0)
        st.apply_circuit(gates)
        v = st.expval(terms)
        st.free()
        return v
    out = run_world(tqd, world, fn)
    ref = orc.expval(orc.run(n, gates), n, terms)
    for v in out:
        assert np.max(np.abs(v - ref)) < TOL[dtype]["val"]


@pytest.mark.parametrize("grid", [0, 3])
@pytest.mark.parametrize("fused", [1, 0])
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("world,n,k,small", [(2, 12, 9, False), (4, 14, 10, True), (8, 15, 9, True), (2, 17, 12, True)])
def test_world_adjoint(tqd, orc, world, n, k, small, dtype, fused, grid):
    """Adjoint gradients with remaps replayed on psi and lambda."""
    gates = W.random_circuit(n, 80, 5 + world, small=small) + W.hea(n, 3, world, small=small)
    terms = W.random_z_terms(n, 5, world) + W.sum_z(n)

    def fn(r, ctx):
        st = tqd.State(ctx, n, dtype)
        st.set_option(tqd.OPT_TILE_QUBITS, k)
        st.set_option(tqd.OPT_SMALL_MAX, 0)
        st.set_option(tqd.OPT_FUSED_REMAP, fused)
        st.set_option(tqd.OPT_GRID_CTAS, grid)
        st.apply_circuit(gates)
        val, grad = st.adjoint_grad(terms)
        st.free()
        return val, grad
    out = run_world(tqd, world, fn)
    rval, rgrad = orc.adjoint(n, gates, terms)
    for val, grad in out:
        assert abs(val - rval) < TOL[dtype]["val"]
        assert np.max(np.abs(grad - rgrad)) < TOL[dtype]["val"]


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("world,n", [(2, 12), (4, 14), (8, 15)])
def test_world_adjoint_pauli(tqd, orc, world, n, dtype):
    """X / Y strings in the adjoint seed, including X / Y on the rank bits (partner-shard exchange)."""
    gates = W.random_circuit(n, 60, 7 * world, small=True) + W.hea(n, 2, world, small=True)
    terms = W.random_pauli_terms(n, 10, world) + [(1, 0, 0.7), (3, 4, -1.1), (2, 1 | (1 << (n - 1)), 0.3)]

    def fn(r, ctx):
        st = tqd.State(ctx, n, dtype)
        st.set_option(tqd.OPT_TILE_QUBITS, 9)
        st.set_option(tqd.OPT_SMALL_MAX, 0)
        st.apply_circuit(gates)
        v = st.adjoint_grad(terms)
        st.free()
        return v
    rval, rgrad = orc.adjoint(n, gates, terms)
    for val, grad in run_world(tqd, world, fn):
        assert abs(val - rval) < TOL[dtype]["val"]
        assert np.max(np.abs(grad - rgrad)) < TOL[dtype]["val"]


def test_world_ghz_global_targets(tqd, orc):
    """GHZ with CNOT targets on the global qubits (forces remaps), read back on every rank."""
    n, world = 14, 4
    gates = [W.Gate("H", (n - 1,), (), None, True)] + [W.Gate("CNOT", (q + 1, q), (), None, True) for q in range(n - 2, -1, -1)]

    def fn(r, ctx):
        st = tqd.State(ctx, n, "c128")
        st.set_option(tqd.OPT_TILE_QUBITS, 9)
        st.apply_circuit(gates)
        amp = st.amplitudes()
        zz = st.expval([(0, 1 | (1 << (n - 1)), 1.0), (0, 1, 1.0)])
        st.free()
        return amp, zz
    for amp, zz in run_world(tqd, world, fn):
        ref = orc.run(n, gates)
        assert np.max(np.abs(amp - ref)) < 1e-12
        assert abs(amp[0] - 2 ** -0.5) < 1e-12 and abs(amp[-1] - 2 ** -0.5) < 1e-12
        assert abs(zz[0] - 1.0) < 1e-12 and abs(zz[1]) < 1e-12


def test_world_matches_single_rank(tqd, orc):
    """World 1 vs 2 vs 4 vs 8 give the same gradients (SPEC-style sharding invariance)."""
    n = 13
    gates = W.hea(n, 4, 11, small=True)
    terms = W.sum_z(n)
    vals = {}
    for world in (1, 2, 4, 8):
        def fn(r, ctx):
            st = tqd.State(ctx, n, "c128")
            st.set_option(tqd.OPT_TILE_QUBITS, 9)
            st.apply_circuit(gates)
            v = st.adjoint_grad(terms)
            st.free()
            return v
        if world == 1:
            ctx = tqd.Context(1, 0, 0)
            vals[world] = fn(0, ctx)
            ctx.close()
        else:
            vals[world] = run_world(tqd, world, fn)[0]
    for world in (2, 4, 8):
        assert abs(vals[world][0] - vals[1][0]) < 1e-11
        assert np.max(np.abs(vals[world][1] - vals[1][1])) < 1e-11


def test_world_fused_remap_repeat(tqd, orc):
    """Fused remaps swap the roles of the shard buffers; rewinding and re-running the
    cached plan (twice), then reading amplitudes, must still match the oracle."""
    n, world = 14, 4
    gates = W.hea(n, 3, 9, small=True)
    terms = W.sum_z(n)

    def fn(r, ctx):
        st = tqd.State(ctx, n, "c128")
        st.set_option(tqd.OPT_TILE_QUBITS, 9)
        st.apply_circuit(gates)
        out = [st.adjoint_grad(terms)]
        for _ in range(2):
            st.rewind()
            out.append(st.adjoint_grad(terms))
        st.reset()
        st.apply_circuit(gates)
        amp = st.amplitudes()
        m = st.metrics()
        st.free()
        return out, amp, m
    rval, rgrad = orc.adjoint(n, gates, terms)
    ref = orc.run(n, gates)
    for out, amp, m in run_world(tqd, world, fn):
        for val, grad in out:
            assert abs(val - rval) < 1e-10 and np.max(np.abs(grad - rgrad)) < 1e-10
        assert np.max(np.abs(amp - ref)) < 1e-12
        assert m["remaps"] > 0


@pytest.mark.parametrize("fused", [1, 0])
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("world,n", [(2, 12), (4, 13), (8, 14)])
def test_world_bounded_staging(tqd, orc, world, n, dtype, fused):
    """Remaps and X / Y partner exchanges through a staging buffer forced to 2 KiB
    (TQD_OPT_STAGING_BYTES), so every block moves in many chunks: amplitudes,
    Pauli expectation values (X / Y on rank bits) and adjoint gradients (psi and
    lambda remapped) against the oracle (SURVEY.md §8(e) bounded exchange)."""
    gates = mixed_circuit(n, 5 * world + n)
    terms = W.random_z_terms(n, 4, world) + [(1, 0, 0.7), (3, 4, -1.1), (2, 1 | (1 << (n - 1)), 0.3)]

    def fn(r, ctx):
        st = tqd.State(ctx, n, dtype)
        st.set_option(tqd.OPT_TILE_QUBITS, 9)
        st.set_option(tqd.OPT_SMALL_MAX, 0)
        st.set_option(tqd.OPT_FUSED_REMAP, fused)
        st.set_option(tqd.OPT_STAGING_BYTES, 2048)
        st.apply_circuit(gates)
        amp = st.amplitudes()
        ev = st.expval(terms)
        st.reset()
        st.apply_circuit(gates)
        val, grad = st.adjoint_grad(terms)
        m = st.metrics()
        st.free()
        return amp, ev, val, grad, m
    ref = orc.run(n, gates)
    rev = orc.expval(ref, n, terms)
    rval, rgrad = orc.adjoint(n, gates, terms)
    for amp, ev, val, grad, m in run_world(tqd, world, fn):
        assert np.max(np.abs(amp - ref)) < TOL[dtype]["amp"]
        assert np.max(np.abs(ev - rev)) < TOL[dtype]["val"]
        assert abs(val - rval) < TOL[dtype]["val"]
        assert np.max(np.abs(grad - rgrad)) < TOL[dtype]["val"]
        assert m["remaps"] > 0 and m["a2a_bytes"] > 0
        # no shard-sized staging: psi + lambda + 2 KiB (+ the fused-forward lambda)
        assert m["peak_device_bytes"] <= 2 * (1 << (n - (world.bit_length() - 1))) * (16 if dtype == "c128" else 8) + 2048


def test_world_unfused_remap_then_fused_race(tqd, orc, monkeypatch):
    """a plan [remap (unfused: nothing before it), sweep, sweep +
    fused remap, ...] with odd ranks held back (device sleep) between receiving and
    unpacking each remap chunk.  Round 1 staged both through the same receive
    buffer, so a fast rank's fused stores could overwrite a slow rank's received
    block before it was unpacked; now unfused remaps use rank-local staging and
    fused stores go to the owners' idle lambda buffers."""
    n, world = 12, 4
    gates = [W.Gate("RX", (0,), (0.3,)), W.Gate("RX", (1,), (0.4,))]
    gates += [W.Gate("CNOT", (q, q + 1)) for q in range(n - 1)] + W.hea(n, 2, 1, small=True)
    kinds = [s["type"] for s in tqd.tqd_debug_plan(n, gates, world=world, k=9, small_max=0)["stages"]]
    assert kinds[0] == "remap" and any(a == "sweep" and b == "remap" for a, b in zip(kinds, kinds[1:])), kinds
    monkeypatch.setenv("TQD_DEBUG_REMAP_DELAY_US", "20000")
    terms = W.sum_z(n) + [(0, 3, 0.5)]

    def fn(r, ctx):
        st = tqd.State(ctx, n, "c128")
        st.set_option(tqd.OPT_TILE_QUBITS, 9)
        st.set_option(tqd.OPT_SMALL_MAX, 0)
        st.set_option(tqd.OPT_STAGING_BYTES, 4096)
        st.apply_circuit(gates)
        out = [st.adjoint_grad(terms)]
        st.rewind()  # the shared peer tables exist now: the race window is open from the first stage
        out.append(st.adjoint_grad(terms))
        st.reset()
        st.apply_circuit(gates)
        amp = st.amplitudes()
        m = st.metrics()
        st.free()
        return out, amp, m
    rval, rgrad = orc.adjoint(n, gates, terms)
    ref = orc.run(n, gates)
    for out, amp, m in run_world(tqd, world, fn):
        for val, grad in out:
            assert abs(val - rval) < 1e-10 and np.max(np.abs(grad - rgrad)) < 1e-10
        assert np.max(np.abs(amp - ref)) < 1e-12
        assert m["fused_remaps"] > 0 and m["remaps"] > m["fused_remaps"]


@pytest.mark.parametrize("fused", [1, 0])
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("world,n", [(2, 12), (4, 13), (8, 14)])
def test_world_product_prefix(tqd, orc, world, n, dtype, fused):
    """Product-state prefix with sharded qubits: each rank writes its shard of the
    product (the rank bits' factor c_r), the prefix gradients of local qubits come from
    the rank-summed environments, those of the sharded qubits from every rank's total
    contraction (small all-reduce).  Against the oracle, prefix on == off."""
    rng = np.random.default_rng(world + n)
    gates = []
    for _ in range(2):
        for q in rng.permutation(n):
            k = ["RY", "RZ", "RX", "U3", "H"][int(rng.integers(5))]
            if k == "U3":
                gates.append(W.Gate(k, (int(q),), tuple(float(v) for v in rng.uniform(0, 6.3, 3))))
            elif k == "H":
                gates.append(W.Gate(k, (int(q),)))
            else:
                gates.append(W.Gate(k, (int(q),), (float(rng.uniform(0, 6.3)),)))
    gates += W.hea(n, 2, world, small=True) + W.random_circuit(n, 40, 7 * world)
    terms = W.random_z_terms(n, 4, world) + W.sum_z(n) + [(1, 0, 0.7)]
    rval, rgrad = orc.adjoint(n, gates, terms)
    ref = orc.run(n, gates)

    def fn(r, ctx):
        out = {}
        for pf in (1, 0):
            st = tqd.State(ctx, n, dtype)
            st.set_option(tqd.OPT_TILE_QUBITS, 9)
            st.set_option(tqd.OPT_SMALL_MAX, 0)
            st.set_option(tqd.OPT_FUSED_REMAP, fused)
            st.set_option(tqd.OPT_PRODUCT_PREFIX, pf)
            st.apply_circuit(gates)
            amp = st.amplitudes()
            st.reset()
            st.apply_circuit(gates)
            val, grad = st.adjoint_grad(terms)
            st.free()
            out[pf] = (amp, val, grad)
        return out
    for out in run_world(tqd, world, fn):
        for pf in (1, 0):
            amp, val, grad = out[pf]
            assert np.max(np.abs(amp - ref)) < TOL[dtype]["amp"], pf
            assert abs(val - rval) < TOL[dtype]["val"], pf
            assert np.max(np.abs(grad - rgrad)) < TOL[dtype]["val"], pf


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("world,n", [(2, 12), (4, 13), (8, 14)])
def test_world_product_prefix_qft(tqd, orc, world, n, dtype):
    """cfg-5 family sharded: X-prep + QFT (+ SWAPs) + HEA as the product prefix with
    sharded qubits among its factors; amplitudes and gradients against the oracle."""
    wl = W.config(5, seed=world, n_override=n)
    rval, rgrad = orc.adjoint(n, wl.gates, wl.terms)
    ref = orc.run(n, wl.gates)

    def fn(r, ctx):
        st = tqd.State(ctx, n, dtype)
        st.set_option(tqd.OPT_TILE_QUBITS, 9)
        st.set_option(tqd.OPT_SMALL_MAX, 0)
        st.set_option(tqd.OPT_PRODUCT_PREFIX, 1)
        st.apply_circuit(wl.gates)
        amp = st.amplitudes()
        npre = st.metrics()["gates_prefix"]
        st.reset()
        st.apply_circuit(wl.gates)
        val, grad = st.adjoint_grad(wl.terms)
        st.free()
        return amp, val, grad, npre
    for amp, val, grad, npre in run_world(tqd, world, fn):
        assert npre == sum(1 for g in wl.gates if g.name in ("X", "H", "SWAP", "MAT2")) + 2 * n
        assert np.max(np.abs(amp - ref)) < TOL[dtype]["amp"]
        assert abs(val - rval) < TOL[dtype]["val"]
        assert np.max(np.abs(grad - rgrad)) < TOL[dtype]["val"]


@pytest.mark.parametrize("fused", [1, 0])
@pytest.mark.parametrize("world,n_loc", [(2, 21), (4, 21), (8, 20)])
def test_world_clifford_large(tqd, orc, world, n_loc, fused):
    """Sharded HEA at Clifford angles with local shards large enough that every CTA
    walks many tiles (2^20-2^21 amplitudes per rank, 23-24 qubits in all), remaps fused
    and staged, against the stabilizer-tableau oracle: every expectation and gradient."""
    from test_gpu_clifford_fullsize import quarter_hea, sensitive_terms
    g = world.bit_length() - 1
    n = n_loc + g
    gates = quarter_hea(n, 6, world + n_loc)
    terms = sensitive_terms(n, gates, 10, world)
    rev = orc.clifford_expval(n, gates, terms)
    rval, rgrad = orc.clifford_grad(n, gates, terms)
    assert np.count_nonzero(rgrad) >= 6

    def fn(r, ctx):
        st = tqd.State(ctx, n, "c64")
        st.set_option(tqd.OPT_FUSED_REMAP, fused)
        st.apply_circuit(gates)
        ev = st.expval(terms)
        st.rewind()
        val, grad = st.adjoint_grad(terms)
        m = st.metrics()
        st.free()
        return ev, val, grad, m
    for ev, val, grad, m in run_world(tqd, world, fn):
        assert m["remaps"] > 0
        assert np.max(np.abs(ev - rev)) < TOL["c64"]["val"]
        assert abs(val - rval) < TOL["c64"]["val"]
        assert np.max(np.abs(grad - rgrad)) < TOL["c64"]["val"]
