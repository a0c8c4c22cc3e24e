"""GPU parity of tqd_adjoint_grad / tqd_expval with observable absorption (TQD_OPT_ABSORB_TAIL):
the trailing diagonal / permutation gates are folded into the Z-string
observable instead of being applied and un-applied.  Every value and gradient is
compared with the float64 oracle applying EVERY gate (tolerances as in
test_gpu_parity.py), with absorption on and off, single GPU and emulated world."""
import numpy as np
import pytest

import workloads as W
from test_gpu_emulated_world import run_world

pytestmark = pytest.mark.gpu

TOL = {"c64": 1e-4, "c128": 1e-10}


@pytest.fixture(scope="module")
def tqd():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need CUDA (run with -m 'not gpu' on CPU)")
    import paper_2511_19291_b200 as t
    return t


@pytest.fixture(scope="module")
def ctx(tqd):
    c = tqd.Context(1, 0, 0)
    yield c
    c.close()


def _run(tqd, ctx, n, gates, terms, dtype, absorb, small_max=None, k=None):
    st = tqd.State(ctx, n, dtype)
    st.set_option(tqd.OPT_ABSORB_TAIL, absorb)
    if small_max is not None:
        st.set_option(tqd.OPT_SMALL_MAX, small_max)
    if k is not None:
        st.set_option(tqd.OPT_TILE_QUBITS, k)
    st.apply_circuit(gates)
    val, grad = st.adjoint_grad(terms)
    m = st.metrics()
    st.free()
    return val, grad, m


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n,small_max,k", [(6, 10, None), (13, 0, 10), (16, 0, 12)])
def test_absorbed_tail_parity(tqd, ctx, orc, n, small_max, k, dtype):
    for seed in range(2):
        prefix = W.random_circuit(n, 60, 300 + seed, small=True) + W.hea(n, 2, seed, small=True)
        gates = prefix + W.diag_perm_tail(n, 40, 400 + seed)
        terms = W.random_z_terms(n, 5, seed) + [(0, 1 << (n - 1), 0.5)]
        rval, rgrad = orc.adjoint(n, gates, terms)
        for absorb in (1, 0):
            val, grad, m = _run(tqd, ctx, n, gates, terms, dtype, absorb, small_max, k)
            assert abs(val - rval) < TOL[dtype], (absorb, val, rval)
            assert np.max(np.abs(grad - rgrad)) < TOL[dtype], absorb
            if absorb:
                assert m["gates_absorbed"] >= 40
            else:
                assert m["gates_absorbed"] == 0


def test_hea_absorption_saves_sweeps(tqd, ctx, orc):
    """cfg-3 family at 18 qubits: the last RZ layer + ring CNOTs (2n gates) are
    absorbed; fewer forward and adjoint sweeps, same value and gradients."""
    n = 18
    gates = W.hea(n, 8, seed=2, small=True)
    terms = W.sum_z(n)
    rval, rgrad = orc.adjoint(n, gates, terms)
    res = {}
    for absorb in (1, 0):
        val, grad, m = _run(tqd, ctx, n, gates, terms, "c64", absorb, small_max=0)
        assert abs(val - rval) < 1e-4 and np.max(np.abs(grad - rgrad)) < 1e-4
        res[absorb] = m
    assert res[1]["gates_absorbed"] == 2 * n
    assert res[1]["fwd_sweeps"] < res[0]["fwd_sweeps"]
    assert res[1]["bwd_sweeps"] <= res[0]["bwd_sweeps"]


def test_plan_cache_with_and_without_absorption(tqd, ctx, orc):
    """expval caches the full plan, adjoint_grad the absorbed one: replays
    (tqd_state_rewind) and re-recordings must never mix them up."""
    n = 14
    gates = W.hea(n, 4, seed=5, small=True) + W.diag_perm_tail(n, 12, 9)
    terms = W.sum_z(n) + [(0, 3, -0.5)]
    rval, rgrad = orc.adjoint(n, gates, terms)
    rexp = orc.expval(orc.run(n, gates), n, terms)
    ramp = orc.run(n, gates)
    st = tqd.State(ctx, n, "c64")
    st.set_option(tqd.OPT_SMALL_MAX, 0)
    try:
        st.apply_circuit(gates)
        for it in range(3):
            e = st.expval(terms)
            assert np.max(np.abs(e - rexp)) < 1e-4, it
            st.rewind()
            val, grad = st.adjoint_grad(terms)
            assert abs(val - rval) < 1e-4 and np.max(np.abs(grad - rgrad)) < 1e-4, it
            st.rewind()
            assert np.max(np.abs(st.amplitudes() - ramp)) < 1e-5, it
            st.rewind()
            val, grad = st.adjoint_grad(terms)
            assert abs(val - rval) < 1e-4 and np.max(np.abs(grad - rgrad)) < 1e-4, it
            st.reset()
            st.apply_circuit(gates)
    finally:
        st.free()


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("world,n,k", [(2, 12, 9), (4, 14, 10), (8, 15, 9)])
def test_world_absorbed_tail(tqd, orc, world, n, k, dtype):
    """Tail CNOT / SWAP / X on global (rank) qubits: the conjugated Z strings
    carry rank bits; every rank's value and gradients match the oracle."""
    gates = W.random_circuit(n, 50, 7 + world, small=True) + W.hea(n, 2, world, small=True)
    tail = W.diag_perm_tail(n, 30, 11 + world) + [W.Gate("CNOT", (n - 1, 0)), W.Gate("SWAP", (0, n - 2)),
                                                   W.Gate("X", (1,)), W.Gate("CNOT", (2, 0))]
    gates = gates + tail
    terms = W.random_z_terms(n, 4, world) + W.sum_z(n)[:3]
    rval, rgrad = orc.adjoint(n, gates, terms)

    def fn(r, ctx):
        st = tqd.State(ctx, n, dtype)
        st.set_option(tqd.OPT_TILE_QUBITS, k)
        st.set_option(tqd.OPT_SMALL_MAX, 0)
        st.apply_circuit(gates)
        val, grad = st.adjoint_grad(terms)
        m = st.metrics()
        st.free()
        return val, grad, m

    for val, grad, m in run_world(tqd, world, fn):
        assert abs(val - rval) < TOL[dtype]
        assert np.max(np.abs(grad - rgrad)) < TOL[dtype]
        assert m["gates_absorbed"] >= len(tail)


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n,small_max", [(6, 10), (14, 0)])
def test_expval_absorbed_tail_stays_pending(tqd, ctx, orc, n, small_max, dtype):
    """tqd_expval with Z strings absorbs the tail and leaves it pending: the next
    X/Y expval, readback or adjoint applies it; every result against the oracle."""
    tol = TOL[dtype]
    gates = W.random_circuit(n, 50, 77, small=True) + W.diag_perm_tail(n, 30, 78)
    zt = W.random_z_terms(n, 5, 1) + W.sum_z(n)
    xt = W.random_pauli_terms(n, 6, 2)
    psi = orc.run(n, gates)
    r_z, r_x = orc.expval(psi, n, zt), orc.expval(psi, n, xt)
    rval, rgrad = orc.adjoint(n, gates, zt)
    amp_tol = 1e-5 if dtype == "c64" else 1e-12

    def fresh():
        st = tqd.State(ctx, n, dtype)
        st.set_option(tqd.OPT_SMALL_MAX, small_max)
        st.apply_circuit(gates)
        return st

    st = fresh()
    try:
        assert np.max(np.abs(st.expval(zt) - r_z)) < tol
        assert st.metrics()["gates_absorbed"] >= 30
        assert np.max(np.abs(st.expval(zt) - r_z)) < tol          # again, still pending
        assert np.max(np.abs(st.expval(xt) - r_x)) < tol          # X/Y: the tail is applied now
        assert np.max(np.abs(st.amplitudes() - psi)) < amp_tol
        assert np.max(np.abs(st.expval(zt) - r_z)) < tol
    finally:
        st.free()
    st = fresh()
    try:
        assert np.max(np.abs(st.expval(zt) - r_z)) < tol
        assert np.max(np.abs(st.amplitudes() - psi)) < amp_tol  # readback applies the tail
    finally:
        st.free()
    st = fresh()
    try:
        assert np.max(np.abs(st.expval(zt) - r_z)) < tol
        val, grad = st.adjoint_grad(zt)                           # adjoint after a pending tail
        assert abs(val - rval) < tol and np.max(np.abs(grad - rgrad)) < tol
    finally:
        st.free()
