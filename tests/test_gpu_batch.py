"""Batched states through the C ABI (tqd_state_init_batch / tqd_apply_gate_batch):
B states share one tape; encoder rotations carry per-state parameters (the
paper's profiled workload: a batch of 16 with Adam on the circuit inputs,
PAPER.md:254, 157).  Every batch element is checked against an independent
float64 oracle run of its own circuit.

Slot layout: a batched gate with np parameters owns batch * np slots in
recording order (element b at slot0 + b * np + i); a shared trainable gate owns
np slots and receives the gradient summed over the batch.
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


@pytest.fixture(scope="module")
def ctx(tqd):
    c = tqd.Context(1, 0, 0)
    yield c
    c.close()


def encoder_inputs(B, n, seed, kind="RY"):
    rng = np.random.default_rng(seed)
    npar = 3 if kind == "U3" else 1
    return rng.uniform(0, np.pi / 3, size=(n, B, npar))  # [qubit][batch][param] (PAPER.md:353 range)


def per_element_gates(x, b, ansatz, kind="RY", enc_trainable=True):
    n = x.shape[0]
    enc = [W.Gate(kind, (q,), tuple(float(v) for v in x[q, b]), None, enc_trainable) for q in range(n)]
    return enc + ansatz


def record_batch(st, x, ansatz, kind="RY", enc_trainable=True):
    for q in range(x.shape[0]):
        st.apply_batch(kind, [q], x[q], trainable=enc_trainable)
    st.apply_circuit(ansatz)


def expected(orc, n, x, ansatz, terms, coeff, kind="RY", enc_trainable=True):
    """(value, grad) of the batched run from per-element oracle adjoints."""
    B, npar = x.shape[1], x.shape[2]
    n_enc = n * npar if enc_trainable else 0
    val, enc, shared = 0.0, np.zeros((n, B, npar)), None
    for b in range(B):
        tb = [(t[0], t[1], float(coeff[b, i])) for i, t in enumerate(terms)]
        v, g = orc.adjoint(n, per_element_gates(x, b, ansatz, kind, enc_trainable), tb)
        val += v
        if enc_trainable:
            enc[:, b, :] = g[:n_enc].reshape(n, npar)
        shared = g[n_enc:] if shared is None else shared + g[n_enc:]
    grad = np.concatenate([enc.reshape(-1) if enc_trainable else np.zeros(0), shared])
    return val, grad


def make(tqd, ctx, n, dtype, B, k=None, small_max=None):
    st = tqd.State(ctx, n, dtype, batch=B)
    if k is not None:
        st.set_option(tqd.OPT_TILE_QUBITS, k)
    if small_max is not None:
        st.set_option(tqd.OPT_SMALL_MAX, small_max)
    return st


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n,B,k,small_max", [(6, 3, None, None), (9, 4, None, None), (12, 3, 10, 0), (14, 5, 12, 0)])
def test_batch_amplitudes_and_expval(tqd, ctx, orc, n, B, k, small_max, dtype):
    x = encoder_inputs(B, n, n + B)
    ansatz = W.hea(n, 2, seed=n) + W.random_circuit(n, 40, n + 1)
    terms = W.random_pauli_terms(n, 6, n) + W.sum_z(n)
    st = make(tqd, ctx, n, dtype, B, k, small_max)
    record_batch(st, x, ansatz)
    amp = st.amplitudes()
    ev = st.expval(terms)
    st.free()
    assert amp.shape == (B << n,) and ev.shape == (B, len(terms))
    for b in range(B):
        gates = per_element_gates(x, b, ansatz)
        psi = orc.run(n, gates)
        assert np.max(np.abs(amp[b << n:(b + 1) << n] - psi)) < TOL[dtype]["amp"], b
        assert np.max(np.abs(ev[b] - orc.expval(psi, n, terms))) < TOL[dtype]["val"], b


@pytest.mark.parametrize("kind", ["RY", "U3", "RZ"])
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n,B,k,small_max", [(7, 3, None, None), (13, 4, 10, 0), (15, 3, 12, 0)])
def test_batch_adjoint_input_gradients(tqd, ctx, orc, n, B, k, small_max, dtype, kind):
    """Input (encoder) gradients per batch element + ansatz gradients summed over the batch."""
    x = encoder_inputs(B, n, 3 * n + B, kind)
    ansatz = W.hea(n, 3, seed=B, small=True)
    terms = W.random_z_terms(n, 3, n) + W.sum_z(n) + [(1, 2, 0.4)]
    rng = np.random.default_rng(n)
    coeff = rng.standard_normal((B, len(terms)))
    st = make(tqd, ctx, n, dtype, B, k, small_max)
    record_batch(st, x, ansatz, kind)
    assert st.n_params == B * n * x.shape[2] + 2 * n * 3
    val, grad = st.adjoint_grad(terms, coeff=coeff)
    st.free()
    rval, rgrad = expected(orc, n, x, ansatz, terms, coeff, kind)
    assert abs(val - rval) < TOL[dtype]["val"]
    assert grad.shape == rgrad.shape
    assert np.max(np.abs(grad - rgrad)) < TOL[dtype]["val"]


def test_batch_shared_coefficients_and_frozen_inputs(tqd, ctx, orc):
    """coeff = None: the terms' own coefficients for every element; non-trainable inputs."""
    n, B = 12, 4
    x = encoder_inputs(B, n, 7)
    ansatz = W.hea(n, 2, seed=2, small=True)
    terms = W.sum_z(n)
    st = make(tqd, ctx, n, "c128", B, 9, 0)
    record_batch(st, x, ansatz, enc_trainable=False)
    assert st.n_params == 2 * n * 2
    val, grad = st.adjoint_grad(terms)
    st.free()
    rval, rgrad = expected(orc, n, x, ansatz, terms, np.ones((B, len(terms))), enc_trainable=False)
    assert abs(val - rval) < 1e-10 and np.max(np.abs(grad - rgrad)) < 1e-10


def test_batch_matches_single_states(tqd, ctx, orc):
    """A batch of B equals B single-state runs (same kernels, same plan)."""
    n, B = 13, 3
    x = encoder_inputs(B, n, 11)
    ansatz = W.hea(n, 2, seed=4, small=True)
    terms = W.sum_z(n)
    st = make(tqd, ctx, n, "c128", B, 10, 0)
    record_batch(st, x, ansatz)
    val, grad = st.adjoint_grad(terms)
    st.free()
    tot, shared = 0.0, 0.0
    enc = np.zeros((n, B))
    for b in range(B):
        s1 = make(tqd, ctx, n, "c128", 1, 10, 0)
        s1.apply_circuit(per_element_gates(x, b, ansatz))
        v, g = s1.adjoint_grad(terms)
        s1.free()
        tot += v
        enc[:, b] = g[:n]
        shared = shared + g[n:]
    assert abs(val - tot) < 1e-11
    assert np.max(np.abs(grad - np.concatenate([enc.reshape(-1), shared]))) < 1e-11


def test_batch_abi_errors(tqd, ctx):
    st = make(tqd, ctx, 5, "c64", 2)
    with pytest.raises(tqd.TqdError) as e:
        st.apply_batch("H", [0], np.zeros((2, 0)))
    assert e.value.code == -1
    with pytest.raises(tqd.TqdError) as e:
        tqd.tqd_apply_gate_batch(st.handle, "RY", [0, 1], np.zeros((2, 1)))
    assert e.value.code == -1
    st.free()
    with pytest.raises(tqd.TqdError) as e:
        tqd.tqd_state_init_batch(ctx.handle, 5, tqd.C64, 0)
    assert e.value.code == -1


@pytest.mark.parametrize("fused", [1, 0])
@pytest.mark.parametrize("world", [2, 4])
def test_batch_emulated_world(tqd, orc, world, fused):
    """Batched states sharded over an emulated world (remaps of every element's shard)."""
    n, B = 13, 3
    x = encoder_inputs(B, n, world)
    ansatz = W.hea(n, 2, seed=world, small=True)
    terms = W.sum_z(n) + [(1, 0, 0.5)]
    lid = tqd.tqd_loopback_id()
    res, err = [None] * world, [None] * world

    def worker(r):
        try:
            ctx = tqd.Context(world, r, 0, lid)
            try:
                st = tqd.State(ctx, n, "c128", batch=B)
                st.set_option(tqd.OPT_TILE_QUBITS, 9)
                st.set_option(tqd.OPT_SMALL_MAX, 0)
                st.set_option(tqd.OPT_FUSED_REMAP, fused)
                record_batch(st, x, ansatz)
                amp = st.amplitudes()
                ev = st.expval(terms)
                vg = st.adjoint_grad(terms)
                m = st.metrics()
                st.free()
                res[r] = (amp, ev, vg, m)
            finally:
                ctx.close()
        except Exception:
            err[r] = traceback.format_exc()

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    assert not any(t.is_alive() for t in th)
    assert not any(err), "\n".join(e for e in err if e)
    rval, rgrad = expected(orc, n, x, ansatz, terms, np.tile([t[2] for t in terms], (B, 1)))
    for amp, ev, (val, grad), m in res:
        assert m["remaps"] > 0
        for b in range(B):
            psi = orc.run(n, per_element_gates(x, b, ansatz))
            assert np.max(np.abs(amp[b << n:(b + 1) << n] - psi)) < 1e-12
            assert np.max(np.abs(ev[b] - orc.expval(psi, n, terms))) < 1e-10
        assert abs(val - rval) < 1e-10 and np.max(np.abs(grad - rgrad)) < 1e-10


def test_batch_training_loop_reuses_plan(tqd, ctx, orc):
    """Adam-on-inputs style loop: new encoder inputs every step, same structure."""
    n, B = 12, 4
    ansatz = W.hea(n, 2, seed=3, small=True)
    terms = W.sum_z(n)
    st = make(tqd, ctx, n, "c128", B, 10, 0)
    for step in range(3):
        x = encoder_inputs(B, n, 50 + step)
        st.reset()
        record_batch(st, x, ansatz)
        val, grad = st.adjoint_grad(terms)
        rval, rgrad = expected(orc, n, x, ansatz, terms, np.ones((B, len(terms))))
        assert abs(val - rval) < 1e-10 and np.max(np.abs(grad - rgrad)) < 1e-10
    assert st.metrics()["plans_reused"] == 2
    st.free()


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_batch_diagonal_runs_with_zero_inputs(tqd, ctx, orc, dtype):
    """Batched RZ encoder inputs that are exactly 0 for some elements, placed after
    dense gates (so they land on lane / warp / base bits) and between controlled-phase
    runs: the kernel-op structure must not depend on the per-element values."""
    n, B = 14, 3
    x = encoder_inputs(B, n, 5, "RZ")
    x[:, 1, :] = 0.0
    x[::3, 2, :] = 0.0
    pre = [W.Gate("H", (q,)) for q in range(n)] + W.qft(n, swaps=False)[:40]
    post = W.qft(n, swaps=False)[40:90] + W.hea(n, 1, seed=2, small=True)
    terms = W.sum_z(n) + W.random_z_terms(n, 3, 4)
    st = make(tqd, ctx, n, dtype, B, 12, 0)
    st.apply_circuit(pre)
    for q in range(n):
        st.apply_batch("RZ", [q], x[q], trainable=True)
    st.apply_circuit(post)
    amp = st.amplitudes()
    st.free()
    for b in range(B):
        enc = [W.Gate("RZ", (q,), (float(x[q, b, 0]),), None, True) for q in range(n)]
        psi = orc.run(n, pre + enc + post)
        assert np.max(np.abs(amp[b << n:(b + 1) << n] - psi)) < TOL[dtype]["amp"], b


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("kind", ["RY", "U3"])
def test_batch_product_prefix(tqd, ctx, orc, dtype, kind):
    """A batch of states with per-state encoder inputs: the encoder (batched gates,
    per-element values and gradient slots), the fixed gates after it and the first
    ansatz layer form each element's product prefix.  Against the per-element oracle,
    prefix on == off, and the prefix gate count (B x per-element prefix)."""
    n, B = 12, 3
    x = encoder_inputs(B, n, 77, kind)
    ansatz = [W.Gate("H", (0,)), W.Gate("S", (1,))] + W.hea(n, 3, seed=5, small=True)
    terms = W.random_z_terms(n, 3, 4) + W.sum_z(n) + [(1, 2, 0.3)]
    coeff = np.random.default_rng(9).standard_normal((B, len(terms)))
    rval, rgrad = expected(orc, n, x, ansatz, terms, coeff, kind)
    out = {}
    for pf in (1, 0):
        st = make(tqd, ctx, n, dtype, B, small_max=0)
        st.set_option(tqd.OPT_PRODUCT_PREFIX, pf)
        record_batch(st, x, ansatz, kind)
        amp = st.amplitudes()
        m = st.metrics()
        st.reset()
        record_batch(st, x, ansatz, kind)
        val, grad = st.adjoint_grad(terms, coeff=coeff)
        st.free()
        # encoder (n) + H + S + the first RY / RZ layer (2n), per element
        assert m["gates_prefix"] == (B * (n + 2 + 2 * n) if pf else 0), m["gates_prefix"]
        for b in range(B):
            psi = orc.run(n, per_element_gates(x, b, ansatz, kind))
            assert np.max(np.abs(amp[b << n:(b + 1) << n] - psi)) < TOL[dtype]["amp"], (pf, b)
        assert abs(val - rval) < TOL[dtype]["val"], pf
        assert np.max(np.abs(grad - rgrad)) < TOL[dtype]["val"], pf
        out[pf] = grad
    assert np.max(np.abs(out[1] - out[0])) < TOL[dtype]["val"]
