"""GPU <-> oracle parity through the C ABI (needs a B200).

Tolerances (BASELINE.json north_star): expectation values and gradients within
1e-4 absolute for complex64 and 1e-10 for complex128; amplitudes within 1e-5
max-abs for complex64 (1e-12 for complex128).
"""
import math

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


def make_state(tqd, ctx, n, dtype, k=None, small_max=None, grid=None):
    st = tqd.State(ctx, n, dtype)
    if k is not None:
        st.set_option(tqd.OPT_TILE_QUBITS, k)
    if small_max is not None:
        st.set_option(tqd.OPT_SMALL_MAX, small_max)
    if grid:
        # a few persistent CTAs: every CTA walks many tiles (tile stepping, next-tile
        # prefetch, accumulators carried across tiles) as at 30 qubits
        st.set_option(tqd.OPT_GRID_CTAS, grid)
    return st


# ---------------------------------------------------------------- amplitudes
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 10])
def test_small_path_amplitudes(tqd, ctx, orc, n, dtype):
    for seed in range(3):
        gates = W.random_circuit(n, 60, seed)
        st = make_state(tqd, ctx, n, dtype)
        st.apply_circuit(gates)
        got = st.amplitudes()
        st.free()
        ref = orc.run(n, gates)
        assert np.max(np.abs(got - ref)) < TOL[dtype]["amp"], (n, seed)


GRIDS = [0, 1, 3, 7]  # 0 = auto (SMs x resident CTAs); 1 / 3 / 7: each CTA loops over many tiles


@pytest.mark.parametrize("grid", GRIDS)
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n,k", [(9, 9), (11, 10), (12, 12), (13, 11), (15, 12), (17, 12), (18, 9)])
def test_sweep_path_amplitudes(tqd, ctx, orc, n, k, dtype, grid):
    """Fused tiled sweeps (forced: small path off); several tiles and k values."""
    for seed in range(2):
        gates = W.random_circuit(n, 120, seed + 10 * n)
        st = make_state(tqd, ctx, n, dtype, k=k, small_max=0, grid=grid)
        st.apply_circuit(gates)
        got = st.amplitudes()
        m = st.metrics()
        st.free()
        assert m["fwd_sweeps"] >= 1
        ref = orc.run(n, gates)
        assert np.max(np.abs(got - ref)) < TOL[dtype]["amp"], (n, k, seed)


def test_incremental_execution(tqd, ctx, orc):
    """Gates recorded after an execution point continue from the permuted layout."""
    n = 14
    g1, g2 = W.random_circuit(n, 50, 1), W.hea(n, 2, 2)
    st = make_state(tqd, ctx, n, "c64", small_max=0)
    st.apply_circuit(g1)
    a1 = st.amplitudes()
    st.apply_circuit(g2)
    a2 = st.amplitudes()
    st.free()
    assert np.max(np.abs(a1 - orc.run(n, g1))) < 1e-5
    assert np.max(np.abs(a2 - orc.run(n, g1 + g2))) < 1e-5


def test_qft_and_ghz(tqd, ctx, orc):
    n = 16
    x = 0xBEEF
    st = make_state(tqd, ctx, n, "c128", small_max=0)
    st.apply_circuit(W.basis_prep(n, x) + W.qft(n))
    got = st.amplitudes()
    st.free()
    N = 1 << n
    ref = np.exp(2j * np.pi * x * np.arange(N) / N) / math.sqrt(N)
    assert np.max(np.abs(got - ref)) < 1e-12
    st = make_state(tqd, ctx, n, "c64", small_max=0)
    st.apply_circuit([W.Gate("H", (0,))] + [W.Gate("CNOT", (q, q + 1)) for q in range(n - 1)])
    a = st.amplitudes()
    zz = st.expval([(0, (1 << i) | (1 << j), 1.0) for i in range(0, n, 3) for j in range(i + 1, n, 4)])
    st.free()
    ref = np.zeros(N, complex)
    ref[0] = ref[-1] = 1 / math.sqrt(2)
    assert np.max(np.abs(a - ref)) < 1e-6
    assert np.allclose(zz, 1.0, atol=1e-5)


def test_amplitude_window(tqd, ctx, orc):
    n = 13
    gates = W.random_circuit(n, 80, 5)
    st = make_state(tqd, ctx, n, "c128", small_max=0)
    st.apply_circuit(gates)
    part = st.amplitudes(1000, 777)
    st.free()
    assert np.max(np.abs(part - orc.run(n, gates)[1000:1777])) < 1e-12


# ---------------------------------------------------------------- expval
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n,small_max", [(6, 10), (10, 10), (13, 0), (16, 0)])
def test_expval_pauli_strings(tqd, ctx, orc, n, small_max, dtype):
    gates = W.random_circuit(n, 100, n)
    terms = W.random_pauli_terms(n, 20, n) + W.random_z_terms(n, 20, n) + W.sum_z(n)
    st = make_state(tqd, ctx, n, dtype, small_max=small_max)
    st.apply_circuit(gates)
    got = st.expval(terms)
    st.free()
    ref = orc.expval(orc.run(n, gates), n, terms)
    assert np.max(np.abs(got - ref)) < TOL[dtype]["val"]


def test_listing1(tqd, ctx):
    """PAPER.md:291-308 Listing 1 -> [0.5, 0.5, 1, 1, 1, 1] (tests/golden)."""
    import json, os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "listing1_measure_allZ.json")))
    st = make_state(tqd, ctx, 6, "c128")
    st.apply("Z", [0])
    st.apply("RY", [0], [math.pi / 3])
    st.apply("CNOT", [0, 1])
    got = st.expval(W.sum_z(6))
    st.free()
    assert np.allclose(got, gold["expected"], atol=1e-12)


# ---------------------------------------------------------------- gradients
def _grad_check(tqd, ctx, orc, n, gates, terms, dtype, **opt):
    st = make_state(tqd, ctx, n, dtype, **opt)
    st.apply_circuit(gates)
    val, grad = st.adjoint_grad(terms)
    st.free()
    rval, rgrad = orc.adjoint(n, gates, terms)
    tol = TOL[dtype]["val"]
    assert abs(val - rval) < tol
    assert grad.shape == rgrad.shape
    err = np.max(np.abs(grad - rgrad)) if len(grad) else 0.0
    assert err < tol, (err, np.max(np.abs(rgrad)))
    return err


@pytest.mark.parametrize("grid", GRIDS)
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n,small_max,k", [(4, 10, None), (9, 10, None), (11, 0, 10), (14, 0, 12), (16, 0, 12)])
def test_adjoint_random_circuits(tqd, ctx, orc, n, small_max, k, dtype, grid):
    for seed in range(2):
        for small in (False, True):
            gates = W.random_circuit(n, 80, seed + 3 * n, small=small)
            terms = W.random_z_terms(n, 5, seed) + [(0, 1 << (n - 1), 0.5)]
            _grad_check(tqd, ctx, orc, n, gates, terms, dtype, small_max=small_max, k=k, grid=grid)


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n,small_max,k", [(5, 10, None), (12, 0, 10), (15, 0, 12)])
def test_adjoint_pauli_terms(tqd, ctx, orc, n, small_max, k, dtype):
    """X / Y / Z strings in the adjoint seed lambda = sum_t c_t P_t psi."""
    for seed in range(2):
        gates = W.random_circuit(n, 70, 40 + seed, small=True) + W.hea(n, 2, seed, small=True)
        terms = W.random_pauli_terms(n, 12, seed) + W.random_z_terms(n, 3, seed) + [(1, 2, 0.5), (3, 0, -0.25)]
        _grad_check(tqd, ctx, orc, n, gates, terms, dtype, small_max=small_max, k=k)


def test_cfg1_exact(tqd, ctx, orc):
    """BASELINE.json configs[0]: 10q HEA depth 4, <Z0> and all 80 gradients, complex128."""
    wl = W.config(1)
    assert wl.n_params == 80 and len(wl.gates) == 120
    _grad_check(tqd, ctx, orc, wl.n, wl.gates, wl.terms, "c128")


@pytest.mark.parametrize("grid", GRIDS)
@pytest.mark.parametrize("small", [False, True])
def test_hea_sweep_grads(tqd, ctx, orc, small, grid):
    n = 18
    gates = W.hea(n, 6, seed=1, small=small)
    _grad_check(tqd, ctx, orc, n, gates, W.sum_z(n), "c64", small_max=0, grid=grid)


# ---------------------------------------------------------------- oracle parity at larger sizes
ALL_KINDS = ["I", "X", "Y", "Z", "H", "S", "SDG", "T", "TDG", "CNOT", "CZ", "SWAP", "MAT1", "MAT2",
             "RX", "RY", "RZ", "U3"]


def _rel(got, ref):
    return float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300))


@pytest.mark.parametrize("small", [False, True])
def test_random_22q_all_kinds_vs_oracle(tqd, ctx, orc, small):
    """22-qubit random circuit over every gate kind (c64, bench launch configuration:
    k = 12, auto grid = 1024 tiles over 296-444 persistent CTAs, so CTAs loop over
    tiles): amplitudes element-wise (1e-5), Z-string values and every gradient
    (1e-4) against the float64 oracle; both angle distributions (R10)."""
    n = 22
    gates = W.random_circuit(n, 300, 2200 + int(small), kinds=ALL_KINDS, small=small)
    st = make_state(tqd, ctx, n, "c64")
    st.apply_circuit(gates)
    amps = st.amplitudes()
    st.free()
    ref = orc.run(n, gates)
    err = float(np.max(np.abs(amps - ref)))
    print(f"22q amplitudes: max abs {err:.2e}, rel {_rel(amps, ref):.2e}")
    assert err < 1e-5
    terms = W.random_z_terms(n, 6, 22) + W.sum_z(n)
    st = make_state(tqd, ctx, n, "c64")
    st.apply_circuit(gates)
    val, grad = st.adjoint_grad(terms)
    st.free()
    rval, rgrad = orc.adjoint(n, gates, terms)
    ge = float(np.max(np.abs(grad - rgrad)))
    print(f"22q value err {abs(val - rval):.2e}; {len(grad)} gradients: max abs {ge:.2e}, rel {_rel(grad, rgrad):.2e}")
    assert abs(val - rval) < 1e-4 and ge < 1e-4


@pytest.mark.parametrize("small", [False, True])
def test_cfg2_24q_hea_vs_oracle(tqd, ctx, orc, small):
    """BASELINE.json configs[1] (SURVEY.md:315): 24-qubit HEA depth 20, complex64,
    forward + adjoint gradient of sum <Z_i>: the value and all 960 gradients
    element-wise against the float64 oracle (1e-4), both angle distributions."""
    n, depth = 24, 20
    gates = W.hea(n, depth, seed=24, small=small)
    st = make_state(tqd, ctx, n, "c64")
    st.apply_circuit(gates)
    val, grad = st.adjoint_grad(W.sum_z(n))
    st.free()
    assert len(grad) == 2 * n * depth
    rval, rgrad = orc.adjoint(n, gates, W.sum_z(n))
    ge = float(np.max(np.abs(grad - rgrad)))
    print(f"cfg2 value err {abs(val - rval):.2e}; 960 gradients: max abs {ge:.2e}, rel {_rel(grad, rgrad):.2e}")
    assert abs(val - rval) < 1e-4 and ge < 1e-4


def test_listing2_vjp(tqd, ctx, orc):
    """encoder RY + 3 x (CX ring, RY layer); loss = sum |<Z_i>|:
    dL/dtheta is one adjoint pass with coefficients sign(<Z_i>) (A22)."""
    n = 12
    rng = np.random.default_rng(0)
    x = rng.uniform(0, math.pi / 3, n)
    gates = [W.Gate("RY", (i,), (float(x[i]),)) for i in range(n)]
    for _ in range(3):
        gates += [W.Gate("CNOT", (i, (i + 1) % n), (), None, False) for i in range(n)]
        gates += [W.Gate("RY", (i,), (float(rng.uniform(0, 2 * math.pi)),)) for i in range(n)]
    st = make_state(tqd, ctx, n, "c64", small_max=0)
    st.apply_circuit(gates)
    ez = st.expval(W.sum_z(n))
    st.free()
    terms = [(0, 1 << q, float(np.sign(ez[q]))) for q in range(n)]
    _grad_check(tqd, ctx, orc, n, gates, terms, "c64", small_max=0)


def test_nontrainable_and_u3(tqd, ctx, orc):
    n = 13
    gates = W.random_circuit(n, 60, 9, kinds=["U3", "RX", "RY", "RZ", "CNOT", "CZ", "H"])
    for g in gates[::3]:
        g.trainable = False
    _grad_check(tqd, ctx, orc, n, gates, W.sum_z(n), "c128", small_max=0)
    _grad_check(tqd, ctx, orc, n, gates, W.sum_z(n), "c128")


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_degenerate_trainable_angles(tqd, ctx, orc, dtype):
    """Trainable gates whose matrix at these angles has another type than their
    generator: U3(0, phi, lam) is diagonal, RX(0) = RY(0) = I are real, RZ(0) = I.
    The gradients must still use each gate's own generator (not the layer type's)."""
    n = 13
    base = W.hea(n, 2, seed=5)
    gates = []
    for i, g in enumerate(base):
        gates.append(g)
        if i % 4 == 0:
            w = g.wires[:1]
            gates.append(W.Gate("U3", w, (0.0, 0.3 + 0.1 * i, -0.2), None, True))
            gates.append(W.Gate("RX", w, (0.0,), None, True))
            gates.append(W.Gate("RZ", w, (0.0,), None, True))
            gates.append(W.Gate("RY", w, (0.0,), None, True))
    terms = W.random_z_terms(n, 4, 1) + W.sum_z(n)
    _grad_check(tqd, ctx, orc, n, gates, terms, dtype, small_max=0)


# ---------------------------------------------------------------- full-size properties
def test_cfg3_entangler_free_factorization(tqd, ctx, orc):
    """30q depth-20 RY/RZ ansatz (cfg 3 shape, same launch configuration as bench.py,
    no CNOTs): E(sum Z_i) and every gradient factor into 1-qubit oracle runs (exact pin)."""
    n, depth = 30, 20
    gates = [g for g in W.hea(n, depth, seed=0, small=True) if g.name != "CNOT"]
    st = make_state(tqd, ctx, n, "c64")
    st.apply_circuit(gates)
    val, grad = st.adjoint_grad(W.sum_z(n))
    st.free()
    ref_val, ref_grad = 0.0, np.zeros(len(grad))
    idx = {id(g): i for i, g in enumerate(gates)}
    for q in range(n):
        sub = [g for g in gates if g.wires[0] == q]
        v, g1 = orc.adjoint(1, [W.Gate(g.name, (0,), g.params) for g in sub], [(0, 1, 1.0)])
        ref_val += v
        for g, d in zip(sub, g1):
            ref_grad[idx[id(g)]] = d
    assert abs(val - ref_val) < 1e-4
    assert np.max(np.abs(grad - ref_grad)) < 1e-4


def test_cfg3_mirror_circuit(tqd, ctx):
    """U then U^dag at 30 qubits returns |0..0>: <Z_i> = 1 and psi_0 = 1."""
    n = 30
    gates = W.hea(n, 6, seed=4)
    inv = []
    for g in reversed(gates):
        if g.name in ("RY", "RZ"):
            inv.append(W.Gate(g.name, g.wires, (-g.params[0],)))
        else:
            inv.append(g)
    st = make_state(tqd, ctx, n, "c64")
    st.apply_circuit(gates + inv)
    ez = st.expval(W.sum_z(n))
    a0 = st.amplitudes(0, 4)
    st.free()
    assert np.allclose(ez, 1.0, atol=1e-4)
    assert abs(a0[0] - 1) < 1e-4 and np.max(np.abs(a0[1:])) < 1e-4


def test_cfg3_parameter_shift_spot(tqd, ctx):
    """Full cfg-3 circuit: adjoint gradients vs parameter shift (two GPU forwards each)."""
    n = 30
    gates = W.hea(n, 20, seed=0, small=True)
    st = make_state(tqd, ctx, n, "c64")
    st.apply_circuit(gates)
    val, grad = st.adjoint_grad(W.sum_z(n))
    st.free()
    par = [i for i, g in enumerate(gates) if g.name in W.PARAMETRIC]
    for pi in (0, 611, 1199):
        gi = par[pi]
        es = []
        for sgn in (+1, -1):
            gg = list(gates)
            g = gg[gi]
            gg[gi] = W.Gate(g.name, g.wires, (g.params[0] + sgn * math.pi / 2,))
            st = make_state(tqd, ctx, n, "c64")
            st.apply_circuit(gg)
            es.append(st.expval(W.sum_z(n)).sum())
            st.free()
        assert abs((es[0] - es[1]) / 2 - grad[pi]) < 1e-4


def test_cfg5_shard_qft_closed_form(tqd, ctx):
    """The 2^33-amplitude shard each GPU holds at cfg 5 (36q / 8 GPUs), run as one
    33-qubit state in bench_configs' launch configuration: X-prep |x> + QFT (diagonal-
    block runs of 528 controlled phases, SWAP relabels).  Sampled amplitudes against
    the closed form omega^{xy} / sqrt(N) (ledger #13) and <Z_i> = 0."""
    n = 33
    N = 1 << n
    x = 0x1_2345_6789 % N
    st = make_state(tqd, ctx, n, "c64")
    try:
        st.apply_circuit(W.basis_prep(n, x) + W.qft(n))
        ez = st.expval(W.sum_z(n))
        for first in (0, (1 << 32) + 12345, N - 64):
            got = st.amplitudes(first, 64)
            y = np.arange(first, first + 64, dtype=np.float64)
            # omega^{xy} with the phase reduced exactly: (x * y) mod N in integers
            ph = np.array([(x * int(v)) % N for v in y], dtype=np.float64) / N
            ref = np.exp(2j * np.pi * ph) / math.sqrt(N)
            # relative to |amplitude| = N^-1/2 (an absolute 1e-5 would be vacuous at 33 qubits)
            assert np.max(np.abs(got - ref)) < 1e-4 / math.sqrt(N), first
    finally:
        st.free()
    assert np.max(np.abs(ez)) < 1e-4


def test_cfg4_entangler_free_33q(tqd, ctx, orc):
    """cfg-4 size at P = 1 (33 qubits, 64 GiB psi + 64 GiB lambda on one B200): RY/RZ
    ansatz depth 10 without CNOTs; E(sum Z_i) and all 660 gradients factor into
    1-qubit oracle runs (exact pin at full size)."""
    n, depth = 33, 10
    gates = [g for g in W.hea(n, depth, seed=3, small=True) if g.name != "CNOT"]
    st = make_state(tqd, ctx, n, "c64")
    try:
        st.apply_circuit(gates)
        val, grad = st.adjoint_grad(W.sum_z(n))
    finally:
        st.free()
    ref_val, ref_grad = 0.0, np.zeros(len(grad))
    idx = {id(g): i for i, g in enumerate(gates)}
    for q in range(n):
        sub = [g for g in gates if g.wires[0] == q]
        v, g1 = orc.adjoint(1, [W.Gate(g.name, (0,), g.params) for g in sub], [(0, 1, 1.0)])
        ref_val += v
        for g, d in zip(sub, g1):
            ref_grad[idx[id(g)]] = d
    assert len(grad) == 2 * n * depth
    assert abs(val - ref_val) < 1e-4
    assert np.max(np.abs(grad - ref_grad)) < 1e-4


# ---------------------------------------------------------------- ABI errors
def test_abi_errors(tqd, ctx):
    st = tqd.State(ctx, 5, "c64")
    with pytest.raises(tqd.TqdError) as e:
        st.set_option(tqd.OPT_TILE_QUBITS, 13)  # > 256 threads per CTA: rejected up front
    assert e.value.code == -1
    with pytest.raises(tqd.TqdError) as e:
        st.apply("CNOT", [1, 1])
    assert e.value.code == -1
    with pytest.raises(tqd.TqdError) as e:
        st.apply("RY", [9], [0.1])
    assert e.value.code == -1
    with pytest.raises(tqd.TqdError) as e:
        st.apply("MAT1", [0], (), np.array([[1, 1], [0, 1]]))
    assert e.value.code == -4
    with pytest.raises(tqd.TqdError) as e:
        tqd.tqd_apply_gate(st.handle, "RY", [0], ())  # missing parameter
    assert e.value.code == -1
    st.apply("RY", [0], [0.3])
    with pytest.raises(tqd.TqdError) as e:
        tqd.tqd_adjoint_grad(st.handle, [(0, 1, 1.0)] * 65)  # more than 64 terms
    assert e.value.code == -8
    v, g = st.adjoint_grad([(0, 1, 1.0)])
    assert abs(v - math.cos(0.3)) < 1e-6 and abs(g[0] + math.sin(0.3)) < 1e-6
    with pytest.raises(tqd.TqdError) as e:
        st.apply("X", [0])  # consumed
    assert e.value.code == -9
    st.reset()
    st.apply("X", [0])
    assert abs(st.expval([(0, 1, 1.0)])[0] + 1) < 1e-6
    st.free()
    with pytest.raises(tqd.TqdError) as e:
        tqd.tqd_state_init(ctx.handle, 0, tqd.C64)
    assert e.value.code == -2


@pytest.mark.parametrize("prefix", [0, 1])
def test_metrics_account_bytes(tqd, ctx, prefix):
    n = 20
    st = make_state(tqd, ctx, n, "c64")
    st.set_option(tqd.OPT_PRODUCT_PREFIX, prefix)
    st.apply_circuit(W.hea(n, 3, 0))
    st.reset_metrics()
    st.adjoint_grad(W.sum_z(n))
    m = st.metrics()
    st.free()
    sb = 8 << n
    assert m["fwd_sweeps"] > 0 and m["bwd_sweeps"] == m["fwd_sweeps"]
    assert m["fwd_sweep_bytes"] == 2 * sb * m["fwd_sweeps"]
    # the last reverse sweep reads psi and lambda but stores neither (with the product
    # prefix it stores lambda: the prefix gates' gradients come from its environments)
    assert m["bwd_sweep_bytes"] == 4 * sb * (m["bwd_sweeps"] - 1) + (3 if prefix else 2) * sb
    # the last layer's RZs and ring CNOTs are absorbed into the Z observable
    assert m["gates_absorbed"] == 2 * n
    assert m["gates_applied"] + m["gates_absorbed"] == 3 * 3 * n
    assert m["a2a_bytes"] == 0 and m["remaps"] == 0


def test_plan_reuse_across_parameter_changes(tqd, ctx, orc):
    """Training loops re-record the same circuit with new angles: the plan is reused
    (metrics.plans_reused) and the results follow the NEW values; a structural change
    (other wires, an identity-valued fixed rotation) plans afresh."""
    n = 14
    st = make_state(tqd, ctx, n, "c64", k=11, small_max=0)
    reused = 0
    for seed in range(3):
        gates = W.hea(n, 3, seed=100 + seed, small=True)
        gates.append(W.Gate("RZ", (3,), (0.0 if seed == 2 else 0.4,), None, False))  # identity at seed 2
        st.reset()
        st.apply_circuit(gates)
        val, grad = st.adjoint_grad(W.sum_z(n))
        rval, rgrad = orc.adjoint(n, gates, W.sum_z(n))
        assert abs(val - rval) < 1e-4 and np.max(np.abs(grad - rgrad)) < 1e-4
        m = st.metrics()
        reused = m["plans_reused"]
        assert reused == (1 if seed == 1 else (0 if seed == 0 else 1))
    st.reset()
    gates = W.hea(n, 3, seed=7, small=True, ring=False)  # other wires: new plan
    st.apply_circuit(gates)
    val, grad = st.adjoint_grad(W.sum_z(n))
    rval, rgrad = orc.adjoint(n, gates, W.sum_z(n))
    assert abs(val - rval) < 1e-4 and np.max(np.abs(grad - rgrad)) < 1e-4
    assert st.metrics()["plans_reused"] == reused
    st.free()


def _diag_heavy(n, seed):
    """Runs of diagonal gates on arbitrary bit pairs (CP, CZ, diagonal MAT2, Z/S/T,
    non-trainable and trainable RZ) between dense gates: K_DBLK merging, incl. more
    than DBLK_TERMS (16) lane / warp / base terms per run."""
    rng = np.random.default_rng(seed)
    gates = []
    for blk in range(6):
        gates += W.random_circuit(n, 6, seed * 10 + blk, kinds=["H", "RY", "U3", "MAT1"])
        for _ in range(int(rng.integers(5, 40))):
            k = ["CP", "CZ", "D2", "Z", "S", "T", "RZ", "RZc"][int(rng.integers(8))]
            if k in ("CP", "CZ", "D2"):
                w = tuple(int(v) for v in rng.choice(n, 2, replace=False))
                if k == "CZ":
                    gates.append(W.Gate("CZ", w))
                elif k == "CP":
                    gates.append(W.Gate("MAT2", w, (), W.cphase_matrix(float(rng.uniform(0, 2 * math.pi))), False))
                else:
                    ph = np.exp(1j * rng.uniform(0, 2 * math.pi, 4))
                    gates.append(W.Gate("MAT2", w, (), np.diag(ph).astype(np.complex128), False))
            else:
                w = (int(rng.integers(n)),)
                if k == "RZ":
                    gates.append(W.Gate("RZ", w, (float(rng.uniform(-0.3, 0.3)),), None, True))
                elif k == "RZc":
                    gates.append(W.Gate("RZ", w, (float(rng.uniform(0, 6.3)),), None, False))
                else:
                    gates.append(W.Gate(k, w))
    return gates + W.random_circuit(n, 4, seed + 99, kinds=["H", "RX"])


@pytest.mark.parametrize("grid", GRIDS)
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n,k", [(12, 9), (15, 10), (18, 12)])
def test_diagonal_blocks(tqd, ctx, orc, n, k, dtype, grid):
    """Merged diagonal runs (K_DBLK phase polynomials) against the oracle applying
    every diagonal gate: amplitudes, QFT = DFT, and adjoint gradients."""
    for seed in range(2):
        gates = _diag_heavy(n, seed)
        st = make_state(tqd, ctx, n, dtype, k=k, small_max=0, grid=grid)
        st.apply_circuit(gates)
        got = st.amplitudes()
        st.free()
        assert np.max(np.abs(got - orc.run(n, gates))) < TOL[dtype]["amp"], seed
        terms = W.random_z_terms(n, 4, seed) + [(1, 2, 0.5)]
        _grad_check(tqd, ctx, orc, n, gates, terms, dtype, small_max=0, k=k, grid=grid)
    x = 0b1011 % (1 << n)
    gates = W.basis_prep(n, x) + W.qft(n)
    st = make_state(tqd, ctx, n, dtype, k=k, small_max=0, grid=grid)
    st.apply_circuit(gates)
    got = st.amplitudes()
    st.free()
    N = 1 << n
    ref = np.exp(2j * np.pi * x * np.arange(N) / N) / math.sqrt(N)
    assert np.max(np.abs(got - ref)) < TOL[dtype]["amp"]


def test_cuda_graph_replay(tqd, ctx, orc):
    """TQD_OPT_USE_GRAPH: replays of the cached plan (rewind, and a re-recorded tape
    with new angles) run as CUDA graphs; values, gradients and metrics unchanged."""
    n = 16
    res = {}
    for graph in (0, 1):
        st = make_state(tqd, ctx, n, "c64", small_max=0)
        st.set_option(tqd.OPT_USE_GRAPH, graph)
        out = []
        try:
            for seed in (0, 1):
                gates = W.hea(n, 5, seed=seed, small=True)
                rval, rgrad = orc.adjoint(n, gates, W.sum_z(n))
                st.reset()
                st.apply_circuit(gates)
                for it in range(3):
                    if it:
                        st.rewind()
                    st.reset_metrics()
                    val, grad = st.adjoint_grad(W.sum_z(n))
                    m = st.metrics()
                    assert abs(val - rval) < 1e-4 and np.max(np.abs(grad - rgrad)) < 1e-4, (graph, seed, it)
                    out.append((m["fwd_sweeps"], m["bwd_sweeps"], m["kernel_launches"], m["hbm_bytes"]))
            ez = None
            st.reset()
            st.apply_circuit(W.hea(n, 5, seed=0, small=True))
            for it in range(2):
                if it:
                    st.rewind()
                ez = st.expval(W.sum_z(n))
            ref = orc.expval(orc.run(n, W.hea(n, 5, seed=0, small=True)), n, W.sum_z(n))
            assert np.max(np.abs(ez - ref)) < 1e-4
        finally:
            st.free()
        res[graph] = out
    assert res[0] == res[1]


def test_cuda_graph_value_dependent_structure(tqd, ctx, orc):
    """CUDA-graph replays when re-recorded VALUES change the kernel-op structure
    (ADVICE r1): non-trainable RZ / controlled phases whose angles are 0 or cancel
    in pairs are dropped from diagonal runs, so the same plan signature encodes to
    other kernel ops.  Every tape is checked against the oracle after rewinds."""
    n = 14
    base = W.hea(n, 3, seed=11, small=True)

    def tape(mode):
        a = {"on": 0.7, "zero": 0.0, "cancel": 0.45, "on2": -1.3}[mode]
        b = -a if mode == "cancel" else 0.25 * a
        gates = []
        for i, g in enumerate(base):
            gates.append(g)
            if i % 7 == 3:
                q = g.wires[0]
                gates.append(W.Gate("RZ", (q,), (a,), None, False))
                gates.append(W.Gate("RZ", (q,), (b,), None, False))
                gates.append(W.Gate("MAT2", (q, (q + 5) % n), (), W.cphase_matrix(a), False))
                gates.append(W.Gate("MAT2", (q, (q + 5) % n), (), W.cphase_matrix(b), False))
        return gates

    st = make_state(tqd, ctx, n, "c64", k=11, small_max=0)
    st.set_option(tqd.OPT_USE_GRAPH, 1)
    try:
        for mode in ("on", "zero", "cancel", "on2", "zero"):
            gates = tape(mode)
            rval, rgrad = orc.adjoint(n, gates, W.sum_z(n))
            st.reset()
            st.apply_circuit(gates)
            for it in range(3):
                if it:
                    st.rewind()
                val, grad = st.adjoint_grad(W.sum_z(n))
                assert abs(val - rval) < 1e-4 and np.max(np.abs(grad - rgrad)) < 1e-4, (mode, it)
    finally:
        st.free()


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_apply_circuit_matches_per_gate(tqd, ctx, orc, dtype):
    """tqd_apply_circuit (one C call) records exactly what G tqd_apply_gate calls record:
    bit-identical amplitudes (same tape, same kernels), value and gradients equal up to the order
    of their fp64 atomic sums, and all-or-nothing errors."""
    n = 13
    gates = W.random_circuit(n, 160, seed=7)
    out = []
    for mode in ("circuit", "per_gate"):
        st = make_state(tqd, ctx, n, dtype, k=10, small_max=0)
        if mode == "circuit":
            st.apply_circuit(gates)
        else:
            for g in gates:
                st.apply(g.name, g.wires, g.params, g.matrix, g.trainable)
        npar = st.n_params
        amps = st.amplitudes()
        st.reset()
        if mode == "circuit":
            st.apply_circuit(gates)
        else:
            for g in gates:
                st.apply(g.name, g.wires, g.params, g.matrix, g.trainable)
        val, grad = st.adjoint_grad(W.sum_z(n))
        st.free()
        out.append((npar, amps, val, np.asarray(grad)))
    assert out[0][0] == out[1][0]
    assert np.array_equal(out[0][1], out[1][1])
    # value / gradients are fp64 sums with atomic (order-free) accumulation across CTAs:
    # equal up to that summation order, not bitwise
    assert abs(out[0][2] - out[1][2]) < 1e-12
    assert np.max(np.abs(out[0][3] - out[1][3])) < 1e-12
    ref = orc.run(n, gates)
    assert np.max(np.abs(out[0][1] - ref)) < TOL[dtype]["amp"]
    # a bad gate anywhere in the list records nothing
    st = make_state(tqd, ctx, n, dtype)
    st.apply_circuit(gates[:5])
    before = st.n_params
    with pytest.raises(tqd.TqdError) as e:
        st.apply_circuit(gates[:5] + [W.Gate("CNOT", (2, 2))])
    assert e.value.code == -1 and st.n_params == before
    with pytest.raises(tqd.TqdError):
        st.apply_circuit([W.Gate("RY", (n,), (0.1,))])
    assert st.n_params == before
    st.apply_circuit([])
    st.free()


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n", [11, 14, 21])
def test_product_prefix(tqd, ctx, orc, n, dtype):
    """TQD_OPT_PRODUCT_PREFIX: every qubit's leading 1-qubit gates (all kinds, trainable
    and fixed, several per qubit) form a product state written directly; their gradients
    come from lambda's environments at the prefix boundary.  Against the oracle applying
    every gate, and prefix on == off."""
    rng = np.random.default_rng(n)
    # fixed 2-qubit gates before the first trainable (prefix) gate: lambda must still be
    # un-applied through them down to the prefix boundary
    gates = [W.Gate("CZ", (n - 1, 0)), W.Gate("CNOT", (1, 2))]
    for _ in range(3):  # prefix: several 1-qubit gates per qubit, interleaved across qubits
        for q in rng.permutation(n):
            k = ["RY", "RZ", "RX", "U3", "H", "S", "MAT1"][int(rng.integers(7))]
            if k == "MAT1":
                gates += W.random_circuit(n, 1, int(rng.integers(1 << 30)), kinds=["MAT1"])
                gates[-1] = W.Gate("MAT1", (int(q),), (), gates[-1].matrix, False)
            elif k in ("RY", "RZ", "RX"):
                gates.append(W.Gate(k, (int(q),), (float(rng.uniform(0, 6.3)),)))
            elif k == "U3":
                gates.append(W.Gate(k, (int(q),), tuple(float(v) for v in rng.uniform(0, 6.3, 3))))
            else:
                gates.append(W.Gate(k, (int(q),)))
    gates += [W.Gate("CNOT", (q, (q + 1) % n)) for q in range(0, n, 2)]
    gates += [W.Gate("RY", (q,), (float(rng.uniform(0, 6.3)),)) for q in range(n)]  # q odd: still prefix
    gates += W.hea(n, 2, seed=n, small=True) + W.random_circuit(n, 30, n + 1)
    terms = W.random_z_terms(n, 4, n) + W.sum_z(n) + [(1, 2, 0.4)]
    rval, rgrad = orc.adjoint(n, gates, terms)
    ref = orc.run(n, gates)
    out = {}
    for pf in (1, 0):
        st = make_state(tqd, ctx, n, dtype, small_max=0)
        st.set_option(tqd.OPT_PRODUCT_PREFIX, pf)
        st.apply_circuit(gates)
        amps = st.amplitudes()
        st.reset()
        st.apply_circuit(gates)
        val, grad = st.adjoint_grad(terms)
        st.rewind()  # the cached plan + prefix replayed
        val2, grad2 = st.adjoint_grad(terms)
        st.free()
        assert np.max(np.abs(amps - ref)) < TOL[dtype]["amp"], pf
        for v, g in ((val, grad), (val2, grad2)):
            assert abs(v - rval) < TOL[dtype]["val"] and np.max(np.abs(g - rgrad)) < TOL[dtype]["val"], pf
        out[pf] = grad
    assert np.max(np.abs(out[1] - out[0])) < TOL[dtype]["val"]


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n", [12, 15])
def test_product_prefix_qft_of_basis_state(tqd, ctx, orc, n, dtype):
    """cfg-5 family: X-prep + QFT + HEA.  The QFT of a basis state is a product state
    (each controlled phase meets a still-unrotated control qubit), so the whole QFT,
    its SWAPs and the HEA's first RY + RZ layer form the product prefix.  Against the
    oracle applying every gate, prefix on == off, and the prefix gate count."""
    wl = W.config(5, seed=n, n_override=n)
    gates = wl.gates
    rval, rgrad = orc.adjoint(n, gates, wl.terms)
    ref = orc.run(n, gates)
    n_pre = sum(1 for g in gates if g.name in ("X", "H", "SWAP") or g.name == "MAT2") + 2 * n  # + first RY, RZ layer
    out = {}
    for pf in (1, 0):
        st = make_state(tqd, ctx, n, dtype, small_max=0)
        st.set_option(tqd.OPT_PRODUCT_PREFIX, pf)
        st.apply_circuit(gates)
        amps = st.amplitudes()
        m = st.metrics()
        st.reset()
        st.apply_circuit(gates)
        val, grad = st.adjoint_grad(wl.terms)
        st.free()
        assert np.max(np.abs(amps - ref)) < TOL[dtype]["amp"], pf
        assert abs(val - rval) < TOL[dtype]["val"] and np.max(np.abs(grad - rgrad)) < TOL[dtype]["val"], pf
        assert m["gates_prefix"] == (n_pre if pf else 0), (pf, m["gates_prefix"], n_pre)
        out[pf] = grad
    assert np.max(np.abs(out[1] - out[0])) < TOL[dtype]["val"]


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_product_prefix_two_qubit_rules(tqd, ctx, orc, seed, dtype):
    """Random prefixes mixing X / H / trainable rotations with fixed CZ / CP / CNOT /
    SWAP / diagonal and controlled MAT2 gates: the 2-qubit gates join the product only
    when one qubit is in a parameter-independent basis state (a trainable rotation,
    even RX(0) exactly, disqualifies its qubit), then random entangling gates.
    Against the oracle and prefix off, including gradients of rotations at angle 0."""
    n = 12
    rng = np.random.default_rng(100 + seed)
    gates = []
    for _ in range(40):
        r = rng.random()
        a, b = (int(v) for v in rng.choice(n, 2, replace=False))
        if r < 0.15:
            gates.append(W.Gate("X", (a,)))
        elif r < 0.25:
            gates.append(W.Gate("H", (a,)))
        elif r < 0.35:
            k = ["RX", "RY", "RZ"][int(rng.integers(3))]
            th = 0.0 if rng.random() < 0.3 else float(rng.uniform(0, 6.3))
            gates.append(W.Gate(k, (a,), (th,)))
        elif r < 0.5:
            gates.append(W.Gate("CZ", (a, b)))
        elif r < 0.6:
            gates.append(W.Gate("MAT2", (a, b), (), W.cphase_matrix(float(rng.uniform(0, 6.3))), False))
        elif r < 0.72:
            gates.append(W.Gate("CNOT", (a, b)))
        elif r < 0.8:
            gates.append(W.Gate("SWAP", (a, b)))
        elif r < 0.9:
            d = np.exp(1j * rng.uniform(0, 6.3, 4))
            gates.append(W.Gate("MAT2", (a, b), (), np.diag(d).astype(np.complex128), False))
        else:  # controlled-U on wire a (block diag(I, U))
            u = W.random_circuit(1, 1, int(rng.integers(1 << 30)), kinds=["MAT1"])[0].matrix
            m = np.eye(4, dtype=np.complex128)
            m[2:, 2:] = u
            gates.append(W.Gate("MAT2", (a, b), (), m, False))
    gates += W.hea(n, 2, seed=seed, small=True) + W.random_circuit(n, 30, seed + 5)
    terms = W.random_z_terms(n, 4, seed) + W.sum_z(n) + [(1 << 3, 1 << 5, 0.3)]
    rval, rgrad = orc.adjoint(n, gates, terms)
    ref = orc.run(n, gates)
    out = {}
    for pf in (1, 0):
        st = make_state(tqd, ctx, n, dtype, small_max=0)
        st.set_option(tqd.OPT_PRODUCT_PREFIX, pf)
        st.apply_circuit(gates)
        amps = st.amplitudes()
        st.reset()
        st.apply_circuit(gates)
        val, grad = st.adjoint_grad(terms)
        st.free()
        assert np.max(np.abs(amps - ref)) < TOL[dtype]["amp"], pf
        assert abs(val - rval) < TOL[dtype]["val"] and np.max(np.abs(grad - rgrad)) < TOL[dtype]["val"], pf
        out[pf] = grad
    assert np.max(np.abs(out[1] - out[0])) < TOL[dtype]["val"]


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_product_prefix_whole_circuit(tqd, ctx, orc, dtype):
    """Edge case: EVERY gate is in the product prefix (no sweep at all): 1-qubit gates,
    SWAPs and the QFT of a basis state; the adjoint seed lambda = H psi is contracted
    directly.  Against the oracle; the tail absorption may take the trailing gates."""
    n = 13
    rng = np.random.default_rng(5)
    gates = [W.Gate("X", (q,)) for q in range(n) if rng.random() < 0.5] + W.qft(n)
    gates += [W.Gate("RY", (q,), (float(rng.uniform(0, 6.3)),)) for q in range(n)]
    gates += [W.Gate("SWAP", (0, n - 1)), W.Gate("RX", (3,), (0.7,)), W.Gate("U3", (5,), (0.3, 1.1, -0.4))]
    terms = W.random_pauli_terms(n, 5, 2) + W.sum_z(n)
    rval, rgrad = orc.adjoint(n, gates, terms)
    ref = orc.run(n, gates)
    st = make_state(tqd, ctx, n, dtype, small_max=0)
    st.set_option(tqd.OPT_PRODUCT_PREFIX, 1)
    st.apply_circuit(gates)
    amps = st.amplitudes()
    m = st.metrics()
    st.reset()
    st.apply_circuit(gates)
    val, grad = st.adjoint_grad(terms)
    m2 = st.metrics()
    st.free()
    assert m["gates_prefix"] == len(gates) and m["fwd_sweeps"] == 0, m
    assert m2["bwd_sweeps"] == 0
    assert np.max(np.abs(amps - ref)) < TOL[dtype]["amp"]
    assert abs(val - rval) < TOL[dtype]["val"] and np.max(np.abs(grad - rgrad)) < TOL[dtype]["val"]
