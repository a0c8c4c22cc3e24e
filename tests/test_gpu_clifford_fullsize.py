"""Full-size parity through the C ABI: the bench ansatz (30 qubits, HEA ring depth 20,
complex64, default options = the launch configuration bench.py times) and the cfg-4
shape (33 qubits, depth 10) at Clifford angles k pi/2, against the stabilizer-tableau
oracle (oracle/clifford.c, pinned in tests/test_oracle_clifford.py).  Expectations and
EVERY gradient element-wise at the north-star tolerance (1e-4, complex64).

Observables with nonzero gradients: for a sample of parameters j, a stabilizer
generator P of the state with theta_j shifted by +pi/2 that is not a stabilizer of the
unshifted state, so dE/dtheta_j = (1 - <P>_-) / 2 != 0 (parameter shift), with X / Y /
Z factors on all qubits (the X/Y adjoint seed path).  The sum-Z runs use circuits whose
rotations are multiples of pi except a few pi/2 in the last layer: the 20 layers of
CNOT ring act on computational basis states, and every <Z_i> is exact."""
import math

import numpy as np
import pytest

import oracle as orc
import workloads as W

pytestmark = pytest.mark.gpu

Q = math.pi / 2
TOL = 1e-4  # north_star, complex64


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


def quarter_hea(n, depth, seed):
    rng = np.random.default_rng(seed)
    gates = W.hea(n, depth, seed)
    for g in gates:
        if g.name in ("RY", "RZ"):
            g.params = (Q * int(rng.integers(0, 4)),)
    return gates


def basis_hea(n, depth, seed, n_half):
    """RY in {0, pi} (bit flips), RZ in {k pi/2} (phases), n_half RY(+-pi/2) in the last layer."""
    rng = np.random.default_rng(seed)
    gates = W.hea(n, depth, seed)
    last_ry = [i for i, g in enumerate(gates) if g.name == "RY" and i >= len(gates) - 3 * n]
    half = set(int(v) for v in rng.choice(last_ry, n_half, replace=False)) if n_half else set()
    for i, g in enumerate(gates):
        if g.name == "RY":
            g.params = ((Q if rng.random() < 0.5 else -Q) if i in half else math.pi * int(rng.integers(0, 2)),)
        elif g.name == "RZ":
            g.params = (Q * int(rng.integers(0, 4)),)
    return gates


def sensitive_terms(n, gates, n_terms, seed):
    """Stabilizers of theta_j + pi/2 circuits that are not stabilizers of the circuit."""
    rng = np.random.default_rng(seed)
    rot = [i for i, g in enumerate(gates) if g.name in ("RY", "RZ")]
    terms = []
    for gi in rng.permutation(rot):
        if len(terms) == n_terms:
            break
        g = gates[gi]
        shifted = list(gates)
        shifted[gi] = W.Gate(g.name, g.wires, (g.params[0] + Q,), None, True)
        stab = orc.clifford_stabilizers(n, shifted)
        ev = orc.clifford_expval(n, gates, [(x, z, 1.0) for x, z, _ in stab])
        cand = [k for k in range(n) if ev[k] == 0.0]
        if not cand:
            continue
        x, z, s = stab[int(rng.choice(cand))]
        terms.append((x, z, float(s) * float(rng.uniform(0.5, 1.0))))
    return terms


def run_gpu(tqd, ctx, n, gates, terms):
    st = tqd.State(ctx, n, "c64")
    try:
        st.apply_circuit(gates)
        ev = st.expval(terms)
        st.rewind()
        val, grad = st.adjoint_grad(terms)
    finally:
        st.free()
    return ev, val, grad


@pytest.mark.parametrize("n,depth,seed", [(30, 20, 0), (30, 20, 1), (33, 10, 2)])
def test_fullsize_clifford_pauli_gradients(tqd, ctx, n, depth, seed):
    gates = quarter_hea(n, depth, seed)
    terms = sensitive_terms(n, gates, 16, seed)
    assert len(terms) >= 12
    # + stabilizers of the state itself: <P> = +-1 (nonzero value, zero gradient)
    rng = np.random.default_rng(seed + 99)
    stab = orc.clifford_stabilizers(n, gates)
    for k in rng.choice(n, 4, replace=False):
        x, z, sg = stab[int(k)]
        terms.append((x, z, float(sg) * float(rng.uniform(0.5, 1.0))))
    rev = orc.clifford_expval(n, gates, terms)
    rval, rgrad = orc.clifford_grad(n, gates, terms)
    assert np.count_nonzero(rgrad) >= 12  # a real gradient check, not zeros
    ev, val, grad = run_gpu(tqd, ctx, n, gates, terms)
    assert np.max(np.abs(ev - rev)) < TOL, np.max(np.abs(ev - rev))
    assert abs(val - rval) < TOL
    assert grad.shape == rgrad.shape
    err = np.max(np.abs(grad - rgrad))
    print(f"n={n} terms={len(terms)} nonzero grads={np.count_nonzero(rgrad)} max |dgrad|={err:.2e}")
    assert err < TOL


@pytest.mark.parametrize("seed,n_half", [(0, 0), (1, 4), (2, 4), (3, 8)])
def test_fullsize_clifford_bench_path_sum_z(tqd, ctx, seed, n_half):
    """The exact bench configuration (30 q, depth 20, sum Z_i: tail absorption and
    product prefix on) at Clifford angles: E and all 1200 gradients."""
    n = 30
    gates = basis_hea(n, 20, seed, n_half)
    terms = W.sum_z(n)
    rz = orc.clifford_expval(n, gates, terms)
    rval, rgrad = orc.clifford_grad(n, gates, terms)
    if n_half == 0:  # a basis state: every <Z_i> = +-1 checks the 20 CNOT rings' bit flips
        assert np.count_nonzero(rz) == n
    ev, val, grad = run_gpu(tqd, ctx, n, gates, terms)
    assert np.max(np.abs(ev - rz)) < TOL
    assert abs(val - rval) < TOL
    assert np.max(np.abs(grad - rgrad)) < TOL
