"""Pins of the float64 oracle against things other than itself (CPU only).

Each test names the passage / closed form it checks.  The brute-force builder
below constructs full 2^n x 2^n operators with numpy ``kron`` from DIFFERENT
definitions than oracle.c uses: rotations as scipy ``expm(-i theta P / 2)``
(reading R4), CNOT / CZ as projector sums, SWAP as (I + XX + YY + ZZ)/2,
2q matrices expanded in the |a><c| (x) |b><d| basis.  A wrong bit order, a
transposed operand, a sign or a dropped term in oracle.c fails one of them.
"""
import json
import math
import os

import numpy as np
import pytest
from scipy.linalg import expm

import workloads as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")

I2 = np.eye(2, dtype=complex)
PX = np.array([[0, 1], [1, 0]], dtype=complex)
PY = np.array([[0, -1j], [1j, 0]], dtype=complex)
PZ = np.array([[1, 0], [0, -1]], dtype=complex)   # Z = (e0, -e1)
P0 = np.array([[1, 0], [0, 0]], dtype=complex)
P1 = np.array([[0, 0], [0, 1]], dtype=complex)


def rot(P, th):
    return expm(-1j * th * P / 2)


def bf_matrix(g):
    """Gate matrix from textbook identities (not oracle.c's entry formulas)."""
    n = g.name
    if n == "I": return I2
    if n == "X": return PX
    if n == "Y": return PY
    if n == "Z": return PZ
    if n == "H": return (PX + PZ) / math.sqrt(2)
    if n == "S": return expm(1j * math.pi / 4 * (I2 - PZ))          # sqrt(Z)
    if n == "SDG": return expm(-1j * math.pi / 4 * (I2 - PZ))
    if n == "T": return expm(1j * math.pi / 8 * (I2 - PZ))          # sqrt(S)
    if n == "TDG": return expm(-1j * math.pi / 8 * (I2 - PZ))
    if n == "RX": return rot(PX, g.params[0])
    if n == "RY": return rot(PY, g.params[0])
    if n == "RZ": return rot(PZ, g.params[0])
    if n == "U3":
        th, ph, la = g.params
        return np.exp(1j * (ph + la) / 2) * rot(PZ, ph) @ rot(PY, th) @ rot(PZ, la)
    if n == "CNOT": return np.kron(P0, I2) + np.kron(P1, PX)
    if n == "CZ": return np.kron(P0, I2) + np.kron(P1, PZ)
    if n == "SWAP": return (np.kron(I2, I2) + np.kron(PX, PX) + np.kron(PY, PY) + np.kron(PZ, PZ)) / 2
    if n in ("MAT1", "MAT2"): return np.asarray(g.matrix)
    raise KeyError(n)


def full_op(nq, ops):
    """kron over qubits 0..nq-1 (qubit 0 leftmost = most significant, R1)."""
    out = np.array([[1.0 + 0j]])
    for q in range(nq):
        out = np.kron(out, ops.get(q, I2))
    return out


def bf_gate(nq, g):
    M = bf_matrix(g)
    if len(g.wires) == 1:
        return full_op(nq, {g.wires[0]: M})
    q0, q1 = g.wires
    U = np.zeros((1 << nq, 1 << nq), dtype=complex)
    E = [[P0, np.array([[0, 1], [0, 0]], complex)], [np.array([[0, 0], [1, 0]], complex), P1]]
    for a in range(2):
        for b in range(2):
            for c in range(2):
                for d in range(2):
                    coef = M[2 * a + b, 2 * c + d]
                    if coef != 0:
                        U += coef * full_op(nq, {q0: E[a][c], q1: E[b][d]})
    return U


def bf_state(nq, gates):
    U = np.eye(1 << nq, dtype=complex)
    for g in gates:
        U = bf_gate(nq, g) @ U
    return U[:, 0], U


def pauli_op(nq, x, z):
    ops = {}
    for q in range(nq):
        xb, zb = (x >> q) & 1, (z >> q) & 1
        if xb and zb: ops[q] = PY
        elif xb: ops[q] = PX
        elif zb: ops[q] = PZ
    return full_op(nq, ops)


# ---------------------------------------------------------------- gates
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_random_circuit_vs_kron_unitary(orc, n, seed):
    """SPEC.md:99 oracle equivalence: 200-gate random circuits, q <= 6, 1e-9."""
    gates = W.random_circuit(n, 200 if n <= 4 else 60, seed)
    psi = orc.run(n, gates)
    ref, _ = bf_state(n, gates)
    assert np.max(np.abs(psi - ref)) < 1e-9


@pytest.mark.parametrize("n", [7, 8])
def test_kron_unitary_n8(orc, n):
    """north star: brute-force 2^n x 2^n unitary products at n <= 8."""
    gates = W.random_circuit(n, 25, seed=n)
    psi = orc.run(n, gates)
    ref, _ = bf_state(n, gates)
    assert np.max(np.abs(psi - ref)) < 1e-9


def test_gate_matrices_algebra(orc):
    """X^2 = Y^2 = Z^2 = H^2 = I, S^2 = Z, T^2 = S, RY(a)RY(b) = RY(a+b), CX.CX = I."""
    m = orc.gate_matrix
    for k in ("X", "Y", "Z", "H"):
        assert np.allclose(m(k) @ m(k), I2, atol=1e-14)
    assert np.allclose(m("Z"), PZ)
    assert np.allclose(m("S") @ m("S"), m("Z"), atol=1e-14)
    assert np.allclose(m("T") @ m("T"), m("S"), atol=1e-14)
    assert np.allclose(m("S") @ m("SDG"), I2, atol=1e-14)
    assert np.allclose(m("T") @ m("TDG"), I2, atol=1e-14)
    assert np.allclose(m("RY", (0.3,)) @ m("RY", (0.5,)), m("RY", (0.8,)), atol=1e-14)
    assert np.allclose(m("CNOT") @ m("CNOT"), np.eye(4), atol=1e-14)
    # Y = i X Z
    assert np.allclose(m("Y"), 1j * m("X") @ m("Z"), atol=1e-14)
    # U3 special cases: U3(th,0,0) = RY(th); U3(th,-pi/2,pi/2) = RX(th)
    assert np.allclose(m("U3", (0.7, 0, 0)), m("RY", (0.7,)), atol=1e-14)
    assert np.allclose(m("U3", (0.7, -math.pi / 2, math.pi / 2)), m("RX", (0.7,)), atol=1e-14)


def test_spec_examples(orc):
    """RY(pi/2)|0>, CNOT|10> = |11>, H|0>."""
    psi = orc.run(1, [W.Gate("RY", (0,), (math.pi / 2,))])
    assert np.allclose(psi, [math.cos(math.pi / 4), math.sin(math.pi / 4)], atol=1e-15)
    psi = orc.run(2, [W.Gate("X", (0,)), W.Gate("CNOT", (0, 1))])
    assert np.allclose(psi, [0, 0, 0, 1])
    psi = orc.run(1, [W.Gate("H", (0,))])
    assert np.allclose(psi, [1 / math.sqrt(2)] * 2)


def test_bell_and_ghz(orc):
    psi = orc.run(2, [W.Gate("H", (0,)), W.Gate("CNOT", (0, 1))])
    assert np.allclose(psi, [1 / math.sqrt(2), 0, 0, 1 / math.sqrt(2)], atol=1e-15)
    for n in (3, 7, 12):
        gates = [W.Gate("H", (0,))] + [W.Gate("CNOT", (q, q + 1)) for q in range(n - 1)]
        psi = orc.run(n, gates)
        ref = np.zeros(1 << n, complex)
        ref[0] = ref[-1] = 1 / math.sqrt(2)
        assert np.max(np.abs(psi - ref)) < 1e-14
        ez = orc.expval(psi, n, [(0, 1 << q, 1.0) for q in range(n)])
        assert np.allclose(ez, 0, atol=1e-14)
        zz = orc.expval(psi, n, [(0, (1 << i) | (1 << j), 1.0) for i in range(n) for j in range(i + 1, n)])
        assert np.allclose(zz, 1, atol=1e-14)
        xall = orc.expval(psi, n, [((1 << n) - 1, 0, 1.0)])
        assert abs(xall[0] - 1) < 1e-13


@pytest.mark.parametrize("n", [1, 3, 5, 8])
def test_qft_is_dft(orc, n):
    """R13: QFT|x> = sum_y w^{xy}/sqrt(N) |y>, w = e^{2 pi i/N} (closed form)."""
    N = 1 << n
    for x in (0, 1, N - 1, (0x5A5A % N)):
        psi = orc.run(n, W.basis_prep(n, x) + W.qft(n))
        ref = np.exp(2j * np.pi * x * np.arange(N) / N) / math.sqrt(N)
        assert np.max(np.abs(psi - ref)) < 1e-12


def test_norm_preserved(orc):
    """PAPER.md:71-72 (sum |alpha|^2 = 1)."""
    for n in (5, 10, 13):
        psi = orc.run(n, W.random_circuit(n, 80, seed=n))
        assert abs(np.vdot(psi, psi).real - 1) < 1e-12


# ---------------------------------------------------------------- expval
@pytest.mark.parametrize("th", [0.0, 0.3, math.pi / 3, 2.0, 4.5])
def test_rotation_closed_forms(orc, th):
    """north star: RY(theta) -> <Z> = cos theta; plus RX / RZ companions."""
    e = orc.expval(orc.run(1, [W.Gate("RY", (0,), (th,))]), 1, [(0, 1, 1.0), (1, 0, 1.0), (1, 1, 1.0)])
    assert np.allclose(e, [math.cos(th), math.sin(th), 0.0], atol=1e-14)
    e = orc.expval(orc.run(1, [W.Gate("RX", (0,), (th,))]), 1, [(0, 1, 1.0), (1, 1, 1.0)])
    assert np.allclose(e, [math.cos(th), -math.sin(th)], atol=1e-14)
    e = orc.expval(orc.run(1, [W.Gate("H", (0,)), W.Gate("RZ", (0,), (th,))]), 1, [(1, 0, 1.0), (1, 1, 1.0)])
    assert np.allclose(e, [math.cos(th), math.sin(th)], atol=1e-14)


def test_listing1_golden(orc):
    """PAPER.md:291-308 (Listing 1), expected values in tests/golden/listing1_measure_allZ.json."""
    with open(os.path.join(GOLDEN, "listing1_measure_allZ.json")) as f:
        gold = json.load(f)
    n = gold["nq"]
    gates = [W.Gate("Z", (0,)), W.Gate("RY", (0,), (math.pi / 3,)), W.Gate("CNOT", (0, 1))]
    e = orc.expval(orc.run(n, gates), n, [(0, 1 << q, 1.0) for q in range(n)])
    assert np.allclose(e, gold["expected"], atol=1e-14)


def test_expval_vs_dense_pauli(orc):
    """<psi|P|psi> vs kron-built Pauli operators."""
    for n in (1, 3, 5):
        psi = orc.run(n, W.random_circuit(n, 40, seed=n + 11))
        terms = W.random_pauli_terms(n, 12, seed=n)
        e = orc.expval(psi, n, terms)
        ref = [c * np.vdot(psi, pauli_op(n, x, z) @ psi).real for x, z, c in terms]
        assert np.allclose(e, ref, atol=1e-12)


def test_basis_and_hadamard_layers(orc):
    """e_0 -> all +1; H^n -> all 0."""
    n = 6
    e = orc.expval(orc.run(n, []), n, W.sum_z(n))
    assert np.allclose(e, 1)
    e = orc.expval(orc.run(n, [W.Gate("H", (q,)) for q in range(n)]), n, W.sum_z(n))
    assert np.allclose(e, 0, atol=1e-14)


# ---------------------------------------------------------------- gradients
def test_single_ry_gradient_closed_form(orc):
    """d<Z>/dtheta for RY(theta)|0> = -sin theta; -sqrt(3)/2 at pi/3."""
    for th in (math.pi / 3, 0.1, 2.5):
        gates = [W.Gate("RY", (0,), (th,))]
        val, g = orc.adjoint(1, gates, [(0, 1, 1.0)])
        assert abs(val - math.cos(th)) < 1e-14
        assert abs(g[0] + math.sin(th)) < 1e-14


def _single_qubit_brute(seq, th_override=None):
    """<Z> of a 1-qubit gate sequence by 2x2 products (brute force)."""
    v = np.array([1, 0], complex)
    for g in seq:
        v = bf_matrix(g) @ v
    return np.vdot(v, PZ @ v).real


def test_entangler_free_factorization(orc):
    """Product circuits: E(sum Z_i) = sum_i E_i (1-qubit brute force); gradients too."""
    n, depth = 5, 4
    gates = [g for g in W.hea(n, depth, seed=3) if g.name != "CNOT"]
    val, grad = orc.adjoint(n, gates, W.sum_z(n))
    ref = sum(_single_qubit_brute([g for g in gates if g.wires[0] == q]) for q in range(n))
    assert abs(val - ref) < 1e-12
    # gradient of each parameter from 1-qubit central differences of the brute force
    p = 0
    for gi, g in enumerate(gates):
        q = g.wires[0]
        h = 1e-5
        def e_of(v):
            seq = []
            for gj, g2 in enumerate(gates):
                if g2.wires[0] != q:
                    continue
                seq.append(W.Gate(g2.name, g2.wires, (v,)) if gj == gi else g2)
            return _single_qubit_brute(seq)
        fd = (e_of(g.params[0] + h) - e_of(g.params[0] - h)) / (2 * h)
        assert abs(grad[p] - fd) < 1e-8
        p += 1


@pytest.mark.parametrize("seed", range(6))
def test_adjoint_vs_shift_vs_fd_vs_stored(orc, seed):
    """Four independent gradient routes agree."""
    n = 4 + seed % 3
    gates = W.random_circuit(n, 40, seed=seed)
    terms = W.random_pauli_terms(n, 3, seed) + W.random_z_terms(n, 2, seed)
    val, ga = orc.adjoint(n, gates, terms)
    vs, gs = orc.adjoint_stored(n, gates, terms)
    gp = orc.param_shift(n, gates, terms)
    gf = orc.finite_diff(n, gates, terms, 1e-6)
    e = orc.expval(orc.run(n, gates), n, terms).sum()
    assert abs(val - e) < 1e-12 and abs(vs - e) < 1e-12
    assert len(ga) == sum(W.PARAMETRIC.get(g.name, 0) for g in gates)
    assert np.max(np.abs(ga - gs)) < 1e-9
    assert np.max(np.abs(ga - gp)) < 1e-9
    assert np.max(np.abs(ga - gf)) < 1e-6


def test_gradient_vs_dense_derivative(orc):
    """d/dtheta <0|U^dag H U|0> from the kron-built product with the expm
    derivative (dR_P/dtheta = -i/2 P R_P) in one factor."""
    n = 3
    gates = W.hea(n, 2, seed=5)
    terms = [(0, 0b011, 0.7), (0b100, 0b000, -0.4)]
    H = sum(c * pauli_op(n, x, z) for x, z, c in terms)
    _, grad = orc.adjoint(n, gates, terms)
    p = 0
    e0 = np.zeros(1 << n, complex); e0[0] = 1
    for k, g in enumerate(gates):
        if g.name not in W.PARAMETRIC:
            continue
        P = {"RX": PX, "RY": PY, "RZ": PZ}[g.name]
        U = np.eye(1 << n, dtype=complex)
        dU = np.eye(1 << n, dtype=complex)
        for j, g2 in enumerate(gates):
            Gj = bf_gate(n, g2)
            U = Gj @ U
            if j == k:
                dU = full_op(n, {g.wires[0]: -0.5j * P}) @ Gj @ dU
            else:
                dU = Gj @ dU
        psi, dpsi = U @ e0, dU @ e0
        ref = 2 * np.vdot(psi, H @ dpsi).real
        assert abs(grad[p] - ref) < 1e-12
        p += 1


def test_trainable_flags(orc):
    """Non-trainable parametric gates get no gradient slot (tqd_apply_gate contract)."""
    gates = W.hea(3, 2, seed=1)
    for g in gates[::2]:
        g.trainable = False
    val, g = orc.adjoint(3, gates, W.sum_z(3))
    assert len(g) == sum(1 for x in gates if x.trainable and x.name in W.PARAMETRIC)
