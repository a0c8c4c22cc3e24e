"""Pins of the stabilizer-tableau oracle (oracle/clifford.c): it must agree with the
independent state-vector oracle (run + expval, adjoint) on random Clifford circuits
and with closed forms of GHZ / Bell states at sizes the state-vector oracle cannot
reach.  CPU only."""
import math

import numpy as np
import pytest

import oracle as orc
import workloads as W

Q = math.pi / 2


def clifford_circuit(n, n_gates, seed, trainable=True):
    rng = np.random.default_rng(seed)
    kinds = ["I", "X", "Y", "Z", "H", "S", "SDG", "CNOT", "CZ", "SWAP", "RX", "RY", "RZ", "U3"]
    gates = []
    for _ in range(n_gates):
        k = kinds[int(rng.integers(len(kinds)))]
        a, b = (int(v) for v in rng.choice(n, 2, replace=False))
        if k in ("RX", "RY", "RZ"):
            gates.append(W.Gate(k, (a,), (Q * int(rng.integers(-4, 8)),), None, trainable))
        elif k == "U3":
            gates.append(W.Gate(k, (a,), tuple(Q * int(v) for v in rng.integers(-4, 8, 3)), None, trainable))
        elif k in ("CNOT", "CZ", "SWAP"):
            gates.append(W.Gate(k, (a, b)))
        else:
            gates.append(W.Gate(k, (a,)))
    return gates


def clifford_hea(n, depth, seed):
    """The bench ansatz (RY / RZ layers + CNOT ring) at angles k pi/2."""
    rng = np.random.default_rng(seed)
    gates = W.hea(n, depth, seed)
    for g in gates:
        if g.name in ("RY", "RZ"):
            g.params = (Q * int(rng.integers(0, 4)),)
    return gates


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("n", [3, 6, 9])
def test_tableau_expval_matches_state_vector(n, seed):
    gates = clifford_circuit(n, 60, 100 * n + seed)
    terms = W.random_pauli_terms(n, 24, seed) + W.random_z_terms(n, 6, seed) + W.sum_z(n)
    ref = orc.expval(orc.run(n, gates), n, terms)
    got = orc.clifford_expval(n, gates, terms)
    assert np.max(np.abs(got - ref)) < 1e-12
    # every <P> is 0 or +-1
    c = np.array([t[2] for t in terms])
    assert np.all(np.isin(np.round(got / c, 12), [-1.0, 0.0, 1.0]))


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("n", [4, 8])
def test_tableau_gradients_match_adjoint(n, seed):
    gates = clifford_circuit(n, 50, 7 * n + seed) + clifford_hea(n, 2, seed)
    terms = W.random_pauli_terms(n, 6, seed) + W.sum_z(n)
    rv, rg = orc.adjoint(n, gates, terms)
    v, g = orc.clifford_grad(n, gates, terms)
    assert abs(v - rv) < 1e-12
    assert g.shape == rg.shape and np.max(np.abs(g - rg)) < 1e-12


def test_tableau_bench_ansatz_small():
    n = 10
    gates = clifford_hea(n, 4, 3)
    rv, rg = orc.adjoint(n, gates, W.sum_z(n))
    v, g = orc.clifford_grad(n, gates, W.sum_z(n))
    assert abs(v - rv) < 1e-12 and np.max(np.abs(g - rg)) < 1e-12


def test_tableau_ghz_and_bell_closed_forms():
    """GHZ_n = (|0..0> + |1..1>)/sqrt 2: <Z_i Z_j> = 1, <Z_i> = 0, <X..X> = 1,
    <Y Y X..X> = -1; Bell pair after H, CNOT: <XX> = 1, <YY> = -1, <ZZ> = 1."""
    n = 40
    gates = [W.Gate("H", (0,))] + [W.Gate("CNOT", (q, q + 1)) for q in range(n - 1)]
    allx = (1 << n) - 1
    terms = [(0, 1, 1.0), (0, 1 | (1 << (n - 1)), 1.0), (allx, 0, 1.0), (allx, 0b11, 1.0), (0, 0b110, 2.0)]
    got = orc.clifford_expval(n, gates, terms)
    assert list(got) == [0.0, 1.0, 1.0, -1.0, 2.0]
    bell = [W.Gate("H", (0,)), W.Gate("CNOT", (0, 1))]
    got = orc.clifford_expval(2, bell, [(3, 0, 1.0), (3, 3, 1.0), (0, 3, 1.0), (1, 0, 1.0)])
    assert list(got) == [1.0, -1.0, 1.0, 0.0]


def test_tableau_rejects_non_clifford():
    with pytest.raises(ValueError):
        orc.clifford_expval(3, [W.Gate("T", (0,))], [(0, 1, 1.0)])
    with pytest.raises(ValueError):
        orc.clifford_expval(3, [W.Gate("RY", (0,), (0.3,))], [(0, 1, 1.0)])


@pytest.mark.parametrize("n", [5, 8])
def test_tableau_stabilizers_stabilize(n):
    """Every reported generator g satisfies sign * P |psi> = |psi> on the state-vector
    oracle's psi (expectation +1), and the generators commute pairwise."""
    gates = clifford_circuit(n, 70, 3 * n)
    psi = orc.run(n, gates)
    stab = orc.clifford_stabilizers(n, gates)
    ev = orc.expval(psi, n, [(x, z, float(s)) for x, z, s in stab])
    assert np.max(np.abs(ev - 1.0)) < 1e-12
    for i in range(n):
        for j in range(n):
            xi, zi, _ = stab[i]
            xj, zj, _ = stab[j]
            assert bin((xi & zj) ^ (zi & xj)).count("1") % 2 == 0
