"""Observable absorption of tqd_adjoint_grad (TQD_OPT_ABSORB_TAIL), host logic
pinned against the float64 oracle (no GPU): a trailing run of diagonal /
permutation gates U_tail is never applied; the Z-string observable is
conjugated instead, E = <psi_p|U_tail^dag H U_tail|psi_p> (Heisenberg picture of
the measurement; seed of the adjoint).

The oracle applies EVERY gate; the absorbed form runs the oracle on the prefix
with the conjugated terms.  Values and gradients must agree to rounding."""
import numpy as np
import pytest

import oracle
import workloads as W


@pytest.fixture(scope="module")
def tqd():
    import paper_2511_19291_b200 as t
    return t


def _terms(n, seed, T=6):
    return W.random_z_terms(n, T, seed) + [(0, 1 << (n - 1), 0.5), (0, 0, 0.25)]


@pytest.mark.parametrize("n", [2, 3, 5, 8])
def test_absorbed_value_and_grads_match_full_circuit(tqd, n):
    for seed in range(6):
        prefix = W.random_circuit(n, 30, 100 + seed)
        tail = W.diag_perm_tail(n, 25, 200 + seed)
        gates = prefix + tail
        terms = _terms(n, seed)
        tb, zout, sg = tqd.tqd_debug_absorb(n, gates, [t[1] for t in terms])
        assert tb <= len(prefix)  # the whole tail is absorbable (and maybe more)
        absorbed = [(0, z, c * s) for (_, _, c), z, s in zip(terms, zout, sg)]
        # value: oracle on the full circuit vs oracle on the prefix with conjugated terms
        e_full = oracle.expval(oracle.run(n, gates), n, terms).sum()
        e_abs = oracle.expval(oracle.run(n, gates[:tb]), n, absorbed).sum()
        assert abs(e_full - e_abs) < 1e-12, (seed, e_full, e_abs)
        # gradients: prefix parameters agree, absorbed (diagonal) parameters have 0
        v_full, g_full = oracle.adjoint(n, gates, terms)
        v_abs, g_abs = oracle.adjoint(n, gates[:tb], absorbed)
        assert abs(v_full - v_abs) < 1e-12
        assert np.max(np.abs(g_full[:len(g_abs)] - g_abs), initial=0.0) < 1e-11
        assert np.max(np.abs(g_full[len(g_abs):]), initial=0.0) < 1e-11


def test_absorption_stops_at_non_diagonal_gates(tqd):
    n = 4
    gates = W.diag_perm_tail(n, 10, 1) + [W.Gate("H", (2,))] + W.diag_perm_tail(n, 7, 2)
    tb, _, _ = tqd.tqd_debug_absorb(n, gates, [1, 2, 4])
    assert tb == 11
    # trainable non-diagonal rotation at the end: nothing is absorbed
    gates = W.diag_perm_tail(n, 5, 3) + [W.Gate("RX", (1,), (0.3,), None, True)]
    assert tqd.tqd_debug_absorb(n, gates, [2])[0] == len(gates)
    # empty circuit, no terms
    assert tqd.tqd_debug_absorb(n, [], [])[0] == 0


def test_conjugation_rules_closed_form(tqd):
    """CNOT[c,t]: Z_t -> Z_c Z_t, Z_c -> Z_c; X / Y: Z -> -Z; SWAP exchanges bits;
    diagonal gates commute (PAPER.md:306 qdev.cx(wires=[control, target]))."""
    n = 3
    G = W.Gate
    tb, z, s = tqd.tqd_debug_absorb(n, [G("CNOT", (0, 1))], [1 << 1, 1 << 0, 1 << 2])
    assert tb == 0 and z == [(1 << 1) | (1 << 0), 1 << 0, 1 << 2] and list(s) == [1, 1, 1]
    tb, z, s = tqd.tqd_debug_absorb(n, [G("X", (2,)), G("Y", (0,))], [1 << 2, 1 << 0, 5, 2])
    assert z == [4, 1, 5, 2] and list(s) == [-1, -1, 1, 1]
    tb, z, s = tqd.tqd_debug_absorb(n, [G("SWAP", (0, 2)), G("T", (1,)), G("CZ", (0, 1))], [1, 3, 5])
    assert z == [4, 6, 5] and list(s) == [1, 1, 1]


def test_hea_tail_is_last_rz_layer_and_ring(tqd):
    """BASELINE cfg 3 family: the last layer's RZs and ring CNOTs are absorbed
    (2n gates); the sum of Z_i becomes a sum of ring-neighbour Z strings."""
    for n in (6, 30):
        gates = W.hea(n, 3 if n == 6 else 20)
        tb, z, s = tqd.tqd_debug_absorb(n, gates, [1 << q for q in range(n)])
        assert tb == len(gates) - 2 * n
        assert all(v == 1 for v in s)
        if n == 6:
            terms = W.sum_z(n)
            absorbed = [(0, m, 1.0) for m in z]
            e_full = oracle.expval(oracle.run(n, gates), n, terms).sum()
            e_abs = oracle.expval(oracle.run(n, gates[:tb]), n, absorbed).sum()
            assert abs(e_full - e_abs) < 1e-12
