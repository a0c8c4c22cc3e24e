"""Pins of the oracle's approximate (Gaussian) shot-noise sampler
against what the mathematics fixes, independent of its own formula:

* the sample conserves the shot count exactly: sum_i y_i = shots, because the
  Householder S maps u = sqrt(p) to e_K and z_K = 0 (any state);
* a basis state |K> = |1...1> has no noise: y = shots e_K;
* over many seeds the sample has the multinomial moments E y = shots p and
  Cov y = shots (diag p - p p^T), and the per-qubit
  estimates have mean <Z_q> and the binomial variance (1 - <Z_q>^2) / shots;
* the counter-based generator has uniform / normal moments.
"""
import numpy as np
import pytest

import workloads as W


def test_generator_moments(orc):
    u = np.array([orc.uniform(7, k) for k in range(20000)])
    assert abs(u.mean() - 0.5) < 0.01 and abs(u.var() - 1 / 12) < 0.005
    assert u.min() >= 0.0 and u.max() < 1.0
    z = np.array([orc.normal(7, i) for i in range(20000)])
    assert abs(z.mean()) < 0.03 and abs(z.var() - 1.0) < 0.04
    assert abs(np.mean(z ** 4) - 3.0) < 0.25  # Gaussian kurtosis
    assert orc.uniform(1, 5) != orc.uniform(2, 5)  # seeds matter


@pytest.mark.parametrize("n,seed", [(3, 0), (5, 1), (8, 2)])
def test_shot_count_conserved(orc, n, seed):
    gates = W.random_circuit(n, 40, seed)
    psi = orc.run(n, gates)
    for shots in (10.0, 1000.0, 1e6):
        y = orc.gauss_sample(psi, n, shots, 123 + seed)
        assert abs(y.sum() - shots) < 1e-9 * shots


def test_basis_state_K_is_noiseless(orc):
    n = 4
    gates = [W.Gate("X", (q,)) for q in range(n)]
    psi = orc.run(n, gates)
    y = orc.gauss_sample(psi, n, 500.0, 9)
    ref = np.zeros(1 << n)
    ref[-1] = 500.0
    assert np.max(np.abs(y - ref)) < 1e-9


def test_multinomial_moments(orc):
    n, shots, S = 2, 400.0, 4000
    gates = [W.Gate("RY", (0,), (1.1,)), W.Gate("RY", (1,), (0.4,)), W.Gate("CNOT", (0, 1))]
    psi = orc.run(n, gates)
    p = np.abs(psi) ** 2
    ys = np.array([orc.gauss_sample(psi, n, shots, s) for s in range(S)])
    mean = ys.mean(0)
    cov = np.cov(ys.T)
    ref_cov = shots * (np.diag(p) - np.outer(p, p))
    assert np.max(np.abs(mean - shots * p)) < 4 * np.sqrt(shots / S)
    assert np.max(np.abs(cov - ref_cov)) < 0.08 * shots * p.max()


def test_z_estimates_mean_and_variance(orc):
    n, shots, S = 3, 200.0, 3000
    gates = [W.Gate("RY", (q,), (0.3 + 0.5 * q,)) for q in range(n)]
    exact = np.cos(0.3 + 0.5 * np.arange(n))  # <Z_q> of the product state
    est = np.array([orc.gauss_z(n, gates, shots, s) for s in range(S)])
    assert np.max(np.abs(est.mean(0) - exact)) < 4 * np.sqrt(1 / (shots * S))
    var = est.var(0)
    ref_var = (1 - exact ** 2) / shots
    assert np.max(np.abs(var / ref_var - 1)) < 0.12
