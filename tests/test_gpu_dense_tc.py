"""Tensor-core dense block (tcgen05.mma kind::tf32, TMEM accumulators; csrc/dense_tc.cu,
include/tqd.h tqd_debug_dense_block): a 6-qubit unitary on the 6 lowest canonical bits.

Pinned to the float64 oracle: the oracle applies the block's gates one by one to a
prepared state; the test builds the 64 x 64 block matrix from the same gates (kron
products of the textbook matrices, MSB-first: logical qubit n-1-b is bit b of the
block index) and the kernel applies it.  3xTF32 must meet the north-star amplitude
tolerance (1e-5, complex64); 1xTF32 is reported for comparison (round 1 measured
~3e-4 relative with cuBLAS TF32)."""
import math

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tqd():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need CUDA")
    import paper_2511_19291_b200 as t
    return t


def _mat1(g):
    c, s = (math.cos(g.params[0] / 2), math.sin(g.params[0] / 2)) if g.params else (1.0, 0.0)
    if g.name == "RY":
        return np.array([[c, -s], [s, c]], complex)
    if g.name == "RZ":
        return np.diag([np.exp(-0.5j * g.params[0]), np.exp(0.5j * g.params[0])])
    if g.name == "RX":
        return np.array([[c, -1j * s], [-1j * s, c]])
    if g.name == "H":
        return np.array([[1, 1], [1, -1]], complex) / math.sqrt(2)
    raise ValueError(g.name)


def _block_matrix(n, gates, m=6):
    """The 2^m x 2^m matrix of `gates` acting on logical qubits n-m .. n-1 (bit b = qubit n-1-b)."""
    D = 1 << m
    U = np.eye(D, dtype=complex)
    idx = np.arange(D)
    for g in gates:
        G = np.zeros((D, D), complex)
        if g.name == "CNOT":
            cb, tb = n - 1 - g.wires[0], n - 1 - g.wires[1]
            for i in range(D):
                j = i ^ (1 << tb) if (i >> cb) & 1 else i
                G[j, i] = 1
        else:
            b = n - 1 - g.wires[0]
            u = _mat1(g)
            for i in range(D):
                bi = (i >> b) & 1
                for bo in (0, 1):
                    G[(i & ~(1 << b)) | (bo << b), i] += u[bo, bi]
        U = G @ U
    return U


def _block_gates(n, seed, layers=2):
    rng = np.random.default_rng(seed)
    qs = list(range(n - 6, n))
    gates = []
    for _ in range(layers):
        gates += [W.Gate("RY", (q,), (float(rng.uniform(0, 2 * math.pi)),)) for q in qs]
        gates += [W.Gate("RZ", (q,), (float(rng.uniform(0, 2 * math.pi)),)) for q in qs]
        gates += [W.Gate("CNOT", (qs[i], qs[i + 1])) for i in range(5)]
    return gates + [W.Gate("H", (qs[2],)), W.Gate("RX", (qs[4],), (0.7,))]


@pytest.mark.parametrize("n", [14, 17])
def test_dense_block_3xtf32_vs_oracle(tqd, orc, n):
    prep = W.random_circuit(n, 80, 100 + n)
    blk = _block_gates(n, n)
    psi0 = orc.run(n, prep)
    ref = orc.run(n, prep + blk)
    U = _block_matrix(n, blk)
    assert np.allclose(U.conj().T @ U, np.eye(64), atol=1e-12)
    got, _ = tqd.tqd_debug_dense_block(n, U, psi0, precision=3)
    err3 = float(np.max(np.abs(got - ref)))
    got1, _ = tqd.tqd_debug_dense_block(n, U, psi0, precision=1)
    err1 = float(np.max(np.abs(got1 - ref)))
    scale = float(np.max(np.abs(ref)))
    print(f"n={n}: 3xTF32 max abs {err3:.2e} (rel {err3 / scale:.2e}); 1xTF32 max abs {err1:.2e} (rel {err1 / scale:.2e})")
    assert err3 < 1e-5
    assert err3 < err1


def test_dense_block_haar_unitary(tqd):
    """A Haar-random 64 x 64 unitary on a random state: 3xTF32 against numpy float64."""
    n = 15
    rng = np.random.default_rng(7)
    z = rng.normal(size=(64, 64)) + 1j * rng.normal(size=(64, 64))
    q, r = np.linalg.qr(z)
    U = q * (np.diag(r) / np.abs(np.diag(r)))
    psi = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    psi /= np.linalg.norm(psi)
    psi = psi.astype(np.complex64)
    got, _ = tqd.tqd_debug_dense_block(n, U, psi, precision=3)
    ref = (psi.astype(np.complex128).reshape(-1, 64) @ U.T).reshape(-1)
    assert np.max(np.abs(got - ref)) < 1e-5
