"""The single-launch register-layout circuit kernel (circuit_l3_kernel,
TQD_OPT_CIRCUIT_LAYOUT = 1, an experiment kept for its measurements: slower than the
default gate-by-gate kernel) for states of 8..10 qubits (BASELINE.json configs[0]):
forward gates, lambda = H psi and the reverse sweep with gradients
in one launch, the state in registers with layout exchanges through swizzled shared
memory.  Every case against the float64 oracle, and layout on == the gate-by-gate
circuit kernel (layout off); the metric circuit_layout_launches proves which ran."""
import numpy as np
import pytest

import workloads as W
from test_gpu_batch import encoder_inputs, expected, record_batch

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


def layout_circuit(n, n_gates, seed, fixed_first=0):
    """Every gate class the layout kernel takes: fixed and trainable 1-qubit gates,
    MAT1, CNOT / CZ / SWAP, controlled-U on either wire, CP and diagonal MAT2."""
    rng = np.random.default_rng(seed)
    kinds = ["X", "Y", "Z", "H", "S", "SDG", "T", "TDG", "I", "RX", "RY", "RZ", "U3", "MAT1",
             "CNOT", "CZ", "SWAP", "CP", "CU0", "CU1", "DIAG2"]
    gates = []
    for i in range(n_gates):
        k = kinds[int(rng.integers(len(kinds)))]
        if i < fixed_first and k in ("RX", "RY", "RZ", "U3"):
            k = "H"
        a, b = (int(v) for v in rng.choice(n, 2, replace=False))
        if k in ("RX", "RY", "RZ"):
            gates.append(W.Gate(k, (a,), (float(rng.uniform(0, 2 * np.pi)),)))
        elif k == "U3":
            gates.append(W.Gate(k, (a,), tuple(float(v) for v in rng.uniform(0, 2 * np.pi, 3))))
        elif k == "MAT1":
            u = W.random_circuit(1, 1, int(rng.integers(1 << 30)), kinds=["MAT1"])[0].matrix
            gates.append(W.Gate("MAT1", (a,), (), u, False))
        elif k in ("CNOT", "CZ", "SWAP"):
            gates.append(W.Gate(k, (a, b)))
        elif k == "CP":
            gates.append(W.Gate("MAT2", (a, b), (), W.cphase_matrix(float(rng.uniform(0, 6.3))), False))
        elif k in ("CU0", "CU1"):
            u = W.random_circuit(1, 1, int(rng.integers(1 << 30)), kinds=["MAT1"])[0].matrix
            m = np.eye(4, dtype=np.complex128)
            idx = [2, 3] if k == "CU0" else [1, 3]  # control wire a (MSB) / wire b
            m[np.ix_(idx, idx)] = u
            gates.append(W.Gate("MAT2", (a, b), (), m, False))
        elif k == "DIAG2":
            d = np.exp(1j * rng.uniform(0, 6.3, 4))
            gates.append(W.Gate("MAT2", (a, b), (), np.diag(d).astype(np.complex128), False))
        else:
            gates.append(W.Gate(k, (a,)))
    return gates


def run_adjoint(tqd, ctx, n, dtype, gates, terms, layout, reps=2):
    st = tqd.State(ctx, n, dtype)
    st.set_option(tqd.OPT_CIRCUIT_LAYOUT, layout)
    st.apply_circuit(gates)
    out = [st.adjoint_grad(terms)]
    for _ in range(reps - 1):
        st.rewind()  # cached op lists replayed
        out.append(st.adjoint_grad(terms))
    m = st.metrics()
    st.free()
    return out, m


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n", [8, 9, 10])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_layout_kernel_vs_oracle(tqd, ctx, orc, n, dtype, seed):
    gates = layout_circuit(n, 90, 10 * n + seed) + W.hea(n, 2, seed=seed)
    terms = W.random_z_terms(n, 4, seed) + W.sum_z(n) + [(0, 1 << (n - 1), 0.5)]
    rval, rgrad = orc.adjoint(n, gates, terms)
    res = {}
    for layout in (1, 0):
        out, m = run_adjoint(tqd, ctx, n, dtype, gates, terms, layout)
        assert m["circuit_layout_launches"] == (len(out) if layout else 0), m
        for val, grad in out:
            assert abs(val - rval) < TOL[dtype]["val"]
            assert np.max(np.abs(grad - rgrad)) < TOL[dtype]["val"], (layout, np.max(np.abs(grad - rgrad)))
        res[layout] = out[0][1]
    assert np.max(np.abs(res[1] - res[0])) < TOL[dtype]["val"]


def test_layout_kernel_cfg1(tqd, ctx, orc):
    """BASELINE.json configs[0] (10q HEA d4, <Z0>, 80 gradients, complex128) on the
    layout kernel: one launch, 1e-10 against the oracle."""
    wl = W.config(1)
    rval, rgrad = orc.adjoint(wl.n, wl.gates, wl.terms)
    out, m = run_adjoint(tqd, ctx, wl.n, "c128", wl.gates, wl.terms, 1, reps=3)
    assert m["circuit_layout_launches"] == 3 and m["kernel_launches"] <= 6  # + the gradient zeroing
    for val, grad in out:
        assert abs(val - rval) < 1e-10 and np.max(np.abs(grad - rgrad)) < 1e-10


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_layout_kernel_late_first_trainable(tqd, ctx, orc, dtype):
    """Fixed gates before the first trainable one are not un-applied (reverse list
    truncated there); the value and gradients stay exact."""
    n = 10
    gates = layout_circuit(n, 50, 77, fixed_first=50) + layout_circuit(n, 40, 78)
    terms = W.random_z_terms(n, 3, 5) + W.sum_z(n)
    rval, rgrad = orc.adjoint(n, gates, terms)
    out, m = run_adjoint(tqd, ctx, n, dtype, gates, terms, 1)
    assert m["circuit_layout_launches"] == 2
    for val, grad in out:
        assert abs(val - rval) < TOL[dtype]["val"] and np.max(np.abs(grad - rgrad)) < TOL[dtype]["val"]


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_layout_kernel_general_two_qubit_falls_back(tqd, ctx, orc, dtype):
    """A general 2-qubit unitary (CL_U2) is not taken: the gate-by-gate circuit kernel
    runs instead, same results."""
    n = 9
    gates = layout_circuit(n, 40, 5) + W.random_circuit(n, 5, 6, kinds=["MAT2"]) + W.hea(n, 1, seed=2)
    terms = W.sum_z(n)
    rval, rgrad = orc.adjoint(n, gates, terms)
    out, m = run_adjoint(tqd, ctx, n, dtype, gates, terms, 1, reps=1)
    assert m["circuit_layout_launches"] == 0
    val, grad = out[0]
    assert abs(val - rval) < TOL[dtype]["val"] and np.max(np.abs(grad - rgrad)) < TOL[dtype]["val"]


@pytest.mark.parametrize("kind", ["RY", "U3"])
@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_layout_kernel_batch(tqd, ctx, orc, dtype, kind):
    """Batch of states (one CTA each) with per-state encoder inputs: input gradients
    per element, ansatz gradients summed (the batched slot layout)."""
    n, B = 9, 3
    x = encoder_inputs(B, n, 31, kind)
    ansatz = W.hea(n, 3, seed=B) + layout_circuit(n, 30, 9)
    terms = W.random_z_terms(n, 3, n) + W.sum_z(n)
    coeff = np.random.default_rng(n).standard_normal((B, len(terms)))
    st = tqd.State(ctx, n, dtype, batch=B)
    st.set_option(tqd.OPT_CIRCUIT_LAYOUT, 1)
    record_batch(st, x, ansatz, kind)
    val, grad = st.adjoint_grad(terms, coeff=coeff)
    m = st.metrics()
    st.free()
    assert m["circuit_layout_launches"] == 1
    rval, rgrad = expected(orc, n, x, ansatz, terms, coeff, kind)
    assert abs(val - rval) < TOL[dtype]["val"]
    assert np.max(np.abs(grad - rgrad)) < TOL[dtype]["val"]
