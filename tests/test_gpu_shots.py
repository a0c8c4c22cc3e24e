"""Shot noise, approximate (Gaussian) sampler through the C ABI vs the oracle
(PAPER.md:200-218): the noisy <Z_q> estimates (tqd_sample_gaussian_z) with the
same counter-based normals, and the reparameterised gradient
(tqd_adjoint_grad_gaussian) vs central finite differences of the ORACLE's
estimates (an independent route: the library's gradient comes from a derived
adjoint seed, the oracle's from re-running the sampler).
"""
import threading
import traceback

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu


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


def make(tqd, ctx, n, dtype, k=None, small_max=None, batch=1):
    st = tqd.State(ctx, n, dtype, batch=batch)
    if k is not None:
        st.set_option(tqd.OPT_TILE_QUBITS, k)
    if small_max is not None:
        st.set_option(tqd.OPT_SMALL_MAX, small_max)
    return st


def fd_grad(orc, n, gates, shots, seed, coeff, h=1e-4):
    """d/dtheta of sum_q coeff_q Zhat_q(theta) by central differences of the oracle,
    Richardson-extrapolated (error O(h^4)).  The estimates contain sqrt(p_i), which is
    smooth only away from p_i = 0: the circuits below keep every p_i well above 0."""
    def L(gg):
        return float(np.dot(coeff, orc.gauss_z(n, gg, shots, seed)))

    out = []
    for gi, g in enumerate(gates):
        if not g.trainable or g.name not in W.PARAMETRIC:
            continue
        for j in range(len(g.params)):
            d = []
            for hh in (h, h / 2):
                vals = []
                for s in (1, -1):
                    p = list(g.params)
                    p[j] += s * hh
                    gg = list(gates)
                    gg[gi] = W.Gate(g.name, g.wires, tuple(p), g.matrix, g.trainable)
                    vals.append(L(gg))
                d.append((vals[0] - vals[1]) / (2 * hh))
            out.append((4 * d[1] - d[0]) / 3)
    return np.array(out)


@pytest.mark.parametrize("dtype,tol", [("c128", 1e-10), ("c64", 1e-4)])
@pytest.mark.parametrize("n,k,small_max", [(5, None, None), (12, 10, 0), (15, 12, 0)])
def test_gaussian_z_estimates(tqd, ctx, orc, n, k, small_max, dtype, tol):
    gates = W.hea(n, 2, seed=n) + W.random_circuit(n, 30, n)
    for shots, seed in ((100.0, 1), (1e4, 7)):
        st = make(tqd, ctx, n, dtype, k, small_max)
        st.apply_circuit(gates)
        got = st.sample_gaussian_z(shots, seed)
        st.free()
        ref = orc.gauss_z(n, gates, shots, seed)
        assert np.max(np.abs(got - ref)) < tol, (shots, seed)


def test_gaussian_noiseless_basis_state(tqd, ctx):
    n = 9
    st = make(tqd, ctx, n, "c128")
    st.apply_circuit([W.Gate("X", (q,)) for q in range(n)])
    z = st.sample_gaussian_z(50.0, 3)
    st.free()
    assert np.max(np.abs(z + 1.0)) < 1e-12


@pytest.mark.parametrize("n,k,small_max", [(6, None, None), (11, 9, 0)])
def test_gaussian_gradient_vs_oracle_fd(tqd, ctx, orc, n, k, small_max):
    gates = W.hea(n, 2, seed=3 * n)  # generic angles: no p_i near 0
    shots, seed = 64.0, 5
    coeff = np.random.default_rng(n).standard_normal(n)
    st = make(tqd, ctx, n, "c128", k, small_max)
    st.apply_circuit(gates)
    val, grad = st.adjoint_grad_gaussian(shots, seed, coeff)
    st.free()
    assert abs(val - float(np.dot(coeff, orc.gauss_z(n, gates, shots, seed)))) < 1e-10
    ref = fd_grad(orc, n, gates, shots, seed, coeff)
    assert grad.shape == ref.shape
    assert np.max(np.abs(grad - ref)) < 1e-6, np.max(np.abs(grad - ref))


def test_gaussian_batch(tqd, ctx, orc):
    """Batch element b draws with seed + b."""
    n, B, shots, seed = 10, 3, 200.0, 11
    ans = W.hea(n, 2, seed=1, small=True)
    x = np.random.default_rng(2).uniform(0, 1.0, size=(n, B))
    st = make(tqd, ctx, n, "c128", 9, 0, batch=B)
    for q in range(n):
        st.apply_batch("RY", [q], x[q].reshape(B, 1))
    st.apply_circuit(ans)
    z = st.sample_gaussian_z(shots, seed)
    coeff = np.random.default_rng(3).standard_normal((B, n))
    val, grad = st.adjoint_grad_gaussian(shots, seed, coeff)
    st.free()
    tot = 0.0
    for b in range(B):
        gates = [W.Gate("RY", (q,), (float(x[q, b]),)) for q in range(n)] + ans
        ref = orc.gauss_z(n, gates, shots, seed + b)
        assert np.max(np.abs(z[b] - ref)) < 1e-10
        tot += float(np.dot(coeff[b], ref))
    assert abs(val - tot) < 1e-10
    assert grad.shape == (B * n + 2 * n * 2,)


@pytest.mark.parametrize("world", [2, 4])
def test_gaussian_emulated_world(tqd, orc, world):
    n, shots, seed = 12, 100.0, 4
    gates = W.hea(n, 2, seed=world)
    coeff = np.linspace(-1, 1, n)
    lid = tqd.tqd_loopback_id()
    res, err = [None] * world, [None] * world

    def worker(r):
        try:
            ctx = tqd.Context(world, r, 0, lid)
            try:
                st = make(tqd, ctx, n, "c128", 9, 0)
                st.apply_circuit(gates)
                z = st.sample_gaussian_z(shots, seed)
                st.reset()
                st.apply_circuit(gates)
                vg = st.adjoint_grad_gaussian(shots, seed, coeff)
                st.free()
                res[r] = (z, vg)
            finally:
                ctx.close()
        except Exception:
            err[r] = traceback.format_exc()

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    assert not any(err), "\n".join(e for e in err if e)
    ref = orc.gauss_z(n, gates, shots, seed)
    gref = fd_grad(orc, n, gates, shots, seed, coeff)
    for z, (val, grad) in res:
        assert np.max(np.abs(z - ref)) < 1e-10
        assert abs(val - float(np.dot(coeff, ref))) < 1e-10
        assert np.max(np.abs(grad - gref)) < 1e-6



# ---------------------------------------------------------------- exact sampler
def chi2_pvalue(counts, p, shots):
    """Pearson chi-square p-value of observed counts against probabilities p (bins with
    expected < 5 merged)."""
    from scipy.stats import chi2
    exp = shots * p
    order = np.argsort(exp)
    obs_b, exp_b, ob, eb = [], [], 0.0, 0.0
    for i in order:
        ob += counts[i]
        eb += exp[i]
        if eb >= 5:
            obs_b.append(ob); exp_b.append(eb); ob = eb = 0.0
    if eb > 0 and exp_b:
        obs_b[-1] += ob; exp_b[-1] += eb
    obs_b, exp_b = np.array(obs_b), np.array(exp_b)
    stat = float(np.sum((obs_b - exp_b) ** 2 / exp_b))
    return float(chi2.sf(stat, len(obs_b) - 1))


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n,k,small_max", [(4, None, None), (8, None, None), (13, 10, 0)])
def test_exact_sampler_distribution(tqd, ctx, orc, n, k, small_max, dtype):
    gates = W.hea(n, 2, seed=n) + W.random_circuit(n, 20, n)
    shots = 200000
    st = make(tqd, ctx, n, dtype, k, small_max)
    st.apply_circuit(gates)
    a = st.sample(shots, 5)
    b = st.sample(shots, 5)
    c = st.sample(shots, 6)
    st.free()
    assert a.shape == (shots,) and np.array_equal(a, b) and not np.array_equal(a, c)
    p = np.abs(orc.run(n, gates)) ** 2
    assert np.all(p[a] > 0)
    counts = np.bincount(a.astype(np.int64), minlength=1 << n)
    assert chi2_pvalue(counts, p, shots) > 1e-6


def test_exact_sampler_ghz_and_basis(tqd, ctx):
    n = 12
    st = make(tqd, ctx, n, "c64", 9, 0)
    st.apply_circuit([W.Gate("H", (0,))] + [W.Gate("CNOT", (q, q + 1)) for q in range(n - 1)])
    s = st.sample(10000, 1)
    st.reset()
    st.apply_circuit([W.Gate("X", (0,)), W.Gate("X", (5,))])
    t = st.sample(1000, 2)
    st.free()
    assert set(np.unique(s)) <= {0, (1 << n) - 1} and abs(np.mean(s == 0) - 0.5) < 0.03
    assert np.all(t == (1 << (n - 1)) | (1 << (n - 6)))


@pytest.mark.parametrize("world", [2, 4])
def test_exact_sampler_emulated_world(tqd, orc, world):
    """Hierarchical sampling over ranks: every rank returns the same shots, with the
    circuit's distribution (groups = shards)."""
    n, shots = 11, 100000
    gates = W.hea(n, 2, seed=world) + [W.Gate("H", (0,)), W.Gate("RY", (1,), (0.7,))]
    lid = tqd.tqd_loopback_id()
    res, err = [None] * world, [None] * world

    def worker(r):
        try:
            ctx = tqd.Context(world, r, 0, lid)
            try:
                st = make(tqd, ctx, n, "c128", 9, 0)
                st.apply_circuit(gates)
                res[r] = st.sample(shots, 3)
                st.free()
            finally:
                ctx.close()
        except Exception:
            err[r] = traceback.format_exc()

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    assert not any(err), "\n".join(e for e in err if e)
    for r in range(1, world):
        assert np.array_equal(res[r], res[0])
    p = np.abs(orc.run(n, gates)) ** 2
    counts = np.bincount(res[0].astype(np.int64), minlength=1 << n)
    assert chi2_pvalue(counts, p, shots) > 1e-6


def test_exact_sampler_batch(tqd, ctx, orc):
    n, B, shots = 9, 3, 50000
    ans = W.hea(n, 2, seed=2)
    x = np.random.default_rng(4).uniform(0, 2.0, size=(n, B))
    st = make(tqd, ctx, n, "c128", batch=B)
    for q in range(n):
        st.apply_batch("RY", [q], x[q].reshape(B, 1))
    st.apply_circuit(ans)
    s = st.sample(shots, 9)
    st.free()
    assert s.shape == (B, shots)
    for b in range(B):
        p = np.abs(orc.run(n, [W.Gate("RY", (q,), (float(x[q, b]),)) for q in range(n)] + ans)) ** 2
        counts = np.bincount(s[b].astype(np.int64), minlength=1 << n)
        assert chi2_pvalue(counts, p, shots) > 1e-6
