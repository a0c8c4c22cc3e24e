"""Randomised parity sweep on the GPU (a robustness check, not a test): random circuits of
every gate kind, random observables and random options (product prefix 0/1/2, tile
qubits, grid, small-state threshold, batch, loopback world size, fused remaps) against
the float64 oracle.  python tools/fuzz_parity.py [seconds] [seed] (FUZZ_N=lo,hi: local-qubit range);
prints one line per failure and a summary."""
import os
import sys
import threading
import time
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as orc  # noqa: E402
import paper_2511_19291_b200 as tqd  # noqa: E402
import workloads as W  # noqa: E402

TOL = {"c64": (1e-5, 1e-4), "c128": (1e-12, 1e-10)}
NMIN, NMAX = (int(v) for v in os.environ.get("FUZZ_N", "11,17").split(","))  # local qubits [NMIN, NMAX)


def run_world(world, fn):
    lid = tqd.tqd_loopback_id()
    res, err = [None] * world, [None] * world

    def worker(r):
        try:
            ctx = tqd.Context(world, r, 0, lid)
            try:
                res[r] = fn(r, ctx)
            finally:
                ctx.close()
        except Exception:
            err[r] = traceback.format_exc()
    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    bad = [e for e in err if e]
    if bad:
        raise RuntimeError(bad[0])
    return res


def case(rng):
    world = int(rng.choice([1, 1, 2, 4]))
    g = world.bit_length() - 1
    n = int(rng.integers(NMIN + g, NMAX + g))
    dtype = str(rng.choice(["c64", "c128"]))
    prefix = int(rng.choice([0, 1, 2]))
    k = int(rng.choice([9, 10, 11, 12])) if dtype == "c64" else int(rng.choice([9, 10, 11]))
    fused = int(rng.integers(0, 2))
    grid = int(rng.choice([0, 0, 3, 7]))
    small = bool(rng.integers(0, 2))
    seed = int(rng.integers(1 << 30))
    gates = []
    if rng.random() < 0.5:  # a product-prefix-friendly start
        gates += [W.Gate("X", (q,)) for q in range(n) if rng.random() < 0.3]
        if rng.random() < 0.5:
            gates += W.qft(n)[: int(rng.integers(5, 40))]
    gates += W.random_circuit(n, int(rng.integers(20, 120)), seed, small=small) + W.hea(n, int(rng.integers(1, 4)), seed, small=small)
    terms = W.random_z_terms(n, 3, seed) + (W.random_pauli_terms(n, 3, seed) if rng.random() < 0.5 else []) + W.sum_z(n)
    batch = int(rng.choice([1, 1, 2, 3]))
    enc = None
    if batch > 1:  # per-element encoder inputs (batched RY / U3 / RZ, trainable or frozen)
        kind = str(rng.choice(["RY", "U3", "RZ"]))
        npar = 3 if kind == "U3" else 1
        enc = (kind, rng.uniform(0, np.pi, size=(n, batch, npar)), bool(rng.integers(0, 2)))
    return dict(world=world, n=n, dtype=dtype, prefix=prefix, k=k, fused=fused, grid=grid, batch=batch), gates, terms, enc


def main():
    secs = float(sys.argv[1]) if len(sys.argv) > 1 else 300
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    t0, ncase, nfail = time.time(), 0, 0
    while time.time() - t0 < secs:
        cfg, gates, terms, enc = case(rng)
        B, n = cfg["batch"], cfg["n"]
        coeff = None
        if enc is None:
            refs = [orc.run(n, gates)]
            rval, rgrad = orc.adjoint(n, gates, terms)
        else:
            # per-element circuits: encoder gates first; batched slots per element, shared summed
            kind, x, trn = enc
            coeff = rng.standard_normal((B, len(terms)))
            refs, rval, encg, shared = [], 0.0, [], None
            for b in range(B):
                eg = [W.Gate(kind, (q,), tuple(float(v) for v in x[q, b]), None, trn) for q in range(n)]
                refs.append(orc.run(n, eg + gates))
                v, g = orc.adjoint(n, eg + gates, [(t[0], t[1], float(coeff[b, i])) for i, t in enumerate(terms)])
                rval += v
                ne = n * x.shape[2] if trn else 0
                if trn:
                    encg.append(g[:ne].reshape(n, x.shape[2]))
                shared = g[ne:] if shared is None else shared + g[ne:]
            rgrad = np.concatenate([np.stack(encg, 1).reshape(-1) if trn else np.zeros(0), shared])

        def fn(r, ctx):
            st = tqd.State(ctx, n, cfg["dtype"], batch=B) if B > 1 else tqd.State(ctx, n, cfg["dtype"])
            st.set_option(tqd.OPT_PRODUCT_PREFIX, cfg["prefix"])
            st.set_option(tqd.OPT_TILE_QUBITS, cfg["k"])
            st.set_option(tqd.OPT_SMALL_MAX, 0)
            st.set_option(tqd.OPT_FUSED_REMAP, cfg["fused"])
            st.set_option(tqd.OPT_GRID_CTAS, cfg["grid"])
            def record():
                if enc is not None:
                    for q in range(n):
                        st.apply_batch(enc[0], [q], enc[1][q], trainable=enc[2])
                st.apply_circuit(gates)
            record()
            amp = st.amplitudes()
            st.reset()
            record()
            val, grad = st.adjoint_grad(terms, coeff=coeff) if coeff is not None else st.adjoint_grad(terms)
            st.free()
            return amp, val, grad
        try:
            if cfg["world"] == 1:
                ctx = tqd.Context(1, 0, 0)
                try:
                    outs = [fn(0, ctx)]
                finally:
                    ctx.close()
            else:
                outs = run_world(cfg["world"], fn)
            ta, tv = TOL[cfg["dtype"]]
            ref = np.concatenate(refs)
            for amp, val, grad in outs:
                ea = float(np.max(np.abs(amp - ref)))
                eg = float(np.max(np.abs(grad - rgrad))) if len(grad) else 0.0
                if ea > ta or abs(val - rval) > tv or eg > tv:
                    nfail += 1
                    print("FAIL", cfg, "amp", ea, "val", abs(val - rval), "grad", eg, flush=True)
                    break
        except Exception as e:  # noqa: BLE001
            nfail += 1
            print("ERROR", cfg, str(e)[:300], flush=True)
        ncase += 1
    print(f"fuzz: {ncase} cases, {nfail} failures, {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()
