"""Batched workload of the paper's profiling section: a batch of
16 states, encoder RY(x_b) on every qubit (per-state inputs, trainable = input
gradients for Adam on the inputs), then a ladder ansatz of CNOT + RY blocks;
one forward + adjoint pass per step, H = sum Z_i.  Compares one batched state
against 16 single states run one after another.  Prints one JSON line.

    python tools/bench_batch.py [--qubits 20] [--batch 16] [--layers 10] [--steps 5]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_19291_b200 as tqd  # noqa: E402
import workloads as W  # noqa: E402


def ladder(n, layers, seed):
    """Fig. [unitary] building block: CNOT(q, q+1) then RY(theta) on q+1, ladder across the width."""
    rng = np.random.default_rng(seed)
    g = []
    for _ in range(layers):
        for q in range(n - 1):
            g.append(W.Gate("CNOT", (q, q + 1), (), None, True))
            g.append(W.Gate("RY", (q + 1,), (float(rng.uniform(0, 2 * np.pi)),), None, False))
    return g


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--qubits", type=int, default=20)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--layers", type=int, default=10)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--prefix", type=int, default=1, help="TQD_OPT_PRODUCT_PREFIX (1: encoder as the product state)")
    a = ap.parse_args()
    import torch
    n, B = a.qubits, a.batch
    x = np.random.default_rng(1).uniform(0, np.pi / 3, size=(n, B))  # PAPER.md:353 input range
    ans = ladder(n, a.layers, 2)
    terms = W.sum_z(n)
    ctx = tqd.Context(1, 0, 0)
    n_gates = B * (n + len(ans))

    # training-loop style: states live across steps; every step re-records the circuit
    # (new inputs in a real Adam loop) -> the plan is reused, values re-encoded
    stb = tqd.State(ctx, n, "c64", batch=B)
    sts = [tqd.State(ctx, n, "c64") for _ in range(B)]
    for s_ in [stb] + sts:
        s_.set_option(tqd.OPT_PRODUCT_PREFIX, a.prefix)

    def run_batched():
        stb.reset()
        for q in range(n):
            stb.apply_batch("RY", [q], x[q].reshape(B, 1), trainable=True)
        stb.apply_circuit(ans)
        return stb.adjoint_grad(terms)

    def run_single():
        out = []
        for b in range(B):
            sts[b].reset()
            sts[b].apply_circuit([W.Gate("RY", (q,), (float(x[q, b]),), None, True) for q in range(n)] + ans)
            out.append(sts[b].adjoint_grad(terms))
        return out

    res = {}
    for name, fn in (("batched", run_batched), ("sequential", run_single)):
        for _ in range(a.warmup):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(a.steps):
            fn()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / a.steps
        res[name] = {"ms_per_step": dt * 1e3, "Gamp_gates_per_s": n_gates * (1 << n) / dt / 1e9}
    vb, gb = run_batched()
    vs = run_single()
    check = max(abs(vb - sum(v for v, _ in vs)), 0.0)
    reused = stb.metrics()["plans_reused"]
    stb.free()
    for s1 in sts:
        s1.free()
    ctx.close()
    print(json.dumps({
        "workload": f"PAPER.md:251-254 ladder ansatz (CNOT + RY), {a.layers} layers, encoder RY(x_b) inputs trainable, "
                    f"batch {B}, {n} qubits, complex64, fwd + adjoint (input gradients) per step through the C ABI "
                    f"(reset + record + adjoint_grad; plan reused), host wall clock",
        "batched": res["batched"], "sequential_single_states": res["sequential"],
        "speedup": res["sequential"]["ms_per_step"] / res["batched"]["ms_per_step"],
        "value_check_abs_diff": check, "plans_reused": reused,
    }))


if __name__ == "__main__":
    main()
