#!/usr/bin/env python
"""Per-config measurements on ONE B200 (BASELINE.json configs).

For each workload: forward (|0> -> sweeps -> expval) and forward + adjoint
gradient (-> lambda = H psi -> reverse sweeps -> gradients) times, CUDA events on
the library stream around K replays of the recorded tape (tqd_state_rewind),
after W warm-up replays; per-kernel averages from the library's PROFILE mode
(a separate pass, so the step times above are not perturbed by per-launch
events).  One JSON line per case on stdout.

  cfg1   10q HEA d4 complex128, <Z0> + 80 gradients (latency: one-tile sweeps, a single CTA)
  cfg2   24q HEA d20 complex64, sum Z_i
  cfg3   30q HEA d20 complex64 (= bench.py), plus a tile-size sweep (--ksweep)
  cfg4   33q HEA d10 complex64 at P = 1 (128 GiB psi + lambda on one GPU)
  cfg5/8 the 2^33-amplitude per-GPU shard of cfg5 (36q over 8 GPUs): 33q
         X-prep + QFT + HEA d4 on one GPU (local sweeps only, no remaps);
         cfg5_8_sweep: the same with the product prefix off (the QFT swept)

  python tools/bench_configs.py [--cases cfg1,cfg2,...] [--steps K] [--warmup W] [--ksweep 9,10,11,12,13]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2511_19291_b200 as tqd  # noqa: E402
import workloads as W  # noqa: E402


def peak_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


GRAPH = 0


def run_case(ctx, name, wl, steps, warmup, tile=0, note="", prefix=2):
    stream = torch.cuda.current_stream()
    n, gates, terms = wl.n, wl.gates, wl.terms
    st = tqd.State(ctx, n, wl.dtype)
    st.set_option(tqd.OPT_PRODUCT_PREFIX, prefix)
    if tile:
        st.set_option(tqd.OPT_TILE_QUBITS, tile)
    if GRAPH:
        st.set_option(tqd.OPT_USE_GRAPH, 1)
    out = {"case": name, "workload": wl.name, "n_qubits": n, "dtype": wl.dtype, "gates": len(gates),
           "tile_k": tile or "default", "cuda_graph": GRAPH, "product_prefix": prefix, "note": note}
    try:
        st.apply_circuit(gates)

        def timed(fn, k):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(k):
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / k

        def fwd():
            st.rewind()
            st.expval(terms)

        res = {}

        def grad():
            st.rewind()
            res["vg"] = st.adjoint_grad(terms)

        grad()  # plans + uploads
        for _ in range(warmup):
            grad()
        out["fwd_grad_ms"] = timed(grad, steps)
        for _ in range(max(1, warmup // 2)):
            fwd()
        out["fwd_ms"] = timed(fwd, steps)
        # per-kernel averages (PROFILE mode: CUDA events around every launch)
        st.set_option(tqd.OPT_PROFILE, 1)
        grad()
        st.reset_metrics()
        grad()
        m = st.metrics()
        shard = (8 if wl.dtype == "c64" else 16) << n
        pk = peak_gbs()
        out["fwd_sweeps"], out["bwd_sweeps"] = m["fwd_sweeps"], m["bwd_sweeps"]
        # gates written as the product-state prefix / absorbed into the observable (not swept)
        out["gates_prefix"], out["gates_absorbed"] = m["gates_prefix"], m["gates_absorbed"]
        if m["fwd_sweeps"] and m["fwd_sweep_ms"] > 0:
            a = m["fwd_sweep_ms"] / m["fwd_sweeps"]
            out["fwd_sweep_avg_ms"] = round(a, 4)
            out["fwd_sweep_gbs"] = round(2 * shard / (a / 1e3) / 1e9, 1)
            out["fwd_sweep_frac"] = round(out["fwd_sweep_gbs"] / pk, 4)
        if m["bwd_sweeps"]:
            a = m["bwd_sweep_ms"] / m["bwd_sweeps"]
            out["bwd_sweep_avg_ms"] = round(a, 4)
            out["bwd_sweep_gbs"] = round(m["bwd_sweep_bytes"] / (m["bwd_sweep_ms"] / 1e3) / 1e9, 1)
            out["bwd_sweep_frac"] = round(out["bwd_sweep_gbs"] / pk, 4)
        out["other_ms"] = round(m["other_ms"], 3)
        out["launches_per_fwd_grad"] = m["kernel_launches"]
        out["peak_device_bytes"] = m["peak_device_bytes"]  # psi + lambda (+ staging at world > 1)
        out["peak_device_gib"] = round(m["peak_device_bytes"] / 2**30, 3)
        out["gamp_gates_per_s_fwd_grad"] = round(len(gates) * (1 << n) / (out["fwd_grad_ms"] / 1e3) / 1e9, 2)
        out["gamp_gates_per_s_fwd"] = round(len(gates) * (1 << n) / (out["fwd_ms"] / 1e3) / 1e9, 2)
        val, g = res["vg"]
        out["value_check"] = {"E": float(val), "n_grad": len(g)}
        out["peak_gbs"] = pk
    except Exception as e:  # report and continue with the next case
        out["error"] = str(e)[:300]
    finally:
        st.free()
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="cfg1,cfg2,cfg3,cfg4,cfg5_8")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--ksweep", default="", help="tile sizes k for a 30q cfg3 sweep, e.g. 9,10,11,12")
    ap.add_argument("--ksweep-qubits", type=int, default=30)
    ap.add_argument("--graph", action="store_true", help="TQD_OPT_USE_GRAPH = 1 (cached plans as CUDA graphs)")
    args = ap.parse_args()
    global GRAPH
    GRAPH = 1 if args.graph else 0
    torch.cuda.set_device(0)
    ctx = tqd.Context.from_torch()
    cases = [c for c in args.cases.split(",") if c]
    try:
        for c in cases:
            if c == "cfg1":
                run_case(ctx, c, W.config(1), max(args.steps, 20), max(args.warmup, 5),
                         note="10 qubits: the whole fwd + lambda seed + reverse sweep in ONE launch "
                              "(circuit_reg_kernel, one CTA), latency-bound")
            elif c == "cfg2":
                run_case(ctx, c, W.config(2), max(args.steps, 5), args.warmup,
                         note="128 MiB psi + 128 MiB lambda: partly L2-resident (126 MB L2)")
            elif c == "cfg3":
                run_case(ctx, c, W.config(3), args.steps, args.warmup)
            elif c == "cfg4":
                run_case(ctx, c, W.config(4), args.steps, args.warmup,
                         note="cfg4 at P = 1: 64 GiB psi + 64 GiB lambda on one B200")
            elif c == "cfg5_8":
                run_case(ctx, c, W.config(5, n_override=33), args.steps, args.warmup,
                         note="the per-GPU shard size of cfg5 (36q over 8 GPUs = 2^33 amplitudes per GPU): "
                              "local sweeps of the same circuit family, no remaps; X-prep + QFT + first "
                              "RY/RZ layer written as the product-state prefix")
            elif c == "cfg5_8_sweep":
                run_case(ctx, c, W.config(5, n_override=33), args.steps, args.warmup, prefix=0,
                         note="cfg5_8 with TQD_OPT_PRODUCT_PREFIX = 0: the QFT swept (diagonal-block stages)")
        for k in [int(x) for x in args.ksweep.split(",") if x]:
            run_case(ctx, f"ksweep_k{k}", W.config(3, n_override=args.ksweep_qubits), args.steps, args.warmup,
                     tile=k, note="tile-size sweep (SURVEY.md §8(d) cfg 3)")
    finally:
        ctx.close()


if __name__ == "__main__":
    main()
