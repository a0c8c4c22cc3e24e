#!/usr/bin/env python
"""bench.py -- fwd+adjoint-gradient throughput of the sharded state-vector path.

One STEP = one forward + adjoint-gradient pass of the BASELINE.json cfg-3
workload (hardware-efficient ansatz, RY/RZ + CNOT ring, depth 20, complex64,
observable sum_i Z_i): |0..0> -> all fused forward sweeps -> lambda = H psi ->
all fused adjoint sweeps -> gradient reduction -> value + 1200 gradients on the
host.  At N GPUs the state has 30 + log2(N) qubits sharded over the ranks
(weak scaling: 2^30 amplitudes per GPU).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (N > 1)

  --config 2|3|4 selects BASELINE.json configs[1..3] (24q d20 / 30q d20 / 33q d10);
  the default (3) is the headline.

value    = gate-amplitude updates per second of the whole job:
           (gates applied per step x 2^n) / (fwd+grad step time) -- the trailing
           gates absorbed into the Z observable are not counted -- device-timed with CUDA events
           on the library's stream, max over ranks, circuit + plan resident
           (tqd_state_rewind re-executes the recorded tape).
e2e      = the same metric through the public C ABI per step, as in a training
           loop (new angles every step): tqd_state_reset, tqd_apply_gate x G from
           host arrays, tqd_adjoint_grad (reuses the cached plan structure,
           rebuilds the op coefficients and uploads them host->device, runs,
           copies value + gradients device->host); wall clock between
           synchronised barriers.
forward  = the same for a forward-only pass (|0..0> -> sweeps -> <Z_i>), with the
           forward sweep's roofline fraction.
roofline = the dominant kernel (the fused adjoint sweep) from live CUDA-event
           timings of every launch: algorithmic bytes (4 x 8 B x 2^n_loc per
           launch: read + write psi and lambda; 2 x 8 B for the last reverse
           sweep, which only reads) / summed launch time, against
           MEASURED_PEAKS.json hbm_gbs.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "circuit fwd+grad time and gate-sweep HBM GB/s at 30/33/36 qubits, 1-8 B200"
UNIT = "Gamp-gates/s (fwd+grad)"
DEPTH = 20
BASE_QUBITS = 30
CPU_SAMPLE_QUBITS = 22   # oracle sample width for cpu_baseline (same ansatz, full circuit; ~12 s on 16 cores)
REF_SAMPLE_QUBITS = 19   # oracle width per --impl reference step


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", type=int, choices=[2, 3, 4], default=3,
                   help="BASELINE.json configs[i-1]: 2 = 24q depth 20, 3 = 30q depth 20 (default, the "
                        "headline), 4 = 33q depth 10 (fixed width: strong scaling over N)")
    p.add_argument("--qubits", type=int, default=0, help="override n (default per --config)")
    p.add_argument("--depth", type=int, default=0, help="override the depth (default per --config)")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--tile", type=int, default=0)
    p.add_argument("--no-absorb", action="store_true",
                   help="apply every gate (TQD_OPT_ABSORB_TAIL = 0) instead of absorbing the trailing "
                        "diagonal / permutation gates into the Z observable")
    return p.parse_args()


CONFIGS = {  # BASELINE.json configs: (base qubits, depth, weak scaling: + log2 N qubits)
    2: (24, 20, True),
    3: (30, 20, True),
    4: (33, 10, False),
}


def resolve(args, world):
    """(n, depth, scaling) of the run: the --config family, weak scaling adds log2 N qubits."""
    g = int(round(math.log2(world)))
    base, depth, weak = CONFIGS[args.config]
    n = args.qubits or (base + g if weak else base)
    return n, args.depth or depth, "weak" if (weak or args.qubits) else "strong"


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic():
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
        return d.get("adjoint_sweep", {}).get("dram_bytes_per_launch"), d
    except Exception:
        return None, None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.tmp = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.index)], stdout=self.tmp, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.tmp.flush()
        rows = []
        with open(self.tmp.name) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.tmp.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max((float(r[3]) for r in rows if r[3].replace(".", "").isdigit()), default=None)}


def oracle_fwd_grad_sample(n: int, depth: int, seed: int):
    """The float64 oracle (as it stands) on the full ansatz at width n: fwd + adjoint grad."""
    import oracle
    import workloads as W
    gates = W.hea(n, depth, seed)
    t0 = time.perf_counter()
    oracle.adjoint(n, gates, W.sum_z(n))
    dt = time.perf_counter() - t0
    return len(gates), dt


def cpu_baseline_line(depth, seed):
    import oracle
    oracle.build()
    G, dt = oracle_fwd_grad_sample(CPU_SAMPLE_QUBITS, depth, seed)
    units = G * (1 << CPU_SAMPLE_QUBITS)
    return {"value": units / dt / 1e9, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"float64 C oracle (OpenMP), full fwd+adjoint-grad of the same ansatz (HEA ring depth "
                      f"{depth}, sum Z_i) at n={CPU_SAMPLE_QUBITS} qubits ({G} gates, {dt:.1f} s); "
                      f"throughput in gate-amplitude updates per second",
            "seconds": dt}


def ref_config(args, world, n_sample):
    """The ours-arm workload this arm samples (same workload string and width), plus the sample."""
    import workloads as W
    n, depth, _ = resolve(args, world)
    G = len(W.hea(n, depth, args.seed))
    return {"workload": f"cfg{args.config}-family HEA ring depth {depth}, {n} qubits complex64, "
                        f"fwd + adjoint grad of sum Z_i ({G} gates)",
            "n_qubits": n, "depth": depth, "gates": G, "seed": args.seed,
            "sample": f"each step: the same ansatz at n={n_sample} qubits on the float64 oracle; "
                      f"throughput in the same unit (gate-amplitude updates per second)"}


def run_reference(args, world, rank):
    """--impl reference: the oracle on this box's host cores (rank 0 only)."""
    if rank != 0:
        return
    # torchrun sets OMP_NUM_THREADS=1 for every rank; rank 0 is the only worker here, so the
    # oracle gets the host's cores as at N=1 (libgomp reads this when liboracle.so loads).
    os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
    import oracle
    oracle.build()
    n = REF_SAMPLE_QUBITS
    _, depth, scaling = resolve(args, world)
    for _ in range(args.warmup):
        oracle_fwd_grad_sample(n, depth, args.seed)
    times = []
    G = 0
    for _ in range(args.steps):
        G, dt = oracle_fwd_grad_sample(n, depth, args.seed)
        times.append(dt)
    t = sum(times) / len(times)
    value = G * (1 << n) / t / 1e9
    cores = oracle.num_threads()
    sample = (f"float64 C oracle (OpenMP, {cores} threads), each step = full fwd+adjoint-grad of the "
              f"ansatz (HEA ring depth {depth}, sum Z_i) at n={n} qubits, {G} gates")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": ref_config(args, world, n),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    import torch
    import torch.distributed as dist
    import paper_2511_19291_b200 as tqd
    import workloads as W

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    g = int(round(math.log2(world)))
    assert 1 << g == world, "world size must be a power of two"
    n, depth, scaling = resolve(args, world)
    args.depth = depth
    gates = W.hea(n, args.depth, args.seed)
    terms = W.sum_z(n)
    G = len(gates)

    ctx = tqd.Context.from_torch()
    st = tqd.State(ctx, n, "c64")
    if args.tile:
        st.set_option(tqd.OPT_TILE_QUBITS, args.tile)
    st.set_option(tqd.OPT_PROFILE, 1)
    if args.no_absorb:
        st.set_option(tqd.OPT_ABSORB_TAIL, 0)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    # record once; first adjoint_grad plans + uploads, later steps replay (tqd_state_rewind)
    st.apply_circuit(gates)
    val, grad = st.adjoint_grad(terms)
    for _ in range(max(args.warmup - 1, 0)):
        st.rewind()
        val, grad = st.adjoint_grad(terms)
    st.reset_metrics()
    barrier()
    torch.cuda.synchronize()

    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.3)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        st.rewind()
        val, grad = st.adjoint_grad(terms)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1) / args.steps
    m = st.metrics()
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # the unit counts the gates the step APPLIES (forward), not the recorded ones: the
    # trailing gates absorbed into the Z observable are never applied nor un-applied
    g_applied = m["gates_applied"] // args.steps
    g_unapplied = m["gates_unapplied"] // args.steps
    g_absorbed = m["gates_absorbed"] // args.steps
    g_prefix = m["gates_prefix"] // args.steps
    units = g_applied * (1 << n)
    value = units / (ms / 1e3) / 1e9

    # forward only (|0..0> -> all fused forward sweeps -> <Z_i>): same unit, device-timed
    st.rewind()
    st.expval(terms)
    st.reset_metrics()
    barrier()
    torch.cuda.synchronize()
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.steps):
        st.rewind()
        st.expval(terms)
    f1.record(stream)
    torch.cuda.synchronize()
    fms = f0.elapsed_time(f1) / args.steps
    mf = st.metrics()
    if world > 1:
        t = torch.tensor([fms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        fms = float(t.item())
    f_applied = mf["gates_applied"] // args.steps

    # roofline of the dominant kernel (live CUDA-event timings of every launch)
    peak, peak_src = measured_peaks()
    fwd_avg = m["fwd_sweep_ms"] / max(m["fwd_sweeps"], 1)
    bwd_avg = m["bwd_sweep_ms"] / max(m["bwd_sweeps"], 1)
    shard = 8 << (n - g)
    # algorithmic bytes of all adjoint sweeps (the last reverse sweep stores nothing) / their time
    bwd_gbs = m["bwd_sweep_bytes"] / (m["bwd_sweep_ms"] / 1e3) / 1e9 if m["bwd_sweep_ms"] > 0 else 0.0
    fwd_gbs = 2 * shard / (fwd_avg / 1e3) / 1e9 if fwd_avg > 0 else 0.0
    dominant = "adjoint_sweep" if m["bwd_sweep_ms"] >= m["fwd_sweep_ms"] else "forward_sweep"
    traffic, _ = ncu_traffic()
    ach = bwd_gbs if dominant == "adjoint_sweep" else fwd_gbs
    roofline = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": traffic, "kernel": dominant,
                "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs, b.copy_)",
                "algorithmic_bytes_per_launch": (round(m["bwd_sweep_bytes"] / max(m["bwd_sweeps"], 1))
                                                 if dominant == "adjoint_sweep" else 2 * shard),
                "avg_launch_ms": round(bwd_avg if dominant == "adjoint_sweep" else fwd_avg, 4),
                "forward_sweep": {"achieved": round(fwd_gbs, 1), "frac": round(fwd_gbs / peak, 4),
                                  "launches_per_step": m["fwd_sweeps"] // args.steps,
                                  "avg_launch_ms": round(fwd_avg, 4)},
                "adjoint_sweep": {"achieved": round(bwd_gbs, 1), "frac": round(bwd_gbs / peak, 4),
                                  "launches_per_step": m["bwd_sweeps"] // args.steps,
                                  "avg_launch_ms": round(bwd_avg, 4)},
                "bytes_per_gate_per_amp_fwd": round(m["fwd_sweep_bytes"] / (m["gates_applied"] * (1 << (n - g))), 3)
                if m["gates_applied"] else None}
    kernel_ms = m["fwd_sweep_ms"] + m["bwd_sweep_ms"] + m["other_ms"] + m["a2a_ms"]
    f_avg = mf["fwd_sweep_ms"] / max(mf["fwd_sweeps"], 1)
    forward = {"ms_per_step": round(fms, 3), "value": round(f_applied * (1 << n) / (fms / 1e3) / 1e9, 3),
               "unit": "Gamp-gates/s (forward)", "gates_applied_per_step": f_applied,
               "sweeps_per_step": mf["fwd_sweeps"] // args.steps,
               "forward_sweep": {"achieved": round(2 * shard / (f_avg / 1e3) / 1e9, 1) if f_avg > 0 else None,
                                 "frac": round(2 * shard / (f_avg / 1e3) / 1e9 / peak, 4) if f_avg > 0 else None,
                                 "avg_launch_ms": round(f_avg, 4)}}

    # end to end through the public ABI with host buffers
    e2e = None
    if not args.no_e2e:
        # a training step: NEW angles every step (same ansatz structure), so the
        # cached plan is reused but its op coefficients are rebuilt on the host and
        # uploaded host->device inside the timed region (counted in h2d_bytes)
        step_gates = [W.hea(n, args.depth, args.seed + 1 + i) for i in range(args.steps)]
        st.reset()
        st.apply_circuit(W.hea(n, args.depth, args.seed + 1000))
        st.adjoint_grad(terms)  # warm: plan structure cached, as in a training loop
        st.reset_metrics()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(args.steps):
            st.reset()
            st.apply_circuit(step_gates[i])
            val, grad = st.adjoint_grad(terms)
        torch.cuda.synchronize()
        barrier()
        te = (time.perf_counter() - t0) / args.steps
        if world > 1:
            t = torch.tensor([te], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        me = st.metrics()
        e2e = {"value": units / te / 1e9, "unit": UNIT, "ms_per_step": te * 1e3,
               "h2d_bytes_per_step": me["h2d_bytes"] // args.steps,
               "d2h_bytes_per_step": me["d2h_bytes"] // args.steps}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_line(args.depth, args.seed)

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": scaling,
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": f"cfg{args.config}-family HEA ring depth {args.depth}, {n} qubits complex64, "
                                       f"fwd + adjoint grad of sum Z_i ({G} gates, {len(grad)} params)",
                           "n_qubits": n, "depth": args.depth, "gates": G, "params": len(grad),
                           "gates_applied_per_step": g_applied, "gates_unapplied_per_step": g_unapplied,
                           "unit_counts": "gates applied per step (recorded minus absorbed) x 2^n",
                           "state_dtype": "complex64 (fp32 arithmetic, fp64 reductions)",
                           "parallelism": f"state sharded over {world} rank(s) by {g} global qubit(s)",
                           "l2": f"inputs larger than L2: {shard * 2 / 2**30:.0f} GiB psi+lambda per GPU",
                           "gates_absorbed_per_step": g_absorbed,
                           "gates_in_product_prefix_per_step": g_prefix,
                           "product_prefix": "leading product-preserving gates written as one product state "
                                             "(counted in gates_applied; gradients from lambda's environments)",
                           "absorption": "trailing diagonal/permutation gates folded into the Z observable "
                                         "(Heisenberg picture; same value and gradients)" if not args.no_absorb
                                         else "off: every gate applied",
                           "seed": args.seed},
                "gpu_launches": int(m["kernel_launches"]),
                "roofline": roofline,
                "forward": forward,
                "cpu_baseline": cpu,
                "e2e": e2e,
                "clocks": clocks,
                "kernel_ms_per_step": round(kernel_ms / args.steps, 3),
                "value_check": {"E": val, "grad_l2": float(sum(x * x for x in grad)) ** 0.5},
                "library": tqd.tqd_version()}
        print(json.dumps(line), flush=True)
    st.free()
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
