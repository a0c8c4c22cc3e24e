"""cfg1 (10q HEA d4 complex128, <Z0> + 80 gradients): the single-launch circuit
kernel (TQD_OPT_CIRCUIT_MAX = 10) vs the staged sweeps (0).  Reports the kernel's
own device time (PROFILE-mode CUDA events around the launch(es)) and the per-call
time of rewind + tqd_adjoint_grad (events on the stream, includes the host round
trip of the value / gradient readback)."""
import json
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_19291_b200 as tqd  # noqa: E402
import workloads as W  # noqa: E402

torch.cuda.set_device(0)
ctx = tqd.Context.from_torch()
wl = W.config(1)
K = 200
for cmax, layout in ((10, 1), (10, 0), (0, 0)):
    st = tqd.State(ctx, wl.n, wl.dtype)
    st.set_option(tqd.OPT_CIRCUIT_MAX, cmax)
    st.set_option(tqd.OPT_CIRCUIT_LAYOUT, layout)
    st.apply_circuit(wl.gates)
    v, g = st.adjoint_grad(wl.terms)
    for _ in range(10):
        st.rewind()
        v, g = st.adjoint_grad(wl.terms)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K):
        st.rewind()
        v, g = st.adjoint_grad(wl.terms)
    e1.record()
    torch.cuda.synchronize()
    call_ms = e0.elapsed_time(e1) / K
    st.set_option(tqd.OPT_PROFILE, 1)
    st.rewind()
    st.adjoint_grad(wl.terms)
    st.reset_metrics()
    for _ in range(K):
        st.rewind()
        v, g = st.adjoint_grad(wl.terms)
    m = st.metrics()
    kern_us = (m["fwd_sweep_ms"] + m["bwd_sweep_ms"] + m["other_ms"]) / K * 1e3
    print(json.dumps({"case": "cfg1", "circuit_max": cmax, "path": ("single launch, register layout" if layout else "single launch, gate by gate") if cmax
                      else "staged sweeps", "layout_launches": m["circuit_layout_launches"] / K,
                      "launches_per_call": m["kernel_launches"] / K, "device_us_per_call": round(kern_us, 2),
                      "sweep_us": round((m["fwd_sweep_ms"] + m["bwd_sweep_ms"]) / K * 1e3, 2),
                      "call_ms": round(call_ms, 4), "E": v, "grad0": float(g[0])}), flush=True)
    st.free()
ctx.close()
