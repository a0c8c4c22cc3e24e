"""Single-launch circuit kernels, register-layout (TQD_OPT_CIRCUIT_LAYOUT = 1) vs
gate-by-gate (0): device time per fwd + adjoint call (PROFILE-mode events) for HEA
depth 4 at 8 / 9 / 10 qubits, complex64 / complex128.  One JSON line per case."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_19291_b200 as tqd  # noqa: E402
import workloads as W  # noqa: E402

torch.cuda.set_device(0)
ctx = tqd.Context.from_torch()
K = 100
for n in (8, 9, 10):
    for dtype in ("c128", "c64"):
        gates = W.hea(n, 4, seed=n)
        terms = [(0, 1, 1.0)]
        row = {"n": n, "dtype": dtype, "gates": len(gates)}
        for layout in (1, 0):
            st = tqd.State(ctx, n, dtype)
            st.set_option(tqd.OPT_CIRCUIT_LAYOUT, layout)
            st.apply_circuit(gates)
            for _ in range(5):
                st.rewind()
                st.adjoint_grad(terms)
            st.set_option(tqd.OPT_PROFILE, 1)
            st.rewind()
            st.adjoint_grad(terms)
            st.reset_metrics()
            for _ in range(K):
                st.rewind()
                st.adjoint_grad(terms)
            m = st.metrics()
            row[f"layout{layout}_us"] = round((m["fwd_sweep_ms"] + m["bwd_sweep_ms"]) / K * 1e3, 2)
            row[f"layout{layout}_runs"] = m["circuit_layout_launches"] / K
            st.free()
        print(json.dumps(row), flush=True)
ctx.close()
