"""One fwd+grad pass of the bench workload (for ncu captures of the sweep kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_19291_b200 as tqd  # noqa: E402
import workloads as W  # noqa: E402

n = int(os.environ.get("TQD_PROF_N", "30"))
depth = int(os.environ.get("TQD_PROF_DEPTH", "20"))
ctx = tqd.Context(1, 0, 0)
st = tqd.State(ctx, n, "c64")
st.apply_circuit(W.hea(n, depth, 0))
val, grad = st.adjoint_grad(W.sum_z(n))
m = st.metrics()
print("E", val, "fwd_sweeps", m["fwd_sweeps"], "bwd_sweeps", m["bwd_sweeps"])
st.free()
ctx.close()
