import sys, time
sys.path.insert(0, '/root/repo')
import torch, numpy as np
import paper_2511_19291_b200 as tqd, workloads as W
torch.cuda.set_device(0)
ctx = tqd.Context.from_torch()
wl = W.config(1)
for sm in (10, 0):
    for graph in (0, 1):
        st = tqd.State(ctx, wl.n, wl.dtype)
        st.set_option(tqd.OPT_SMALL_MAX, sm)
        st.set_option(tqd.OPT_USE_GRAPH, graph)
        st.apply_circuit(wl.gates)
        v, g = st.adjoint_grad(wl.terms)
        for _ in range(5):
            st.rewind(); v, g = st.adjoint_grad(wl.terms)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            st.rewind(); v, g = st.adjoint_grad(wl.terms)
        e1.record(); torch.cuda.synchronize()
        m = st.metrics()
        print("small_max", sm, "graph", graph, "fwd+grad ms", e0.elapsed_time(e1) / 50, "sweeps", m["fwd_sweeps"], m["bwd_sweeps"], "E", v)
        st.free()
ctx.close()
