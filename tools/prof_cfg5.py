"""One forward pass of the cfg-5 circuit family (X-prep + QFT + HEA d4) at n
qubits for launch lists / ncu captures: python tools/prof_cfg5.py [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_19291_b200 as tqd  # noqa: E402
import workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 31
torch.cuda.set_device(0)
ctx = tqd.Context.from_torch()
wl = W.config(5, n_override=n)
st = tqd.State(ctx, n, "c64")
st.apply_circuit(wl.gates)
print(st.expval(wl.terms)[:2], st.metrics()["fwd_sweeps"])
st.free()
ctx.close()
