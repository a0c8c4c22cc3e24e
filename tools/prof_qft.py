"""One forward pass of X-prep + QFT (cfg-5 circuit family) for ncu captures of
the diagonal-block sweeps: python tools/prof_qft.py [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_19291_b200 as tqd  # noqa: E402
import workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
torch.cuda.set_device(0)
ctx = tqd.Context.from_torch()
st = tqd.State(ctx, n, "c64")
st.set_option(tqd.OPT_PROFILE, 1)
st.set_option(tqd.OPT_PRODUCT_PREFIX, 0)  # sweep the QFT (its basis-state input would make it a product prefix)
st.apply_circuit(W.basis_prep(n, 12345 % (1 << n)) + W.qft(n))
print(st.expval(W.sum_z(n))[:2], st.metrics()["fwd_sweeps"], st.metrics()["fwd_sweep_ms"])
st.free()
ctx.close()
