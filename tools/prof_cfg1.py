import sys; sys.path.insert(0, '.')
import torch, paper_2511_19291_b200 as tqd, workloads as W
torch.cuda.set_device(0)
ctx = tqd.Context.from_torch()
wl = W.config(1)
st = tqd.State(ctx, wl.n, wl.dtype)
st.apply_circuit(wl.gates)
v, g = st.adjoint_grad(wl.terms)
for _ in range(3):
    st.rewind(); v, g = st.adjoint_grad(wl.terms)
torch.cuda.synchronize()
print("ok", v)
