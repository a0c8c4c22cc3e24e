"""ADVICE r1 (high) race demonstration: plan [remap (unfused), sweep, sweep + fused remap, ...]
in an emulated world of 4 ranks on one GPU, with odd ranks held back by a device sleep
between receiving and unpacking each remap block (TQD_DEBUG_REMAP_DELAY_US).  Prints the
max error against the float64 oracle.  Runs with whichever binding / library is first on
PYTHONPATH: the current one, or round 1's (tools/r1_pkg, built from b2c9927 + the delay hook).

  PYTHONPATH=tools/r1_pkg:. python tools/race_demo.py     # round 1: expected to fail
  python tools/race_demo.py                               # round 2: matches the oracle
"""
import json
import os
import sys
import threading
import traceback

import numpy as np

sys.path.append(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))  # after PYTHONPATH: r1_pkg can shadow
import paper_2511_19291_b200 as tqd  # noqa: E402

import oracle  # noqa: E402  (test infrastructure: the reference result)
import workloads as W  # noqa: E402

os.environ.setdefault("TQD_DEBUG_REMAP_DELAY_US", "20000")
n, world = 12, 4
gates = [W.Gate("RX", (0,), (0.3,)), W.Gate("RX", (1,), (0.4,))]
gates += [W.Gate("CNOT", (q, q + 1)) for q in range(n - 1)] + W.hea(n, 2, 1, small=True)
terms = W.sum_z(n) + [(0, 3, 0.5)]
lid = tqd.tqd_loopback_id()
res, err = [None] * world, [None] * world


def worker(r):
    try:
        ctx = tqd.Context(world, r, 0, lid)
        st = tqd.State(ctx, n, "c128")
        st.set_option(tqd.OPT_TILE_QUBITS, 9)
        st.set_option(tqd.OPT_SMALL_MAX, 0)
        st.apply_circuit(gates)
        out = [st.adjoint_grad(terms)]
        st.rewind()
        out.append(st.adjoint_grad(terms))
        m = st.metrics()
        st.free()
        ctx.close()
        res[r] = (out, m)
    except Exception:
        err[r] = traceback.format_exc()


th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
for t in th:
    t.start()
for t in th:
    t.join(600)
rval, rgrad = oracle.adjoint(n, gates, terms)
worst = 0.0
for r in range(world):
    if err[r]:
        print(json.dumps({"rank": r, "error": err[r].splitlines()[-1]}))
        worst = float("inf")
        continue
    out, m = res[r]
    for val, grad in out:
        worst = max(worst, abs(val - rval), float(np.max(np.abs(grad - rgrad))))
    fr = m.get("fused_remaps", 0)
print(json.dumps({"library": tqd.LIB_PATH, "version": tqd.tqd_version(), "delay_us": os.environ["TQD_DEBUG_REMAP_DELAY_US"],
                  "max_err_vs_oracle": worst, "fused_remaps": fr, "pass_1e-10": worst < 1e-10}))
