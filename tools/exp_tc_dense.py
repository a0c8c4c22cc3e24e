"""Tensor cores for a fused dense block at 30 qubits.

tcgen05.mma (kind::tf32, TMEM accumulators) applying a 6-qubit (64 x 64) dense
block to the 2^30-amplitude complex64 state (include/tqd.h tqd_debug_dense_block),
3xTF32 and 1xTF32, against the fused SIMT sweep of the bench (per gate: one 6-qubit
HEA layer = 6 RY + 6 RZ + 5 CNOT = 17 gates per block).  One JSON line per case."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2511_19291_b200 as tqd  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
rng = np.random.default_rng(0)
z = rng.normal(size=(64, 64)) + 1j * rng.normal(size=(64, 64))
q, r = np.linalg.qr(z)
U = q * (np.diag(r) / np.abs(np.diag(r)))
amps = 1 << n
rows = amps // 64
for prec in (3, 1):
    _, ms = tqd.tqd_debug_dense_block(n, U, None, precision=prec, iters=10)
    flops = 2.0 * rows * 128 * 128 * prec
    gbs = 16.0 * amps / (ms * 1e-3) / 1e9
    print(json.dumps({"case": f"tcgen05 dense 6-qubit block, {prec}xTF32", "n": n, "ms_per_block": round(ms, 4),
                      "ms_per_gate_hea17": round(ms / 17, 4), "hbm_GBps": round(gbs, 1),
                      "tensor_TFLOPs": round(flops / (ms * 1e-3) / 1e12, 1)}), flush=True)
