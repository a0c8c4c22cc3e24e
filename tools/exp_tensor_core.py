#!/usr/bin/env python
"""SURVEY.md §8(f) rank 4 experiment: does a dense fused 2^m x 2^m block on tensor
cores ever beat the SIMT fused sweep for this path?

A fused block of gates on m qubits is one dense complex 2^m x 2^m matrix U.
Applying it to the state = one complex GEMM  Psi' = Psi_(2^(n-m) x 2^m) @ U^T
(the block's qubits placed on the low index bits), i.e. one HBM read + write of
the state, 8 * 2^m real flops per amplitude.  This script times that GEMM with
cuBLAS (torch.matmul on complex64: CGEMM, fp32 SIMT; with TF32 allowed: 1xTF32
tensor cores; the best a library GEMM can do for the contraction) at n = 30 and
reports, per block size m:
  - ms per application, effective GB/s (16 B per amplitude) and fraction of HBM,
  - the amplitude error of each variant against complex128, absolute and
    relative to the largest amplitude (the north-star complex64 amplitude
    tolerance 1e-5 is absolute on small states whose amplitudes are O(1), so
    the relative error is what decides),
  - the HEA gates a block of m qubits can hold per state sweep (one layer's
    RY + RZ on m qubits + the m - 1 ring CNOTs between them; the ring CNOT
    ladder stops a block from absorbing the next layer) vs the fused SIMT tile.
One JSON line per (m, mode) on stdout.  python tools/exp_tensor_core.py [--n 30]
"""
import argparse
import json

import torch


def haar(dim, gen):
    z = torch.complex(torch.randn(dim, dim, generator=gen, dtype=torch.float64),
                      torch.randn(dim, dim, generator=gen, dtype=torch.float64))
    q, r = torch.linalg.qr(z)
    d = torch.diagonal(r)
    return q * (d / d.abs())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--ms", default="2,3,4,5,6,7,8,9,10")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    n = args.n
    N = 1 << n
    gen = torch.Generator().manual_seed(0)
    psi = torch.randn(N, dtype=torch.complex64, device=dev)
    psi /= torch.linalg.vector_norm(psi)
    out = torch.empty_like(psi)
    # accuracy check on a 2^24 slice against complex128
    acc_rows = 1 << 24
    for m in [int(x) for x in args.ms.split(",")]:
        U64 = haar(1 << m, gen)
        Ut = U64.to(torch.complex64).t().contiguous().to(dev)
        A = psi.view(N >> m, 1 << m)
        O = out.view(N >> m, 1 << m)
        ref = (psi[:acc_rows].to(torch.complex128).view(-1, 1 << m) @ U64.t().to(dev))
        for mode in ("fp32", "tf32"):
            torch.backends.cuda.matmul.allow_tf32 = mode == "tf32"
            torch.matmul(A, Ut, out=O)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.reps):
                torch.matmul(A, Ut, out=O)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.reps
            err = (O.view(-1)[:acc_rows].to(torch.complex128).view(-1, 1 << m) - ref).abs().max().item()
            rel = err / ref.abs().max().item()
            gbs = 16 * N / (ms / 1e3) / 1e9
            tflops = 8 * (1 << m) * N / (ms / 1e3) / 1e12
            hea_gates = 2 * m + (m - 1)
            print(json.dumps({"n": n, "m": m, "mode": mode, "ms": round(ms, 3), "eff_gbs": round(gbs, 1),
                              "tflops": round(tflops, 1), "max_abs_err_vs_c128": err, "rel_err_vs_c128": rel,
                              "meets_c64_amp_tol_1e-5_at_unit_scale": rel <= 1e-5,
                              "hea_gates_per_sweep": hea_gates,
                              "ms_per_hea_gate": round(ms / hea_gates, 4)}), flush=True)
    torch.backends.cuda.matmul.allow_tf32 = False


if __name__ == "__main__":
    main()
