"""Seeded synthetic workloads shared by the tests, bench.py and the oracle harness.

This module holds NO arithmetic of the method (no gate application, no
expectation value, no gradient): it only draws circuits and observables from
numpy's ``default_rng(seed)`` and describes them as plain records that both the
CUDA binding and the oracle wrapper translate themselves (by gate NAME).

Recipes:
  * ``hea(n, depth, seed)``: hardware-efficient ansatz of BASELINE.json configs
    (RY/RZ + CNOT ladder), reading R9: layer l = [RY(theta_{l,q}) for all q]
    [RZ(phi_{l,q}) for all q] [CNOT(q, (q+1) mod n) for all q] (ring, R8).
    Parameter index 2nl + q (RY), 2nl + n + q (RZ).  Angles U[0, 2pi) in
    parameter order (R10); ``small=True`` draws U[-0.3, 0.3] instead.
  * ``random_circuit(n, n_gates, seed)``: gate kind uniform over the ABI's
    gate set, distinct uniform wires, Haar MAT1/MAT2 (QR of complex Gaussian,
    column phases fixed), angles U[0, 2pi).
  * ``qft(n)``: textbook QFT (R13): for j: H(j); for k > j: CP(2pi/2^{k-j+1})
    on (k, j) as a diagonal MAT2; then qubit reversal by SWAPs.
  * ``basis_prep(n, x)``: X gates preparing |x> (MSB-first).
  * Observables are lists of (x_mask, z_mask, coeff); bit q <-> logical qubit q.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

ONE_QUBIT_FIXED = ("I", "X", "Y", "Z", "H", "S", "SDG", "T", "TDG")
TWO_QUBIT_FIXED = ("CNOT", "CZ", "SWAP")
PARAMETRIC = {"RX": 1, "RY": 1, "RZ": 1, "U3": 3}


@dataclass
class Gate:
    name: str
    wires: tuple
    params: tuple = ()
    matrix: Optional[np.ndarray] = None
    trainable: bool = True


@dataclass
class Workload:
    name: str
    n: int
    gates: list
    terms: list = field(default_factory=list)
    dtype: str = "c64"

    @property
    def n_params(self) -> int:
        return sum(PARAMETRIC.get(g.name, 0) for g in self.gates if g.trainable)


def haar_unitary(dim: int, rng: np.random.Generator) -> np.ndarray:
    z = (rng.standard_normal((dim, dim)) + 1j * rng.standard_normal((dim, dim))) / math.sqrt(2)
    q, r = np.linalg.qr(z)
    d = np.diag(r)
    return q * (d / np.abs(d))


def hea(n: int, depth: int, seed: int = 0, small: bool = False, ring: bool = True) -> list:
    rng = np.random.default_rng(seed)
    if small:
        ang = rng.uniform(-0.3, 0.3, size=2 * n * depth)
    else:
        ang = rng.uniform(0.0, 2 * math.pi, size=2 * n * depth)
    gates = []
    for layer in range(depth):
        base = 2 * n * layer
        for q in range(n):
            gates.append(Gate("RY", (q,), (float(ang[base + q]),)))
        for q in range(n):
            gates.append(Gate("RZ", (q,), (float(ang[base + n + q]),)))
        if n >= 2:
            last = n if (ring and n > 2) else n - 1
            for q in range(last):
                gates.append(Gate("CNOT", (q, (q + 1) % n)))
    return gates


def random_circuit(n: int, n_gates: int, seed: int = 0, kinds: Optional[Sequence[str]] = None,
                   small: bool = False) -> list:
    rng = np.random.default_rng(seed)
    if kinds is None:
        kinds = list(ONE_QUBIT_FIXED) + list(PARAMETRIC) + ["MAT1"]
        if n >= 2:
            kinds += list(TWO_QUBIT_FIXED) + ["MAT2"]
    gates = []
    for _ in range(n_gates):
        k = kinds[int(rng.integers(len(kinds)))]
        two = k in TWO_QUBIT_FIXED or k == "MAT2"
        wires = tuple(int(w) for w in rng.choice(n, size=2 if two else 1, replace=False))
        params = ()
        if k in PARAMETRIC:
            if small:
                params = tuple(float(v) for v in rng.uniform(-0.3, 0.3, size=PARAMETRIC[k]))
            else:
                params = tuple(float(v) for v in rng.uniform(0, 2 * math.pi, size=PARAMETRIC[k]))
        mat = None
        if k == "MAT1":
            mat = haar_unitary(2, rng)
        elif k == "MAT2":
            mat = haar_unitary(4, rng)
        gates.append(Gate(k, wires, params, mat, True))
    return gates


def diag_perm_tail(n: int, n_gates: int, seed: int = 0) -> list:
    """Random run of gates that are diagonal or permutations-with-phase (what
    tqd_adjoint_grad's observable absorption takes): X, Y, Z, S, T, trainable RZ,
    CNOT, CZ, SWAP, diagonal MAT2 (controlled phase), anti-diagonal MAT1 with
    random phases, controlled anti-diagonal MAT2 (control on either wire)."""
    rng = np.random.default_rng(seed)
    kinds = ["X", "Y", "Z", "S", "T", "RZ", "MAT1"]
    if n >= 2:
        kinds += ["CNOT", "CZ", "SWAP", "MAT2D", "MAT2C"]
    gates = []
    for _ in range(n_gates):
        k = kinds[int(rng.integers(len(kinds)))]
        two = k in ("CNOT", "CZ", "SWAP", "MAT2D", "MAT2C")
        wires = tuple(int(w) for w in rng.choice(n, size=2 if two else 1, replace=False))
        ph = np.exp(1j * rng.uniform(0, 2 * math.pi, size=4))
        if k == "RZ":
            gates.append(Gate("RZ", wires, (float(rng.uniform(0, 2 * math.pi)),), None, True))
        elif k == "MAT1":
            gates.append(Gate("MAT1", wires, (), np.array([[0, ph[0]], [ph[1], 0]], np.complex128), False))
        elif k == "MAT2D":
            gates.append(Gate("MAT2", wires, (), np.diag(ph).astype(np.complex128), False))
        elif k == "MAT2C":
            m = np.eye(4, dtype=np.complex128)
            if rng.integers(2):  # control = wires[0]: |1x> block anti-diagonal
                m[2:, 2:] = [[0, ph[0]], [ph[1], 0]]
            else:                # control = wires[1]: indices {1, 3} carry the anti-diagonal
                m[1, 1] = m[3, 3] = 0
                m[1, 3], m[3, 1] = ph[0], ph[1]
            gates.append(Gate("MAT2", wires, (), m, False))
        else:
            gates.append(Gate(k, wires))
    return gates


def cphase_matrix(phi: float) -> np.ndarray:
    return np.diag([1, 1, 1, np.exp(1j * phi)]).astype(np.complex128)


def qft(n: int, swaps: bool = True) -> list:
    gates = []
    for j in range(n):
        gates.append(Gate("H", (j,)))
        for k in range(j + 1, n):
            gates.append(Gate("MAT2", (k, j), (), cphase_matrix(2 * math.pi / 2 ** (k - j + 1)), False))
    if swaps:
        for j in range(n // 2):
            gates.append(Gate("SWAP", (j, n - 1 - j)))
    return gates


def basis_prep(n: int, x: int) -> list:
    return [Gate("X", (q,)) for q in range(n) if (x >> (n - 1 - q)) & 1]


def sum_z(n: int) -> list:
    return [(0, 1 << q, 1.0) for q in range(n)]


def random_z_terms(n: int, n_terms: int, seed: int) -> list:
    rng = np.random.default_rng(seed + 7919)
    out = []
    for _ in range(n_terms):
        z = 0
        for q in range(n):
            if rng.random() < 0.5:
                z |= 1 << q
        out.append((0, z, float(rng.standard_normal())))
    return out


def random_pauli_terms(n: int, n_terms: int, seed: int) -> list:
    rng = np.random.default_rng(seed + 104729)
    out = []
    for _ in range(n_terms):
        x = z = 0
        for q in range(n):
            p = int(rng.integers(4))
            if p in (1, 3):
                x |= 1 << q
            if p in (2, 3):
                z |= 1 << q
        out.append((x, z, float(rng.standard_normal())))
    return out


# --- BASELINE.json configs (reading R14 for cfg 5) ------------------------------
def config(idx: int, seed: int = 0, n_override: Optional[int] = None) -> Workload:
    if idx == 1:
        n = n_override or 10
        return Workload("cfg1_hea10_d4_c128", n, hea(n, 4, seed), [(0, 1, 1.0)], "c128")
    if idx == 2:
        n = n_override or 24
        return Workload("cfg2_hea24_d20_c64", n, hea(n, 20, seed), sum_z(n), "c64")
    if idx == 3:
        n = n_override or 30
        return Workload("cfg3_hea30_d20_c64", n, hea(n, 20, seed), sum_z(n), "c64")
    if idx == 4:
        n = n_override or 33
        return Workload("cfg4_hea33_d10_c64", n, hea(n, 10, seed), sum_z(n), "c64")
    if idx == 5:
        n = n_override or 36
        rng = np.random.default_rng(seed)
        x = int(rng.integers(1 << min(n, 62)))
        gates = basis_prep(n, x) + qft(n)
        for g in gates:
            g.trainable = False
        gates += hea(n, 4, seed)
        return Workload("cfg5_qft36_hea4_c64", n, gates, sum_z(n), "c64")
    raise ValueError(idx)
