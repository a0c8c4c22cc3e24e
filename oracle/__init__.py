"""Test oracle: plain float64 CPU state-vector simulator (ctypes wrapper over oracle.c).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
package.  It shares no code with the CUDA path (``paper_2511_19291_b200``) and
never imports it; the CUDA path never imports this.

The arithmetic lives in ``oracle.c`` (see its header for the paper passages it
follows).  This file only marshals arguments.  Gate kinds are looked up by
NAME in this file's own table, so no constant is shared with the CUDA side.

Parity status per function:
  run / apply            pinned: kron-built unitaries (n <= 8), Bell, GHZ, QFT = DFT
  expval                 pinned: cos(theta) closed forms, Listing 1, GHZ correlators
  adjoint                pinned: parameter shift, finite differences, stored mode,
                         single-qubit closed forms (-sin theta)
  adjoint_stored         pinned: as adjoint (agreement <= 1e-9)
  param_shift            pinned: finite differences, closed forms
  finite_diff            pinned: closed forms
  clifford_expval / clifford_grad (clifford.c, stabilizer tableau; any n <= 63)
                         pinned: run + expval / adjoint on random Clifford circuits
                         (n <= 9), GHZ / Bell closed forms at n = 40
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

# This oracle's own gate-code table (oracle.h enum order).
KIND = {
    "I": 0, "X": 1, "Y": 2, "Z": 3, "H": 4, "S": 5, "SDG": 6, "T": 7, "TDG": 8,
    "CNOT": 9, "CZ": 10, "SWAP": 11, "MAT1": 12, "MAT2": 13,
    "RX": 14, "RY": 15, "RZ": 16, "U3": 17,
}
NPARAMS = {"RX": 1, "RY": 1, "RZ": 1, "U3": 3}


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C99, -O2, OpenMP)."""
    srcs = [os.path.join(_HERE, f) for f in ("oracle.c", "clifford.c")]
    if (not force and os.path.exists(_SO)
            and os.path.getmtime(_SO) >= max([os.path.getmtime(f) for f in srcs]
                                             + [os.path.getmtime(os.path.join(_HERE, "oracle.h"))])):
        return _SO
    tmp = _SO + f".tmp{os.getpid()}"
    cmd = ["gcc", "-std=gnu99", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, *srcs, "-lm"]
    subprocess.check_call(cmd)
    os.replace(tmp, _SO)
    return _SO


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_SO)
            i, d, p = ctypes.c_int, ctypes.c_double, ctypes.c_void_p
            for name, args in {
                "orc_run": [i, i, p, p, p, p, p],
                "orc_expval": [p, i, i, p, p, p, p],
                "orc_adjoint": [i, i, p, p, p, p, p, i, p, p, p, p, p],
                "orc_adjoint_stored": [i, i, p, p, p, p, p, i, p, p, p, p, p],
                "orc_param_shift": [i, i, p, p, p, p, p, i, p, p, p, p],
                "orc_finite_diff": [i, i, p, p, p, p, p, i, p, p, p, d, p],
                "orc_gate_matrix": [i, p, p, p],
                "orc_gate_dmatrix": [i, p, i, p],
                "orc_num_threads": [],
                "orc_gauss_sample": [p, i, d, ctypes.c_uint64, p],
                "orc_gauss_z": [p, i, d, ctypes.c_uint64, p],
                "orc_clifford_expval": [i, i, p, p, p, i, p, p, p, p],
                "orc_clifford_grad": [i, i, p, p, p, p, i, p, p, p, p, p],
                "orc_clifford_stabilizers": [i, i, p, p, p, p, p, p],
            }.items():
                f = getattr(lib, name)
                f.argtypes = args
                f.restype = ctypes.c_int
            for name in ("orc_uniform", "orc_normal"):
                f = getattr(lib, name)
                f.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
                f.restype = ctypes.c_double
            _lib = lib
    return _lib


def num_threads() -> int:
    return _load().orc_num_threads()


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class _Packed:
    """Circuit -> the parallel arrays oracle.h documents."""

    def __init__(self, gates):
        G = len(gates)
        self.G = G
        self.kinds = np.zeros(max(G, 1), dtype=np.int32)
        self.wires = np.zeros(2 * max(G, 1), dtype=np.int32)
        self.params = np.zeros(3 * max(G, 1), dtype=np.float64)
        self.mats = np.zeros(32 * max(G, 1), dtype=np.float64)
        self.trainable = np.zeros(max(G, 1), dtype=np.int32)
        for g, gate in enumerate(gates):
            self.kinds[g] = KIND[gate.name]
            for k, w in enumerate(gate.wires):
                self.wires[2 * g + k] = w
            for k, v in enumerate(gate.params):
                self.params[3 * g + k] = v
            if gate.matrix is not None:
                m = np.asarray(gate.matrix, dtype=np.complex128).reshape(-1)
                self.mats[32 * g:32 * g + 2 * m.size:2] = m.real
                self.mats[32 * g + 1:32 * g + 2 * m.size:2] = m.imag
            self.trainable[g] = 1 if (gate.trainable and gate.name in NPARAMS) else 0

    def args(self):
        return (self.G, _ptr(self.kinds), _ptr(self.wires), _ptr(self.params), _ptr(self.mats))

    def n_params(self):
        return int(sum(NPARAMS.get(_name, 0) for _name, t in zip(self._names(), self.trainable) if t))

    def _names(self):
        inv = {v: k for k, v in KIND.items()}
        return [inv[int(k)] for k in self.kinds[:self.G]]


def _terms(terms):
    T = len(terms)
    x = np.array([t[0] for t in terms] or [0], dtype=np.uint64)
    z = np.array([t[1] for t in terms] or [0], dtype=np.uint64)
    c = np.array([t[2] if len(t) > 2 else 1.0 for t in terms] or [0.0], dtype=np.float64)
    return T, x, z, c


def _check(rc, what):
    if rc != 0:
        raise ValueError(f"oracle {what} rejected its arguments")


def run(n: int, gates) -> np.ndarray:
    """psi = U_G ... U_1 |0..0>, canonical MSB-first order, complex128."""
    pk = _Packed(gates)
    psi = np.zeros(1 << n, dtype=np.complex128)
    _check(_load().orc_run(n, *pk.args(), _ptr(psi)), "run")
    return psi


def expval(psi: np.ndarray, n: int, terms) -> np.ndarray:
    """out[t] = c_t <psi|P_t|psi>; terms = [(x_mask, z_mask, coeff), ...]."""
    psi = np.ascontiguousarray(psi, dtype=np.complex128)
    T, x, z, c = _terms(terms)
    out = np.zeros(max(T, 1), dtype=np.float64)
    _check(_load().orc_expval(_ptr(psi), n, T, _ptr(x), _ptr(z), _ptr(c), _ptr(out)), "expval")
    return out[:T]


def _grad_call(fn, n, gates, terms, *extra, value=True):
    pk = _Packed(gates)
    T, x, z, c = _terms(terms)
    P = pk.n_params()
    grad = np.zeros(max(P, 1), dtype=np.float64)
    val = ctypes.c_double(0.0)
    args = [n, *pk.args(), _ptr(pk.trainable), T, _ptr(x), _ptr(z), _ptr(c)]
    if value:
        args.append(ctypes.byref(val))
    args.extend(extra)
    args.append(_ptr(grad))
    _check(fn(*args), fn.__name__)
    return (val.value, grad[:P]) if value else grad[:P]


def adjoint(n: int, gates, terms):
    """(E, dE/dtheta) by the invertible reverse sweep."""
    return _grad_call(_load().orc_adjoint, n, gates, terms)


def adjoint_stored(n: int, gates, terms):
    """(E, dE/dtheta) by stored-activation reverse mode (n <= 16)."""
    return _grad_call(_load().orc_adjoint_stored, n, gates, terms)


def param_shift(n: int, gates, terms):
    return _grad_call(_load().orc_param_shift, n, gates, terms, value=False)


def clifford_expval(n: int, gates, terms) -> np.ndarray:
    """out[t] = c_t <P_t> of a Clifford circuit by the stabilizer tableau (clifford.c;
    any n <= 63): exact values in {-c_t, 0, c_t}."""
    pk = _Packed(gates)
    T, x, z, c = _terms(terms)
    out = np.zeros(max(T, 1), dtype=np.float64)
    _check(_load().orc_clifford_expval(n, pk.G, _ptr(pk.kinds), _ptr(pk.wires), _ptr(pk.params), T, _ptr(x),
                                       _ptr(z), _ptr(c), _ptr(out)), "clifford_expval")
    return out[:T]


def clifford_stabilizers(n: int, gates):
    """The n stabilizer generators (x_mask, z_mask, sign) of the Clifford circuit's
    final state: sign * P |psi> = |psi>."""
    pk = _Packed(gates)
    x = np.zeros(n, dtype=np.uint64)
    z = np.zeros(n, dtype=np.uint64)
    sg = np.zeros(n, dtype=np.int32)
    _check(_load().orc_clifford_stabilizers(n, pk.G, _ptr(pk.kinds), _ptr(pk.wires), _ptr(pk.params), _ptr(x),
                                            _ptr(z), _ptr(sg)), "clifford_stabilizers")
    return [(int(x[k]), int(z[k]), int(sg[k])) for k in range(n)]


def clifford_grad(n: int, gates, terms):
    """(E, dE/dtheta) of a Clifford circuit (angles k pi/2): tableau + parameter shift."""
    pk = _Packed(gates)
    T, x, z, c = _terms(terms)
    P = pk.n_params()
    grad = np.zeros(max(P, 1), dtype=np.float64)
    val = ctypes.c_double(0.0)
    _check(_load().orc_clifford_grad(n, pk.G, _ptr(pk.kinds), _ptr(pk.wires), _ptr(pk.params), _ptr(pk.trainable),
                                     T, _ptr(x), _ptr(z), _ptr(c), ctypes.byref(val), _ptr(grad)), "clifford_grad")
    return val.value, grad[:P]


def finite_diff(n: int, gates, terms, eps: float = 1e-6):
    return _grad_call(_load().orc_finite_diff, n, gates, terms, ctypes.c_double(eps), value=False)


def gate_matrix(name: str, params=(), matrix=None) -> np.ndarray:
    p = np.zeros(3)
    p[:len(params)] = params
    m = np.zeros(32)
    if matrix is not None:
        mm = np.asarray(matrix, dtype=np.complex128).reshape(-1)
        m[0:2 * mm.size:2] = mm.real
        m[1:2 * mm.size:2] = mm.imag
    out = np.zeros(32)
    _check(_load().orc_gate_matrix(KIND[name], _ptr(p), _ptr(m), _ptr(out)), "gate_matrix")
    dim = 4 if name in ("CNOT", "CZ", "SWAP", "MAT2") else 2
    return (out[0:2 * dim * dim:2] + 1j * out[1:2 * dim * dim:2]).reshape(dim, dim)


# ---- shot noise, approximate (Gaussian) sampler ----------
def uniform(seed: int, k: int) -> float:
    return _load().orc_uniform(seed, k)


def normal(seed: int, i: int) -> float:
    return _load().orc_normal(seed, i)


def gauss_sample(psi: np.ndarray, n: int, shots: float, seed: int) -> np.ndarray:
    """y = shots p + sqrt(shots) D S z over the 2^n canonical outcomes."""
    psi = np.ascontiguousarray(psi, dtype=np.complex128)
    y = np.zeros(1 << n, dtype=np.float64)
    _check(_load().orc_gauss_sample(_ptr(psi), n, float(shots), seed, _ptr(y)), "gauss_sample")
    return y


def gauss_z(n: int, gates, shots: float, seed: int) -> np.ndarray:
    """Per-qubit <Z_q> estimates from the approximate shot sample of the circuit's state."""
    psi = run(n, gates)
    out = np.zeros(n, dtype=np.float64)
    _check(_load().orc_gauss_z(_ptr(psi), n, float(shots), seed, _ptr(out)), "gauss_z")
    return out
