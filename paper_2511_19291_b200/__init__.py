"""Python binding of libtqd.so (include/tqd.h): argument marshalling only.

Every step of the forward / expectation / adjoint path runs in the library's
CUDA kernels (sm_100a) and NCCL; this module only converts Python arguments to
the C ABI and raises on error.  There is no CPU fallback: if the library is
missing and cannot be built, import of the binding fails loudly.

Raw ABI names are exposed one-to-one (``tqd_state_init`` ...); the small
``Context`` / ``State`` classes below wrap them for tests and bench.py.
PyTorch is used only for plumbing: the current CUDA stream and, for world > 1,
broadcasting the NCCL unique id over ``torch.distributed``.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# TQD_LIB: another in-tree build of the same library (kernel experiment variants, tools/build_variant.sh)
LIB_PATH = os.environ.get("TQD_LIB") or os.path.join(_HERE, "libtqd.so")

# this binding's own copy of the tqd_gate enum (include/tqd.h)
GATES = {
    "I": 0, "X": 1, "Y": 2, "Z": 3, "H": 4, "S": 5, "SDG": 6, "T": 7, "TDG": 8,
    "CNOT": 9, "CZ": 10, "SWAP": 11, "MAT1": 12, "MAT2": 13,
    "RX": 14, "RY": 15, "RZ": 16, "U3": 17,
}
C64, C128 = 0, 1
OPT_TILE_QUBITS, OPT_SMALL_MAX, OPT_PROFILE, OPT_GRID_CTAS, OPT_USE_GRAPH, OPT_FUSED_REMAP, OPT_ABSORB_TAIL, \
    OPT_STAGING_BYTES, OPT_CIRCUIT_MAX, OPT_PRODUCT_PREFIX, OPT_CIRCUIT_LAYOUT = 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10
ERRORS = {0: "TQD_OK", -1: "TQD_ERR_ARG", -2: "TQD_ERR_QUBITS", -3: "TQD_ERR_WORLD",
          -4: "TQD_ERR_NOT_UNITARY", -5: "TQD_ERR_OOM", -6: "TQD_ERR_CUDA", -7: "TQD_ERR_NCCL",
          -8: "TQD_ERR_UNSUPPORTED", -9: "TQD_ERR_STATE"}


class TqdError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class Metrics(ctypes.Structure):
    _fields_ = [
        ("fwd_sweeps", ctypes.c_uint64), ("bwd_sweeps", ctypes.c_uint64), ("remaps", ctypes.c_uint64),
        ("gates_applied", ctypes.c_uint64), ("gates_unapplied", ctypes.c_uint64),
        ("hbm_bytes", ctypes.c_uint64), ("a2a_bytes", ctypes.c_uint64),
        ("fwd_sweep_ms", ctypes.c_double), ("bwd_sweep_ms", ctypes.c_double),
        ("other_ms", ctypes.c_double), ("a2a_ms", ctypes.c_double),
        ("fwd_sweep_bytes", ctypes.c_uint64), ("bwd_sweep_bytes", ctypes.c_uint64),
        ("peak_device_bytes", ctypes.c_uint64), ("kernel_launches", ctypes.c_uint64),
        ("h2d_bytes", ctypes.c_uint64), ("d2h_bytes", ctypes.c_uint64), ("fused_remaps", ctypes.c_uint64),
        ("plans_reused", ctypes.c_uint64), ("gates_absorbed", ctypes.c_uint64),
        ("gates_prefix", ctypes.c_uint64), ("circuit_layout_launches", ctypes.c_uint64),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lock = threading.Lock()
_lib = None

_P = ctypes.c_void_p
_SIG = {
    "tqd_nccl_unique_id": [_P],
    "tqd_loopback_id": [_P],
    "tqd_ctx_create": [ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, _P, ctypes.POINTER(_P)],
    "tqd_ctx_destroy": [_P],
    "tqd_state_bytes": [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)],
    "tqd_state_init": [_P, ctypes.c_int, ctypes.c_int, _P, ctypes.c_size_t, ctypes.POINTER(_P)],
    "tqd_state_init_batch": [_P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)],
    "tqd_apply_gate_batch": [_P, ctypes.c_int, _P, ctypes.c_int, _P, ctypes.c_int],
    "tqd_sample": [_P, ctypes.c_uint64, ctypes.c_uint64, _P],
    "tqd_sample_gaussian_z": [_P, ctypes.c_double, ctypes.c_uint64, _P],
    "tqd_adjoint_grad_gaussian": [_P, ctypes.c_double, ctypes.c_uint64, _P, ctypes.POINTER(ctypes.c_double), _P,
                                  ctypes.c_int],
    "tqd_state_reset": [_P],
    "tqd_state_rewind": [_P],
    "tqd_state_free": [_P],
    "tqd_state_set_option": [_P, ctypes.c_int, ctypes.c_int64],
    "tqd_apply_gate": [_P, ctypes.c_int, _P, ctypes.c_int, _P, _P, ctypes.c_int],
    "tqd_apply_circuit": [_P, ctypes.c_int, _P, _P, _P, _P, _P],
    "tqd_num_params": [_P, ctypes.POINTER(ctypes.c_int)],
    "tqd_state_info": [_P, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)],
    "tqd_expval": [_P, ctypes.c_int, _P, _P, _P, _P],
    "tqd_adjoint_grad": [_P, ctypes.c_int, _P, _P, _P, ctypes.POINTER(ctypes.c_double), _P, ctypes.c_int],
    "tqd_get_amplitudes": [_P, ctypes.c_uint64, ctypes.c_uint64, _P],
    "tqd_get_metrics": [_P, ctypes.POINTER(Metrics)],
    "tqd_reset_metrics": [_P],
    "tqd_debug_plan": [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                       _P, _P, _P, _P, _P, ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)],
    "tqd_debug_remap_schedule": [ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, _P, _P, _P],
    "tqd_debug_absorb": [ctypes.c_int, ctypes.c_int, _P, _P, _P, _P, _P, ctypes.c_int, _P, _P, _P, _P],
    "tqd_debug_dense_block": [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, _P, _P, ctypes.c_int,
                              ctypes.POINTER(ctypes.c_double)],
}
EXPORTS = list(_SIG) + ["tqd_last_error", "tqd_version"]


def lib():
    """Load libtqd.so (building it in-tree with nvcc if it is missing or stale)."""
    global _lib
    with _lock:
        if _lib is None:
            from . import build as _build
            if LIB_PATH == _build.SO and not _build.up_to_date():
                _build.build()
            L = ctypes.CDLL(LIB_PATH)
            for name, args in _SIG.items():
                f = getattr(L, name)
                f.argtypes = args
                f.restype = ctypes.c_int
            L.tqd_last_error.argtypes = []
            L.tqd_last_error.restype = ctypes.c_char_p
            L.tqd_version.argtypes = []
            L.tqd_version.restype = ctypes.c_char_p
            _lib = L
    return _lib


def _call(name, *args):
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        raise TqdError(rc, lib().tqd_last_error().decode())
    return rc


def _arr(a, dtype):
    return np.ascontiguousarray(np.asarray(a, dtype=dtype))


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


# ---- raw ABI (same names as include/tqd.h) ---------------------------------------
def tqd_version() -> str:
    return lib().tqd_version().decode()


def tqd_loopback_id() -> bytes:
    """128-byte id of an in-process loopback world (W ranks on one device, one thread each)."""
    buf = ctypes.create_string_buffer(128)
    _call("tqd_loopback_id", ctypes.cast(buf, _P))
    return buf.raw


def tqd_nccl_unique_id() -> bytes:
    buf = (ctypes.c_char * 128)()
    _call("tqd_nccl_unique_id", ctypes.cast(buf, _P))
    return bytes(buf)


def tqd_ctx_create(world: int, rank: int, device: int, nccl_id: bytes | None, stream: int | None):
    out = _P()
    idbuf = (ctypes.c_char * 128).from_buffer_copy(nccl_id) if nccl_id else None
    _call("tqd_ctx_create", world, rank, device, ctypes.cast(idbuf, _P) if idbuf is not None else None,
          _P(stream) if stream else None, ctypes.byref(out))
    return out


def tqd_ctx_destroy(ctx):
    _call("tqd_ctx_destroy", ctx)


def tqd_state_bytes(n: int, dtype: int, world: int, with_adjoint: int) -> int:
    out = ctypes.c_size_t()
    _call("tqd_state_bytes", n, dtype, world, with_adjoint, ctypes.byref(out))
    return out.value


def tqd_state_init(ctx, n: int, dtype: int, dev_buf: int | None = None, buf_bytes: int = 0):
    out = _P()
    _call("tqd_state_init", ctx, n, dtype, _P(dev_buf) if dev_buf else None, buf_bytes, ctypes.byref(out))
    return out


def tqd_state_reset(st):
    _call("tqd_state_reset", st)


def tqd_state_rewind(st):
    _call("tqd_state_rewind", st)


def tqd_state_free(st):
    _call("tqd_state_free", st)


def tqd_state_set_option(st, opt: int, value: int):
    _call("tqd_state_set_option", st, opt, int(value))


def _gate_code(gate) -> int:
    g = GATES[gate] if isinstance(gate, str) else int(gate)
    if not 0 <= g < len(GATES):
        raise TqdError(-1, f"unknown gate kind {gate!r}")
    return g


def tqd_apply_gate(st, gate, wires, params=(), matrix=None, trainable=True):
    # the C call takes no array lengths: check what it will read (errors, not over-reads)
    g = _gate_code(gate)
    w = _arr(wires, np.int32)
    if w.size != _ARITY[g]:
        raise TqdError(-1, f"gate {gate}: {w.size} wires, needs {_ARITY[g]}")
    pp = np.asarray(params, dtype=np.float64).reshape(-1)
    if pp.size != _NPARAMS[g]:
        raise TqdError(-1, f"gate {gate}: {pp.size} params, needs {_NPARAMS[g]}")
    p = _arr(pp, np.float64) if pp.size else None
    m = None
    if g in (GATES["MAT1"], GATES["MAT2"]):
        if matrix is None:
            raise TqdError(-1, f"gate {gate}: matrix required")
        mm = np.asarray(matrix, dtype=np.complex128).reshape(-1)
        if mm.size != (4 if g == GATES["MAT1"] else 16):
            raise TqdError(-1, f"gate {gate}: matrix has {mm.size} entries")
        m = np.empty(2 * mm.size, dtype=np.float64)
        m[0::2], m[1::2] = mm.real, mm.imag
    _call("tqd_apply_gate", st, g, _ptr(w), int(w.size), _ptr(p), _ptr(m), 1 if trainable else 0)


def tqd_apply_circuit(st, gates):
    """Record a whole gate list with one C call (same result as tqd_apply_gate per gate)."""
    if not len(gates):
        return
    kinds, wires, params, mats, tr = _gate_arrays(gates)
    _call("tqd_apply_circuit", st, len(gates), _ptr(kinds), _ptr(wires), _ptr(params), _ptr(mats), _ptr(tr))


def tqd_state_init_batch(ctx, n: int, dtype: int, batch: int):
    out = _P()
    _call("tqd_state_init_batch", ctx, n, dtype, batch, ctypes.byref(out))
    return out


def tqd_state_info(st):
    """(n_qubits, batch, dtype) of a state handle."""
    n, b, d = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _call("tqd_state_info", st, ctypes.byref(n), ctypes.byref(b), ctypes.byref(d))
    return n.value, b.value, d.value


def tqd_apply_gate_batch(st, gate, wires, params, trainable=True):
    """params: (batch, n_params_of_gate) per-state parameters."""
    g = _gate_code(gate)
    w = _arr(wires, np.int32)
    p = _arr(np.asarray(params, dtype=np.float64).reshape(-1), np.float64)
    batch = tqd_state_info(st)[1]
    if w.size != 1:
        raise TqdError(-1, "batched gates act on one wire")
    if p.size != batch * max(int(_NPARAMS[g]), 1):
        raise TqdError(-1, f"params: {p.size} values for batch {batch} x {_NPARAMS[g]} parameters")
    _call("tqd_apply_gate_batch", st, g, _ptr(w), int(w.size), _ptr(p), 1 if trainable else 0)


def tqd_num_params(st) -> int:
    out = ctypes.c_int()
    _call("tqd_num_params", st, ctypes.byref(out))
    return out.value


def _terms(terms):
    x = _arr([t[0] for t in terms] or [0], np.uint64)
    z = _arr([t[1] for t in terms] or [0], np.uint64)
    c = _arr([t[2] if len(t) > 2 else 1.0 for t in terms] or [0.0], np.float64)
    return len(terms), x, z, c


def tqd_expval(st, terms, batch: int | None = None) -> np.ndarray:
    T, x, z, c = _terms(terms)
    hb = tqd_state_info(st)[1]
    if batch is not None and batch != hb:
        raise TqdError(-1, f"batch {batch} != the state's batch {hb}")
    batch = hb
    out = np.zeros(max(T * batch, 1), dtype=np.float64)
    _call("tqd_expval", st, T, _ptr(x), _ptr(z), _ptr(c), _ptr(out))
    return out[:T * batch] if batch == 1 else out[:T * batch].reshape(batch, T)


def tqd_adjoint_grad(st, terms, n_grad: int | None = None, coeff=None):
    """coeff: optional (batch, n_terms) VJP weights for a batch (default: the terms' own)."""
    T, x, z, c = _terms(terms)
    batch = tqd_state_info(st)[1]
    if coeff is not None:
        c = _arr(np.asarray(coeff, dtype=np.float64).reshape(-1), np.float64)
        if c.size != batch * T:
            raise TqdError(-1, f"coeff: {c.size} values for batch {batch} x {T} terms")
    elif batch > 1:
        c = _arr(np.tile(c[:T], batch), np.float64)  # every element uses the terms' own coefficients
    if n_grad is None:
        n_grad = tqd_num_params(st)
    g = np.zeros(max(n_grad, 1), dtype=np.float64)
    val = ctypes.c_double()
    _call("tqd_adjoint_grad", st, T, _ptr(x), _ptr(z), _ptr(c), ctypes.byref(val), _ptr(g), n_grad)
    return val.value, g[:n_grad]


def tqd_sample(st, shots: int, seed: int, batch: int | None = None) -> np.ndarray:
    batch = tqd_state_info(st)[1]
    out = np.zeros(max(batch * shots, 1), dtype=np.uint64)
    _call("tqd_sample", st, int(shots), int(seed), _ptr(out))
    out = out[:batch * shots]
    return out if batch == 1 else out.reshape(batch, shots)


def tqd_sample_gaussian_z(st, n: int | None, shots: float, seed: int, batch: int | None = None) -> np.ndarray:
    n, batch, _ = tqd_state_info(st)
    out = np.zeros(batch * n, dtype=np.float64)
    _call("tqd_sample_gaussian_z", st, float(shots), int(seed), _ptr(out))
    return out if batch == 1 else out.reshape(batch, n)


def tqd_adjoint_grad_gaussian(st, shots: float, seed: int, coeff=None, n_grad: int | None = None):
    if n_grad is None:
        n_grad = tqd_num_params(st)
    n, batch, _ = tqd_state_info(st)
    c = None if coeff is None else _arr(np.asarray(coeff, dtype=np.float64).reshape(-1), np.float64)
    if c is not None and c.size != batch * n:
        raise TqdError(-1, f"coeff: {c.size} values for batch {batch} x {n} qubits")
    g = np.zeros(max(n_grad, 1), dtype=np.float64)
    val = ctypes.c_double()
    _call("tqd_adjoint_grad_gaussian", st, float(shots), int(seed), _ptr(c), ctypes.byref(val), _ptr(g), n_grad)
    return val.value, g[:n_grad]


def tqd_get_amplitudes(st, first: int, count: int, dtype: int | None = None) -> np.ndarray:
    dtype = tqd_state_info(st)[2]
    out = np.zeros(count, dtype=np.complex128 if dtype == C128 else np.complex64)
    _call("tqd_get_amplitudes", st, first, count, _ptr(out))
    return out


def tqd_get_metrics(st) -> dict:
    m = Metrics()
    _call("tqd_get_metrics", st, ctypes.byref(m))
    return m.as_dict()


def tqd_reset_metrics(st):
    _call("tqd_reset_metrics", st)


def tqd_last_error() -> str:
    return lib().tqd_last_error().decode()


_ARITY = np.array([2 if k in ("CNOT", "CZ", "SWAP", "MAT2") else 1
                   for k in sorted(GATES, key=GATES.get)], np.int32)
_NPARAMS = np.array([{"RX": 1, "RY": 1, "RZ": 1, "U3": 3}.get(k, 0)
                     for k in sorted(GATES, key=GATES.get)], np.int32)


def _gate_arrays(gates):
    G = len(gates)
    m = max(G, 1)
    kinds = np.zeros(m, np.int32)
    wires = np.zeros((m, 2), np.int32)
    params = np.zeros((m, 3), np.float64)
    mats = np.zeros(32 * m, np.float64)
    tr = np.zeros(m, np.int32)
    if G:
        kinds[:G] = [GATES[g.name] for g in gates]
        wires[:G] = [(tuple(g.wires) + (0, 0))[:2] for g in gates]
        params[:G] = [(tuple(g.params) + (0.0, 0.0, 0.0))[:3] for g in gates]
        tr[:G] = [1 if g.trainable else 0 for g in gates]
    wires, params = wires.reshape(-1), params.reshape(-1)
    if G:  # the packed arrays carry no counts: check them as tqd_apply_gate does (errors, not padding)
        nw = np.fromiter((len(g.wires) for g in gates), np.int32, G)
        npar = np.fromiter((len(g.params) for g in gates), np.int32, G)
        kk = np.clip(kinds[:G], 0, len(_ARITY) - 1)
        bad = np.flatnonzero((nw != _ARITY[kk]) | (npar < _NPARAMS[kk]) | (npar > 3))
        if bad.size:
            i = int(bad[0])
            raise TqdError(-1, f"gate {i} ({gates[i].name}): {len(gates[i].wires)} wires / "
                               f"{len(gates[i].params)} params do not fit the gate")
    for i, g in enumerate(gates):
        if g.matrix is not None:
            mm = np.asarray(g.matrix, np.complex128).reshape(-1)
            mats[32 * i:32 * i + 2 * mm.size:2] = mm.real
            mats[32 * i + 1:32 * i + 2 * mm.size:2] = mm.imag
    return kinds, wires, params, mats, tr


def tqd_debug_plan(n: int, gates, world: int = 1, k: int = 12, small_max: int = 8, c128: bool = False) -> dict:
    """Planner diagnostic (host only, no GPU): stages of `gates` as a dict."""
    import json
    G = len(gates)
    kinds, wires, params, mats, tr = _gate_arrays(gates)
    need = ctypes.c_size_t(0)
    cap = 1 << 16
    while True:
        buf = ctypes.create_string_buffer(cap)
        rc = lib().tqd_debug_plan(n, world, k, small_max, 1 if c128 else 0, G, _ptr(kinds), _ptr(wires),
                                  _ptr(params), _ptr(mats), _ptr(tr), buf, cap, ctypes.byref(need))
        if rc == 0:
            return json.loads(buf.value.decode())
        if need.value > cap:
            cap = need.value
            continue
        raise TqdError(rc, tqd_last_error())


def tqd_debug_absorb(n: int, gates, z_masks):
    """Observable absorption of tqd_adjoint_grad (host only, no GPU):
    (tail_begin, z_out, sign_out) -- see include/tqd.h tqd_debug_absorb."""
    kinds, wires, params, mats, tr = _gate_arrays(gates)
    T = len(z_masks)
    zin = np.array(list(z_masks) or [0], np.uint64)
    zout = np.zeros(max(T, 1), np.uint64)
    sg = np.zeros(max(T, 1), np.float64)
    tb = ctypes.c_int(0)
    _call("tqd_debug_absorb", n, len(gates), _ptr(kinds), _ptr(wires), _ptr(params), _ptr(mats), _ptr(tr), T,
          _ptr(zin), _ptr(zout), _ptr(sg), ctypes.byref(tb))
    return tb.value, [int(v) for v in zout[:T]], sg[:T].copy()


def tqd_debug_dense_block(n: int, U, psi=None, precision: int = 3, iters: int = 0, device: int = 0):
    """Tensor-core experiment: U (2^6 x 2^6 complex) on the 6 lowest bits of a 2^n complex64
    state by tcgen05.mma (include/tqd.h).  Returns (result or None, ms per timed application)."""
    U = np.asarray(U, np.complex128)
    m = int(round(np.log2(U.shape[0])))
    if U.shape != (1 << m, 1 << m):
        raise TqdError(-1, "U must be square 2^m x 2^m")
    uu = np.empty(2 * U.size, np.float64)
    uu[0::2], uu[1::2] = U.real.reshape(-1), U.imag.reshape(-1)
    pin = None if psi is None else np.ascontiguousarray(np.asarray(psi, np.complex64))
    if pin is not None and pin.size != (1 << n):
        raise TqdError(-1, "psi must have 2^n amplitudes")
    out = None if psi is None else np.zeros(1 << n, np.complex64)
    ms = ctypes.c_double(0.0)
    _call("tqd_debug_dense_block", device, n, m, precision, _ptr(uu), _ptr(pin), _ptr(out), iters, ctypes.byref(ms))
    return out, ms.value


def tqd_debug_remap_schedule(rank: int, n_loc: int, gpos, lpos):
    """(peer[b], recv_block[b]) for every send block b of one rank's remap (host only)."""
    m = len(gpos)
    g = _arr(gpos or [0], np.int32)
    l_ = _arr(lpos or [0], np.int32)
    peer = np.zeros(1 << m, np.int32)
    recv = np.zeros(1 << m, np.int32)
    _call("tqd_debug_remap_schedule", rank, n_loc, m, _ptr(g), _ptr(l_), _ptr(peer), _ptr(recv))
    return peer, recv


# ---- convenience wrappers ----------------------------------------------------
class Context:
    """One per process = one GPU.  world > 1 bootstraps NCCL over torch.distributed."""

    def __init__(self, world: int = 1, rank: int = 0, device: int = 0, nccl_id: bytes | None = None,
                 stream: int | None = None):
        self.world, self.rank, self.device = world, rank, device
        self.handle = tqd_ctx_create(world, rank, device, nccl_id, stream)

    @classmethod
    def from_torch(cls, use_current_stream: bool = True):
        """Context for this rank: RANK / WORLD_SIZE / LOCAL_RANK from torch.distributed / env."""
        import torch
        import torch.distributed as dist
        world = dist.get_world_size() if dist.is_initialized() else 1
        rank = dist.get_rank() if dist.is_initialized() else 0
        device = int(os.environ.get("LOCAL_RANK", 0)) if world > 1 else torch.cuda.current_device()
        torch.cuda.set_device(device)
        nid = None
        if world > 1:
            obj = [tqd_nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            nid = obj[0]
        stream = torch.cuda.current_stream(device).cuda_stream if use_current_stream else None
        return cls(world, rank, device, nid, stream)

    def close(self):
        if self.handle:
            tqd_ctx_destroy(self.handle)
            self.handle = None


class State:
    def __init__(self, ctx: Context, n: int, dtype: str = "c64", dev_buf: int | None = None, buf_bytes: int = 0,
                 batch: int = 1):
        self.ctx, self.n, self.batch = ctx, n, batch
        self.dtype = C128 if dtype in ("c128", C128) else C64
        if batch == 1:
            self.handle = tqd_state_init(ctx.handle, n, self.dtype, dev_buf, buf_bytes)
        else:
            self.handle = tqd_state_init_batch(ctx.handle, n, self.dtype, batch)

    def set_option(self, opt: int, value: int):
        tqd_state_set_option(self.handle, opt, value)

    def reset(self):
        tqd_state_reset(self.handle)

    def rewind(self):
        tqd_state_rewind(self.handle)

    def apply(self, name, wires, params=(), matrix=None, trainable=True):
        tqd_apply_gate(self.handle, name, wires, params, matrix, trainable)

    def apply_circuit(self, gates):
        tqd_apply_circuit(self.handle, gates)

    @property
    def n_params(self) -> int:
        return tqd_num_params(self.handle)

    def apply_batch(self, gate, wires, params, trainable=True):
        """Per-state parameters: params has shape (batch, n_params_of_gate)."""
        tqd_apply_gate_batch(self.handle, gate, wires, params, trainable)

    def expval(self, terms) -> np.ndarray:
        return tqd_expval(self.handle, terms, self.batch)

    def adjoint_grad(self, terms, coeff=None):
        """coeff: (batch, n_terms) VJP weights; default: every element uses the terms' own."""
        return tqd_adjoint_grad(self.handle, terms, coeff=coeff)

    def amplitudes(self, first: int = 0, count: int | None = None) -> np.ndarray:
        if count is None:
            count = (self.batch << self.n) - first
        return tqd_get_amplitudes(self.handle, first, count, self.dtype)

    def sample(self, shots: int, seed: int) -> np.ndarray:
        """Exact shot sample: canonical outcomes."""
        return tqd_sample(self.handle, shots, seed, self.batch)

    def sample_gaussian_z(self, shots: float, seed: int) -> np.ndarray:
        """Noisy <Z_q> estimates from the approximate shot sample."""
        return tqd_sample_gaussian_z(self.handle, self.n, shots, seed, self.batch)

    def adjoint_grad_gaussian(self, shots: float, seed: int, coeff=None):
        """(L, dL/dtheta) for L = sum coeff * Zhat (reparameterised, differentiable)."""
        return tqd_adjoint_grad_gaussian(self.handle, shots, seed, coeff)

    def metrics(self) -> dict:
        return tqd_get_metrics(self.handle)

    def reset_metrics(self):
        tqd_reset_metrics(self.handle)

    def free(self):
        if self.handle:
            tqd_state_free(self.handle)
            self.handle = None
