"""C-ABI library checks that need no GPU: it loads, exports every symbol that
include/tqd.h declares, and its host-only entry points validate arguments."""
import ctypes
import os
import re

import numpy as np
import pytest

import workloads as W

tqd = pytest.importorskip("paper_2511_19291_b200")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "tqd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tqd_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(tqd.LIB_PATH)
    names = header_functions()
    assert len(names) >= 18
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(tqd.EXPORTS)


def test_version_string():
    v = tqd.tqd_version()
    assert "sm_100a" in v and "NCCL" in v


def test_state_bytes():
    assert tqd.tqd_state_bytes(30, tqd.C64, 1, 1) == 2 * 8 * (1 << 30)
    # the north-star target, 36 qubits complex64 fwd+grad on 8 GPUs: psi + lambda (2 x 64 GiB)
    # plus the bounded exchange staging (1 GiB), within a B200's ~179 GB (SURVEY.md §8(e) memory)
    shard = 8 * (1 << 33)
    assert tqd.tqd_state_bytes(36, tqd.C64, 8, 1) == 2 * shard + (1 << 30)
    assert tqd.tqd_state_bytes(36, tqd.C64, 8, 1) <= 130 * 2**30 < 179e9
    assert tqd.tqd_state_bytes(36, tqd.C64, 8, 0) == shard + (1 << 30)
    # small shards: staging = two shards at most
    assert tqd.tqd_state_bytes(12, tqd.C128, 2, 1) == 2 * 16 * (1 << 11) + 2 * 16 * (1 << 11)
    with pytest.raises(tqd.TqdError) as e:
        tqd.tqd_state_bytes(3, tqd.C64, 4, 0)        # n < log2(world) + 2
    assert e.value.code == -2
    with pytest.raises(tqd.TqdError) as e:
        tqd.tqd_state_bytes(10, tqd.C64, 3, 0)       # world not a power of two
    assert e.value.code == -3


def test_debug_plan_rejects_bad_gates():
    with pytest.raises(tqd.TqdError) as e:
        tqd.tqd_debug_plan(4, [W.Gate("CNOT", (1, 1))])
    assert e.value.code == -1
    with pytest.raises(tqd.TqdError) as e:
        tqd.tqd_debug_plan(4, [W.Gate("RY", (7,), (0.1,))])
    assert e.value.code == -1
    import numpy as np
    bad = np.array([[1, 1], [0, 1]], complex)
    with pytest.raises(tqd.TqdError) as e:
        tqd.tqd_debug_plan(4, [W.Gate("MAT1", (0,), (), bad)])
    assert e.value.code == -4


def test_product_path_does_not_import_oracle():
    """The CUDA path never routes through the oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2511_19291_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "oracle.h" not in txt, f


def test_gate_arrays_checks_counts():
    """The packed gate arrays of tqd_apply_circuit carry no per-gate counts: wrong wire or
    parameter counts are rejected in the binding (as tqd_apply_gate rejects them), never padded."""
    import paper_2511_19291_b200 as tqd
    k, w, p, m, tr = tqd._gate_arrays([W.Gate("RY", (3,), (0.5,)), W.Gate("CNOT", (1, 2))])
    assert list(k) == [tqd.GATES["RY"], tqd.GATES["CNOT"]] and list(w) == [3, 0, 1, 2]
    assert list(p) == [0.5, 0, 0, 0, 0, 0] and list(tr) == [1, 1] and m.size == 64
    for bad in (W.Gate("CNOT", (1,)), W.Gate("RY", (1,), ()), W.Gate("U3", (0,), (0.1, 0.2)),
                W.Gate("X", (0, 1))):
        with pytest.raises(tqd.TqdError):
            tqd._gate_arrays([W.Gate("H", (0,)), bad])


def test_apply_gate_binding_checks_counts():
    """tqd_apply_gate takes no lengths: the binding rejects wrong wire / parameter /
    matrix sizes before the C call could read past a numpy buffer."""
    for gate, wires, params, mat in (("U3", [0], (0.1,), None), ("RY", [0], (), None), ("RY", [0, 1], (0.1,), None),
                                     ("CNOT", [0], (), None), ("X", [0], (0.3,), None), ("MAT1", [0], (), None),
                                     ("MAT2", [0, 1], (), np.eye(2))):
        with pytest.raises(tqd.TqdError) as e:
            tqd.tqd_apply_gate(None, gate, wires, params, mat)  # raised before the handle is used
        assert e.value.code == -1
