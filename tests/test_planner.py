"""Host-side planner checks (CPU only, no GPU): tqd_debug_plan through the C ABI.

The plan (fused sweep stages, register layouts, output bit permutations,
remaps, the qubit map pi) is replayed here on a full numpy state vector with
the ORACLE's gate matrices: every op is applied on the physical bits the
planner resolved, every sweep's store permutation and every remap's bit swap
is applied, and the final physical vector is mapped back to canonical order
through the final pi.  It must equal the oracle's run of the original circuit.
This checks the planner's index bookkeeping independently of the kernels.
"""
import numpy as np
import pytest

import workloads as W

tqd = pytest.importorskip("paper_2511_19291_b200")


def apply_phys(psi, n, M, bits):
    """Apply M on physical bit positions `bits` (bits[0] = MSB of M's index)."""
    N = psi.size
    idx = np.arange(N)
    if len(bits) == 1:
        b = 1 << bits[0]
        i0 = idx[(idx & b) == 0]
        i1 = i0 | b
        a0, a1 = psi[i0].copy(), psi[i1].copy()
        psi[i0] = M[0, 0] * a0 + M[0, 1] * a1
        psi[i1] = M[1, 0] * a0 + M[1, 1] * a1
    else:
        b0, b1 = 1 << bits[0], 1 << bits[1]
        base = idx[(idx & (b0 | b1)) == 0]
        ids = [base, base | b1, base | b0, base | b0 | b1]
        v = [psi[i].copy() for i in ids]
        for r in range(4):
            psi[ids[r]] = sum(M[r, c] * v[c] for c in range(4))


def permute_bits(psi, n, src, dst):
    """Data at physical bit src[i] moves to bit dst[i] (other bits fixed)."""
    N = psi.size
    idx = np.arange(N)
    new = idx.copy()
    for s in src:
        new &= ~(1 << s)
    for s, d in zip(src, dst):
        new |= ((idx >> s) & 1) << d
    out = np.empty_like(psi)
    out[new] = psi
    return out


def replay(n, gates, plan, orc):
    psi = np.zeros(1 << n, complex)
    psi[0] = 1
    prev_after = [n - 1 - q for q in range(n)]
    for st in plan["stages"]:
        assert st["pos_before"] == prev_after
        if st["type"] in ("sweep", "small"):
            for op in st["ops"]:
                g = gates[op["gate"]]
                M = orc.gate_matrix(g.name, g.params, g.matrix)
                bits = [op["wp0"]] if len(g.wires) == 1 else [op["wp0"], op["wp1"]]
                apply_phys(psi, n, M, bits)
            if st["type"] == "sweep" and st["ops"]:
                psi = permute_bits(psi, n, st["ld_phys"], st["st_phys"])
        else:
            src = st["gpos"] + st["lpos"]
            dst = st["lpos"] + st["gpos"]
            psi = permute_bits(psi, n, src, dst)
        prev_after = st["pos_after"]
    pos = prev_after
    N = 1 << n
    c = np.arange(N)
    phys = np.zeros(N, dtype=np.int64)
    for q in range(n):
        phys |= ((c >> (n - 1 - q)) & 1) << pos[q]
    return psi[phys]


def check_invariants(plan):
    for st in plan["stages"]:
        if st["type"] != "sweep":
            continue
        k, R, Wb, C = st["k"], st["R"], st["W"], st["c_low"]
        ld, stp, lays = st["ld_phys"], st["st_phys"], st["layouts"]
        assert ld[:C] == list(range(C))
        assert lays[0]["lane"][:C] == list(range(C))
        assert sorted(ld) == sorted(stp) and len(set(ld)) == k
        for L in lays:
            bits = L["reg"] + L["lane"] + L["warp"]
            assert sorted(bits) == list(range(k)) and len(L["reg"]) == R and len(L["warp"]) == Wb
        last = lays[-1]["lane"]
        assert [stp[t] for t in last[:C]] == list(range(C))
        segs = [op["seg"] for op in st["ops"]]
        assert segs == sorted(segs)
        # warp-local exchanges: same warp bits on both sides and no
        # permutation gate of the segment targets a warp bit
        for s, um in enumerate(st["xumask"][: len(lays) - 1]):
            # warp groups: a kept warp-index bit is the same tile bit on both sides and
            # no permutation gate of the segment targets it
            for i in range(st["W"]):
                if (um >> i) & 1:
                    assert lays[s]["warp"][i] == lays[s + 1]["warp"][i]
                    for op in st["ops"]:
                        if op["perm"] and op["seg"] == s:
                            assert ld.index(op["tp0"]) != lays[s]["warp"][i]
            assert st["xwarp"][s] == (1 if um == (1 << st["W"]) - 1 else 0)
        for op in st["ops"]:
            if op["perm"]:  # CNOT / X folded into a layout-change map: target only needs to be in the tile
                assert op["tp0"] in ld
                continue
            for key in ("tp0", "tp1"):
                if op[key] >= 0:
                    assert ld.index(op[key]) in lays[op["seg"]]["reg"]


@pytest.mark.parametrize("n,k,seed", [(11, 9, 0), (12, 10, 1), (13, 11, 2), (14, 12, 3), (16, 12, 4), (15, 9, 5)])
def test_random_circuit_plan_replay(orc, n, k, seed):
    gates = W.random_circuit(n, 150, seed)
    plan = tqd.tqd_debug_plan(n, gates, world=1, k=k, small_max=0)
    check_invariants(plan)
    assert all(s["type"] == "sweep" for s in plan["stages"])
    got = replay(n, gates, plan, orc)
    ref = orc.run(n, gates)
    assert np.max(np.abs(got - ref)) < 1e-10


@pytest.mark.parametrize("n,depth", [(12, 3), (14, 4), (16, 2)])
def test_hea_plan_replay(orc, n, depth):
    gates = W.hea(n, depth, seed=n)
    plan = tqd.tqd_debug_plan(n, gates, world=1, k=12, small_max=0)
    check_invariants(plan)
    got = replay(n, gates, plan, orc)
    assert np.max(np.abs(got - orc.run(n, gates))) < 1e-10


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("small_max", [0, 12])
def test_sharded_plan_replay(orc, world, small_max):
    """Remap stages (global <-> local bit swaps) keep the state consistent."""
    n = 13
    gates = W.random_circuit(n, 120, seed=world) + W.hea(n, 2, seed=world)
    plan = tqd.tqd_debug_plan(n, gates, world=world, k=9, small_max=small_max)
    check_invariants(plan)
    assert any(s["type"] == "remap" for s in plan["stages"])
    got = replay(n, gates, plan, orc)
    assert np.max(np.abs(got - orc.run(n, gates))) < 1e-10


def test_qft_relabels(orc):
    n = 12
    gates = W.basis_prep(n, 1234) + W.qft(n)
    plan = tqd.tqd_debug_plan(n, gates, world=1, k=10, small_max=0)
    check_invariants(plan)
    got = replay(n, gates, plan, orc)
    assert np.max(np.abs(got - orc.run(n, gates))) < 1e-10


def test_fusion_counts_hea30():
    """cfg 3 workload: every stage fuses many gates (bytes per gate per amplitude << 16)."""
    gates = W.hea(30, 20, seed=0)
    plan = tqd.tqd_debug_plan(30, gates, world=1, k=12)
    sweeps = [s for s in plan["stages"] if s["type"] == "sweep"]
    assert sum(s["n_gates"] for s in sweeps) == len(gates)
    assert len(sweeps) <= 120
    for s in sweeps:
        assert len(s["layouts"]) <= 24
