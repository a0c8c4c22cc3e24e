"""Multi-rank (world 2 and 4) host-path tests on CPU with the gloo backend.

The N > 1 device path (NCCL send/recv of remap blocks, rank-bit conditioned
diagonal gates / controls) cannot run on this 1-GPU build, so these tests run
the library's own HOST logic across real processes:

  * every rank plans the same circuit (tqd_debug_plan) -> identical plans
    (the collectives' symmetric-call contract);
  * the plan is executed on per-rank numpy shards: ops on the physical bits
    the planner resolved (global bits = this rank's bits), the sweeps' store
    permutations, and every REMAP exchanged between the processes over gloo
    following the library's schedule (tqd_debug_remap_schedule: which block
    goes to which peer and where the received block lands);
  * the gathered state, mapped to canonical order through the final qubit map,
    equals the float64 oracle.
"""
import hashlib
import json
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _apply_local(shard, n_loc, rank, M, bits):
    """Apply M on physical bits; bits >= n_loc are this rank's (fixed) bits."""
    gl = [b >= n_loc for b in bits]
    val = [((rank >> (b - n_loc)) & 1) if g else None for b, g in zip(bits, gl)]
    idx = np.arange(shard.size)
    if len(bits) == 1:
        if gl[0]:
            v = val[0]
            assert M[0, 1] == 0 and M[1, 0] == 0, "non-diagonal action on a global qubit"
            shard *= M[v, v]
            return
        b = 1 << bits[0]
        i0 = idx[(idx & b) == 0]
        i1 = i0 | b
        a0, a1 = shard[i0].copy(), shard[i1].copy()
        shard[i0] = M[0, 0] * a0 + M[0, 1] * a1
        shard[i1] = M[1, 0] * a0 + M[1, 1] * a1
        return
    if gl[0] and gl[1]:
        k = 2 * val[0] + val[1]
        assert np.count_nonzero(M[k, :]) <= 1 and np.count_nonzero(M[:, k]) <= 1
        shard *= M[k, k]
        return
    if gl[0] or gl[1]:
        if gl[0]:
            v = val[0]
            sub = M[2 * v:2 * v + 2, 2 * v:2 * v + 2]
            off = np.delete(M[2 * v:2 * v + 2, :], [2 * v, 2 * v + 1], axis=1)
            loc = bits[1]
        else:
            v = val[1]
            sub = M[np.ix_([v, 2 + v], [v, 2 + v])]
            off = np.delete(M[[v, 2 + v], :], [v, 2 + v], axis=1)
            loc = bits[0]
        assert np.all(off == 0), "gate mixes a global qubit"
        _apply_local(shard, n_loc, rank, sub, [loc])
        return
    b0, b1 = 1 << bits[0], 1 << bits[1]
    base = idx[(idx & (b0 | b1)) == 0]
    ids = [base, base | b1, base | b0, base | b0 | b1]
    v = [shard[i].copy() for i in ids]
    for r in range(4):
        shard[ids[r]] = sum(M[r, c] * v[c] for c in range(4))


def _permute_bits(x, src, dst):
    idx = np.arange(x.size)
    new = idx.copy()
    for s in src:
        new &= ~(1 << s)
    for s, d in zip(src, dst):
        new |= ((idx >> s) & 1) << d
    out = np.empty_like(x)
    out[new] = x
    return out


def _remap(shard, n_loc, rank, gpos, lpos, tqd, dist, torch):
    m = len(gpos)
    peer, recv_block = tqd.tqd_debug_remap_schedule(rank, n_loc, gpos, lpos)
    rest = [p for p in range(n_loc) if p not in lpos]
    idx = np.arange(shard.size)
    blkid = np.zeros(shard.size, dtype=np.int64)
    for i, p in enumerate(lpos):
        blkid |= ((idx >> p) & 1) << i
    within = np.zeros(shard.size, dtype=np.int64)
    for i, p in enumerate(rest):
        within |= ((idx >> p) & 1) << i
    nblk = 1 << m
    bsz = shard.size // nblk
    blocks = np.zeros((nblk, bsz), complex)
    blocks[blkid, within] = shard
    out = np.zeros_like(blocks)
    reqs = []
    bufs = {}
    for b in range(nblk):
        if peer[b] == rank:
            out[recv_block[b]] = blocks[b]
        else:
            send = torch.from_numpy(np.ascontiguousarray(blocks[b]).view(np.float64).copy())
            rbuf = torch.zeros(2 * bsz, dtype=torch.float64)
            bufs[b] = rbuf
            reqs.append(dist.isend(send, int(peer[b])))
            reqs.append(dist.irecv(rbuf, int(peer[b])))
    for r in reqs:
        r.wait()
    for b, rbuf in bufs.items():
        out[recv_block[b]] = rbuf.numpy().view(np.complex128)
    new = np.zeros_like(shard)
    new[idx] = out[blkid, within]
    return new


def _worker(rank, world, port, n, seed, k, small_max, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        import oracle
        import paper_2511_19291_b200 as tqd
        import workloads as W
        gates = W.random_circuit(n, 90, seed) + W.hea(n, 2, seed) + W.qft(n)[:20]
        plan = tqd.tqd_debug_plan(n, gates, world=world, k=k, small_max=small_max)
        digest = hashlib.sha256(json.dumps(plan, sort_keys=True).encode()).hexdigest()
        digests = [None] * world
        dist.all_gather_object(digests, digest)
        assert len(set(digests)) == 1, "ranks planned differently"
        g = world.bit_length() - 1
        n_loc = n - g
        shard = np.zeros(1 << n_loc, complex)
        if rank == 0:
            shard[0] = 1.0
        n_remaps = 0
        for st in plan["stages"]:
            if st["type"] in ("sweep", "small"):
                for op in st["ops"]:
                    gate = gates[op["gate"]]
                    M = oracle.gate_matrix(gate.name, gate.params, gate.matrix)
                    bits = [op["wp0"]] if len(gate.wires) == 1 else [op["wp0"], op["wp1"]]
                    _apply_local(shard, n_loc, rank, M, bits)
                if st["type"] == "sweep" and st["ops"]:
                    shard = _permute_bits(shard, st["ld_phys"], st["st_phys"])
            else:
                shard = _remap(shard, n_loc, rank, st["gpos"], st["lpos"], tqd, dist, torch)
                n_remaps += 1
        pos = plan["stages"][-1]["pos_after"]
        parts = [None] * world
        dist.all_gather_object(parts, shard)
        if rank == 0:
            full = np.concatenate(parts)
            N = 1 << n
            c = np.arange(N)
            phys = np.zeros(N, dtype=np.int64)
            for qb in range(n):
                phys |= ((c >> (n - 1 - qb)) & 1) << pos[qb]
            got = full[phys]
            ref = oracle.run(n, gates)
            q.put(("ok", float(np.max(np.abs(got - ref))), n_remaps))
    except Exception as e:  # report to the parent
        import traceback
        q.put(("error", traceback.format_exc(), 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,k,small_max", [(2, 12, 9, 0), (4, 13, 9, 0), (2, 9, 9, 10)])
def test_distributed_replay_gloo(world, n, k, small_max):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, 3, k, small_max, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    status, val, nrem = q.get(timeout=10)
    assert status == "ok", val
    assert nrem > 0
    assert val < 1e-10


def test_remap_schedule_pairs():
    """Every send has a matching receive: rank r sends block b to p iff p's
    schedule receives from r, and each rank receives every block index once."""
    import paper_2511_19291_b200 as tqd
    n_loc, gpos, lpos = 10, [11, 10], [3, 7]
    world = 4
    sched = {r: tqd.tqd_debug_remap_schedule(r, n_loc, gpos, lpos) for r in range(world)}
    for r in range(world):
        peer, recv = sched[r]
        assert sorted(recv) == list(range(4))
        for b, p in enumerate(peer):
            pp, _ = sched[int(p)]
            assert r in list(pp)
