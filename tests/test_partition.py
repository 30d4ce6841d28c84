"""Multi-GPU cell partition, host side, on CPU.

The exchange plan (bt_xchg_plan_host) and the protocol — local groups
summed in place, rank-spanning groups through a buffer that is summed over
ranks and reduced in member order — must reproduce the single-process
sync_additive (the reference oracle, fe_function.hpp:400-423) bitwise on
every rank's cells, for any rank count. The last test runs the protocol
with real collectives: two processes over torch.distributed gloo."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2308_01792_b200 as bt
from oracle.pyoracle import Oracle


def p1_groups(o, level):
    off, cell, g, t = o.groups(level)
    out = []
    for q in range(len(off) - 1):
        a, b = off[q], off[q + 1]
        if g[a] == 0:
            out.append((cell[a:b].copy(), t[a:b].copy()))
    return out


def local_sync(v, groups, cs, begin, end):
    """Groups whose members all lie in [begin, end): member-order sums."""
    out = v.copy()
    for cells, ts in groups:
        if len(cells) < 2 or not np.all((cells >= begin) & (cells < end)):
            continue
        slots = cells.astype(np.int64) * cs + ts
        s = 0.0
        for q in slots:
            s += v[q]
        out[slots] = s
    return out


def pack(v, plan):
    buf = np.zeros(plan["buf_size"])
    buf[plan["buf"]] = v[plan["slot"]]
    return buf


def combine(out, buf, plan):
    for slot, base, count in zip(plan["slot"], plan["base"], plan["count"]):
        s = 0.0
        for m in range(count):
            s += buf[base + m]
        out[slot] = s
    return out


MESHES = {
    "cube_kuhn": lambda: bt.cube_kuhn_text(),
    "cubes2": lambda: bt.cubes_mesh_text(2, 0.1, 0),
}


@pytest.mark.parametrize("mesh", sorted(MESHES))
@pytest.mark.parametrize("nranks", [2, 3, 5])
def test_partition_protocol_all_ranks(mesh, nranks):
    text = MESHES[mesh]()
    level = 3
    o = Oracle(text, 2, level, with_edges=False)
    nc = o.ncells
    cs = bt.n_tet((1 << level) + 1)
    v = np.random.default_rng(7).uniform(-1, 1, nc * cs)
    expected = o.sync(level, v)
    groups = p1_groups(o, level)
    plans = [bt.xchg_plan_host(text, level, r, nranks) for r in range(nranks)]
    sizes = {p["buf_size"] for p in plans}
    assert len(sizes) == 1
    # every buffer slot is written by exactly one rank
    owners = np.zeros(plans[0]["buf_size"], np.int64)
    for p in plans:
        np.add.at(owners, p["buf"], 1)
    assert np.all(owners == 1)
    total = sum(pack(v, p) for p in plans)  # the allreduce
    for r, p in enumerate(plans):
        b, e = bt.partition_range(nc, r, nranks)
        out = combine(local_sync(v, groups, cs, b, e), total, p)
        assert np.array_equal(out[b * cs:e * cs], expected[b * cs:e * cs])


def test_single_rank_plan_is_empty():
    p = bt.xchg_plan_host(bt.cube_kuhn_text(), 3, 0, 1)
    assert p["buf_size"] == 0 and len(p["slot"]) == 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, text, level):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        o = Oracle(text, 2, level, with_edges=False)
        nc = o.ncells
        cs = bt.n_tet((1 << level) + 1)
        v = np.random.default_rng(11).uniform(-1, 1, nc * cs)  # same on every rank
        expected = o.sync(level, v)
        plan = bt.xchg_plan_host(text, level, rank, world)
        buf = torch.from_numpy(pack(v, plan))
        dist.all_reduce(buf)
        b, e = bt.partition_range(nc, rank, world)
        out = combine(local_sync(v, p1_groups(o, level), cs, b, e), buf.numpy(), plan)
        assert np.array_equal(out[b * cs:e * cs], expected[b * cs:e * cs])
        # GPU-count-invariant dot: per-cell partials summed in cell order
        per = np.zeros(nc)
        for c in range(b, e):
            per[c] = 1.0 + c / 7.0
        t = torch.from_numpy(per)
        dist.all_reduce(t)
        s = 0.0
        for x in t.tolist():
            s += x
        ref = 0.0
        for c in range(nc):
            ref += 1.0 + c / 7.0
        assert s == ref
    finally:
        dist.destroy_process_group()


def test_partition_protocol_gloo_world2():
    mp.spawn(_worker, args=(2, _free_port(), bt.cubes_mesh_text(2, 0.1, 0), 3), nprocs=2, join=True)


# ---- the native data plane's neighbour-only exchange (bt_comm) ------------
# Rank r sends peer p its members of the groups the two share and receives
# p's: the buffer positions every rank's member-order combine reads must end
# up holding exactly what the allreduce of the whole buffer gives, and the
# message of r to p must list the same positions in the same order as p's
# receive from r (NCCL send/recv pairs carry no indices).

def neighbour_exchange(bufs, peers):
    """Apply every rank's grouped send/recv to the per-rank packed buffers."""
    out = [b.copy() for b in bufs]
    for r, pl in enumerate(peers):
        rp, rpos = pl["recvs"]
        for q in np.unique(rp):
            sp, spos = peers[q]["sends"]
            msg = bufs[q][spos[sp == r]]          # what q sends r, in q's order
            out[r][rpos[rp == q]] = msg           # where r puts it, in r's order
    return out


@pytest.mark.parametrize("mesh,nranks", [("cube_kuhn", 2), ("cube_kuhn", 3), ("cubes2", 2), ("cubes2", 5),
                                         ("cubes2", 8), ("blocked", 8)])
def test_neighbour_plan_matches_allreduce(mesh, nranks):
    text = bt.blocked_mesh_text(4, 4, 4, (2, 2, 2)) if mesh == "blocked" else MESHES[mesh]()
    level = 3
    plans = [bt.xchg_plan_host(text, level, r, nranks) for r in range(nranks)]
    peers = [bt.xchg_peers_host(text, level, r, nranks) for r in range(nranks)]
    rng = np.random.default_rng(3)
    bufs = []
    for p in plans:
        b = np.zeros(p["buf_size"])
        b[p["buf"]] = rng.uniform(-1, 1, len(p["buf"]))
        bufs.append(b)
    total = sum(bufs)
    got = neighbour_exchange(bufs, peers)
    moved = 0
    for r, p in enumerate(plans):
        # message pairing: r -> q positions (r's send order) == q's recv order from r
        for q in range(nranks):
            sp, spos = peers[r]["sends"]
            rp, rpos = peers[q]["recvs"]
            assert np.array_equal(spos[sp == q], rpos[rp == r])
        assert not np.any(peers[r]["sends"][0] == r) and not np.any(peers[r]["recvs"][0] == r)
        read = np.concatenate([np.arange(b, b + c) for b, c in zip(p["base"], p["count"])]) if len(p["base"]) else []
        assert np.array_equal(got[r][read], total[read])
        moved += len(peers[r]["sends"][1])
    # neighbour-only: every rank receives only positions of groups it is in
    assert moved <= sum(len(p["buf"]) for p in plans) * (nranks - 1)


def _worker_nbr(rank, world, port, text, level):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        o = Oracle(text, 2, level, with_edges=False)
        nc = o.ncells
        cs = bt.n_tet((1 << level) + 1)
        v = np.random.default_rng(13).uniform(-1, 1, nc * cs)
        expected = o.sync(level, v)
        plan = bt.xchg_plan_host(text, level, rank, world)
        pl = bt.xchg_peers_host(text, level, rank, world)
        buf = pack(v, plan)
        sp, spos = pl["sends"]
        rp, rpos = pl["recvs"]
        reqs, rbufs = [], {}
        for q in sorted(set(sp.tolist()) | set(rp.tolist())):
            if np.any(sp == q):
                reqs.append(dist.isend(torch.from_numpy(buf[spos[sp == q]].copy()), q))
            if np.any(rp == q):
                rbufs[q] = torch.zeros(int(np.sum(rp == q)), dtype=torch.float64)
                reqs.append(dist.irecv(rbufs[q], q))
        for rq in reqs:
            rq.wait()
        for q, t in rbufs.items():
            buf[rpos[rp == q]] = t.numpy()
        b, e = bt.partition_range(nc, rank, world)
        out = combine(local_sync(v, p1_groups(o, level), cs, b, e), buf, plan)
        assert np.array_equal(out[b * cs:e * cs], expected[b * cs:e * cs])
    finally:
        dist.destroy_process_group()


def test_neighbour_exchange_gloo_world3():
    mp.spawn(_worker_nbr, args=(3, _free_port(), bt.cubes_mesh_text(2, 0.1, 0), 3), nprocs=3, join=True)
