"""The native NCCL data plane (bt_comm, csrc/bt_comm.cpp) on the one GPU a
test box has: NCCL loads and a communicator initialises, the ABI checks the
communicator against the grid's partition, and an apply / dot / V-cycle on
a grid with the communicator attached are bitwise those without it.

NCCL refuses two ranks on one device, so the multi-rank neighbour exchange
itself is covered by (a) tests/test_partition.py (plan pairing and
coverage, emulated and over gloo) and (b) tests/test_gpu_multiprocess.py,
where the library's gather / per-peer messages / scatter run across two
real processes with torch.distributed as the transport; bt_comm only swaps
the transport for grouped ncclSend / ncclRecv."""
import pytest
import torch

import paper_2308_01792_b200 as bt

pytestmark = pytest.mark.gpu


def test_comm_single_rank():
    uid = bt.Comm.unique_id()
    assert len(uid) == 128
    comm = bt.Comm(uid, 0, 1, 0)
    try:
        text = bt.cubes_mesh_text(2, 0.1, 0)
        L = 4
        res = []
        for use in (False, True):
            g = bt.Grid(text, 2, L, device=0)
            g.set_partition(0, 1, comm=comm if use else None)
            assert g.data_plane() == ("nccl" if use else "allreduce")
            x, y = bt.allocate(bt.p1_space(), g), bt.allocate(bt.p1_space(), g)
            bt.random_fill(x, L, 5)
            t = bt.compute_stencil(bt.FormId.diffusion(), g, L)
            bt.apply_stencil(t, x, y, L)
            res.append((y.level(L).clone(), bt.dot(x, y, L)))
        assert torch.equal(res[0][0], res[1][0]) and res[0][1] == res[1][1]
        # the communicator must be the grid's partition
        g = bt.Grid(text, 2, L, device=0)
        g.set_partition(1, 2, comm=None)
        with pytest.raises(bt.LogicError):
            g.set_comm(comm)
    finally:
        comm.close()
