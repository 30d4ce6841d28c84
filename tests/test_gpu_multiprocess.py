"""The library's own exchange across real processes.

Two processes (torch.multiprocessing, gloo process group over 127.0.0.1), each
with its own bt_grid partitioned by Grid.set_partition(rank, 2): once with
the default data plane for a non-NCCL group (the library's neighbour-only
exchange, torch.distributed send/recv as the transport) and once with the
allreduce hook (torch.distributed.all_reduce on the library's exchange
buffer), both called by the library itself inside every collective entry
point. Each process also runs the same program on an unpartitioned
grid and checks its slice of every result bitwise: apply_stencil (both BCs),
the elementwise apply, diagonals and transfers, a V-cycle with Chebyshev
smoothing and coarse CG (solution, residual norms and CG history), and the
N1E1 apply (fe_function.hpp:400-423, solvers.hpp:509-541).

Both processes drive cuda:0 (the pool gives one GPU per call). The gloo
allreduce stages the device buffer through the host after a stream sync, so
no kernel of one process waits on a kernel of the other."""
import os
import socket
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, failures, xchg):
    try:
        os.environ["BT_XCHG"] = xchg
        import paper_2308_01792_b200 as bt
        from test_gpu_partition_solvers import n1e1_body, operators_body, vcycle_body

        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        try:
            def part(g):
                g.set_partition(rank, world)  # default data plane for a gloo group
                assert g.data_plane() == ("allreduce" if xchg == "allreduce" else "sendrecv")

            text = bt.cubes_mesh_text(2, 0.1, 0)
            L = 4
            ob = operators_body(text, L)
            full, mine = ob(lambda g: None), ob(part)
            _, _, b, e = mine["part"]
            cs = {L: bt.n_tet((1 << L) + 1), L - 1: bt.n_tet((1 << (L - 1)) + 1)}
            for k in ("x", "stencil0", "stencil1", "elementwise", "diag_ew", "diag_stencil", "prolongate", "sync"):
                assert torch.equal(mine[k], full[k][b * cs[L]:e * cs[L]]), k
            assert torch.equal(mine["restrict"], full["restrict"][b * cs[L - 1]:e * cs[L - 1]])
            assert mine["dot"] == full["dot"]

            vb = vcycle_body(text, 2, L, bt.KernelKind.Elementwise)
            full, mine = vb(lambda g: None), vb(part)
            assert torch.equal(mine["x"], full["x"][b * cs[L]:e * cs[L]])
            assert mine["hist"] == full["hist"] and mine["cg"] == full["cg"]

            nb = n1e1_body(text, 3)
            full, mine = nb(lambda g: None), nb(part)
            g = bt.Grid(text, 2, 3)
            ce = g.space_size(2, 3) // g.n_cells()
            _, _, b, e = mine["part"]
            for k in ("x", "y0", "y1", "sync"):
                assert torch.equal(mine[k], full[k][b * ce:e * ce]), k
            assert mine["dot"] == full["dot"]
        finally:
            dist.destroy_process_group()
    except BaseException as ex:  # noqa: BLE001 - reported to the parent
        failures.put(f"rank {rank}: {type(ex).__name__}: {ex}")
        raise


@pytest.mark.parametrize("xchg", ["auto", "allreduce"])
def test_library_exchange_two_processes(xchg):
    """auto: the library's neighbour-only exchange (gather, per-peer
    messages, scatter) with torch.distributed as the transport; allreduce:
    the allreduce hook over the whole exchange buffer."""
    ctx = mp.get_context("spawn")
    failures = ctx.Queue()
    mp.start_processes(_worker, args=(2, _free_port(), failures, xchg), nprocs=2, join=True, start_method="spawn")
    assert failures.empty()
