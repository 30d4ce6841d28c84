"""Multi-GPU cell partition on the device. One process plays
R ranks in sequence (no kernel waits on another). Each rank's handle holds
only its own cells (memory-sharded vectors):
  random_fill  local cells of the single-GPU stream, then a broadcast exchange;
  apply        the stencil on its cells, pack its replica values;
the buffers are summed (the allreduce) and each rank finishes its groups. The
rank slices, concatenated, must equal the single-handle vectors bitwise, for
both BC modes, and the per-cell dot partials summed in cell order must equal
bt.dot bitwise."""
import numpy as np
import pytest
import torch

import paper_2308_01792_b200 as bt

pytestmark = pytest.mark.gpu


def exchange(ranks, fns, level, mode, srcs=None):
    """The protocol with the allreduce played by a sum over the virtual ranks."""
    bufs = []
    for g, f in zip(ranks, fns):
        buf = g.xchg_buffer(level)
        if buf is not None and mode in (0, 1, 2):
            bt.xchg_pack(f, level, buf)
        bufs.append(buf)
    live = [b for b in bufs if b is not None]
    total = torch.stack(live).sum(0) if live else None
    for r, (g, f) in enumerate(zip(ranks, fns)):
        if bufs[r] is not None and total is not None:
            bufs[r].copy_(total)
        bt.xchg_finish(f, level, mode, bufs[r], srcs[r] if srcs else None)


def run_partitioned(text, level, nranks, bc):
    full = bt.Grid(text, 2, level)
    x = bt.allocate(bt.p1_space(), full, level, level)
    bt.random_fill(x, level, 3)
    yref = bt.allocate(bt.p1_space(), full, level, level)
    bt.apply_stencil(bt.compute_stencil(bt.FormId.diffusion(), full, level), x, yref, level, bc)
    cs = bt.n_tet((1 << level) + 1)
    grids, xs, ys = [], [], []
    for r in range(nranks):
        g = bt.Grid(text, 2, level)
        g.set_partition(r, nranks)
        _, _, b, e = g.partition()
        assert g.space_size(0, level) == (e - b) * cs  # memory-sharded
        xr = bt.allocate(bt.p1_space(), g, level, level)
        assert xr.values[level].numel() == (e - b) * cs
        bt.api._check(bt.api._L.bt_random_fill(g.handle, 0, level, 3, bt.api._ptr(xr.values[level]), None))
        grids.append(g)
        xs.append(xr)
    exchange(grids, xs, level, 2)  # broadcast of rank-spanning groups
    for g, xr in zip(grids, xs):
        _, _, b, e = g.partition()
        assert torch.equal(xr.values[level], x.values[level][b * cs:e * cs])
    for g, xr in zip(grids, xs):
        yr = bt.allocate(bt.p1_space(), g, level, level)
        t = bt.compute_stencil(bt.FormId.diffusion(), g, level)
        bt.api._check(bt.api._L.bt_apply_stencil_cells(t.handle, bt.api._ptr(xr.values[level]),
                                                       bt.api._ptr(yr.values[level]), None))
        ys.append(yr)
    exchange(grids, ys, level, 1 if bc else 0, xs)
    y = torch.empty_like(yref.values[level])
    for g, yr in zip(grids, ys):
        _, _, b, e = g.partition()
        assert not torch.isnan(yr.values[level]).any()
        y[b * cs:e * cs] = yr.values[level]
    torch.cuda.synchronize()
    assert torch.equal(y, yref.values[level])  # bitwise
    # dot: per-cell partials in cell order
    per = sum(bt.dot_cells(xr, yr, level) for xr, yr in zip(xs, ys))
    s = 0.0
    for v in per:
        s += v
    yfull = bt.allocate(bt.p1_space(), full, level, level)
    yfull.values[level].copy_(y)
    assert s == bt.dot(x, yfull, level)


@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("bc", [bt.BC.None_, bt.BC.DirichletIdentity])
def test_partitioned_stencil_cube_kuhn(nranks, bc):
    run_partitioned(bt.cube_kuhn_text(), 5, nranks, bc)


@pytest.mark.parametrize("nranks", [2, 4])
def test_partitioned_stencil_perturbed_cubes(nranks):
    run_partitioned(bt.cubes_mesh_text(2, 0.1, 0), 4, nranks, bt.BC.DirichletIdentity)


def test_partitioned_impose_and_zero_dirichlet():
    text, level, nranks = bt.cubes_mesh_text(2, 0.1, 0), 4, 3
    full = bt.Grid(text, 2, level)
    x = bt.allocate(bt.p1_space(), full, level, level)
    bt.random_fill(x, level, 5)
    z = bt.allocate(bt.p1_space(), full, level, level)
    z.values[level].copy_(x.values[level])
    bt.zero_dirichlet(z, level)
    cs = bt.n_tet((1 << level) + 1)
    for r in range(nranks):
        g = bt.Grid(text, 2, level)
        g.set_partition(r, nranks)
        _, _, b, e = g.partition()
        xr = bt.allocate(bt.p1_space(), g, level, level)
        xr.values[level].copy_(x.values[level][b * cs:e * cs])
        bt.zero_dirichlet(xr, level)
        assert torch.equal(xr.values[level], z.values[level][b * cs:e * cs])
        yr = bt.allocate(bt.p1_space(), g, level, level)
        bt.impose_dirichlet(xr, yr, level)  # yr = 0 except Dirichlet slots, which are 0 in xr too
        assert not torch.isnan(yr.values[level]).any()


def test_partitioned_n1e1_needs_the_allreduce_hook():
    g = bt.Grid(bt.cube_kuhn_text(), 2, 3)
    bt.api._check(bt.api._L.bt_grid_set_partition(g.handle, 0, 2))  # no allreduce hook
    op = bt.N1E1Operator(g, 3)
    x, y = bt.allocate(bt.edge_space(), g, 3, 3), bt.allocate(bt.edge_space(), g, 3, 3)
    with pytest.raises(bt.LogicError):
        bt.apply_n1e1(op, x, y, 3)
