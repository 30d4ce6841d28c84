"""Multi-GPU cell partition on the device. One process plays
R ranks in sequence (no kernel waits on another): each rank's handle applies
the stencil to its own cells and packs its replica values; the buffers are
summed (the allreduce); each rank finishes its groups. The assembled result
must equal the single-handle apply_stencil bitwise, for both BC modes, and
the per-cell dot partials summed in cell order must equal bt.dot bitwise."""
import numpy as np
import pytest
import torch

import paper_2308_01792_b200 as bt

pytestmark = pytest.mark.gpu


def run_partitioned(text, level, nranks, bc):
    full = bt.Grid(text, 2, level)
    x = bt.allocate(bt.p1_space(), full, level, level)
    bt.random_fill(x, level, 3)
    yref = bt.allocate(bt.p1_space(), full, level, level)
    bt.apply_stencil(bt.compute_stencil(bt.FormId.diffusion(), full, level), x, yref, level, bc)
    cs = bt.n_tet((1 << level) + 1)
    ranks = []
    for r in range(nranks):
        g = bt.Grid(text, 2, level)
        g.set_partition(r, nranks)
        xr = bt.allocate(bt.p1_space(), g, level, level)
        bt.random_fill(xr, level, 3)  # every rank holds the full input
        assert torch.equal(xr.values[level], x.values[level])
        yr = bt.allocate(bt.p1_space(), g, level, level)
        bt.assign(yr, level, float("nan"))  # other ranks' cells must stay untouched
        t = bt.compute_stencil(bt.FormId.diffusion(), g, level)
        bt.api._check(bt.api._L.bt_apply_stencil_cells(t.handle, bt.api._ptr(xr.values[level]),
                                                       bt.api._ptr(yr.values[level]), None))
        buf = g.xchg_buffer(level)
        bt.xchg_pack(yr, level, buf)
        ranks.append((g, xr, yr, t, buf))
    bufs = [b for (_, _, _, _, b) in ranks if b is not None]
    total = torch.stack(bufs).sum(0) if bufs else None
    y = torch.empty_like(yref.values[level])
    for r, (g, xr, yr, t, buf) in enumerate(ranks):
        if buf is not None:
            buf.copy_(total)
        bt.xchg_finish(yr, level, 1 if bc else 0, buf, xr)
        _, _, b, e = g.partition()
        seg = yr.values[level][b * cs:e * cs]
        assert not torch.isnan(seg).any()
        y[b * cs:e * cs] = seg
    torch.cuda.synchronize()
    assert torch.equal(y, yref.values[level])  # bitwise
    # dot: per-cell partials in cell order
    per = sum(bt.dot_cells(xr, yr, level) for (_, xr, yr, _, _) in ranks)
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


def test_partitioned_grid_refuses_full_sync():
    g = bt.Grid(bt.cube_kuhn_text(), 2, 3)
    g.set_partition(0, 2)
    x = bt.allocate(bt.p1_space(), g, 3, 3)
    with pytest.raises(bt.LogicError):
        bt.apply_elementwise(bt.FormId.mass(), x, bt.allocate(bt.p1_space(), g, 3, 3), 3)
