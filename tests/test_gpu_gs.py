"""Hybrid Gauss-Seidel (gauss_seidel_sweep operators.hpp:327-387, the
reference's default smoother) on the device, against the
compiled reference (oracle/_ref) and the C restatement.

The interior of every cell is swept by hyperplane wavefronts i + 2j + 3k =
const, which reproduce the lexicographic order exactly: after one sweep from
the same input, interior values are bitwise the reference's. The Jacobi step
on the other vertices uses typed partial rows, whose association differs from
the reference's per-micro-cell sums, so everything else is compared within
relative L2 1e-12."""
import math

import numpy as np
import pytest

import paper_2308_01792_b200 as bt
from pyoracle import Oracle, Reference

pytestmark = pytest.mark.gpu
REL = 1e-12
GS = bt.SmootherConfig.gauss_seidel()


def host(fn, l):
    return fn.values[l].cpu().numpy()


def upload(fn, l, a):
    fn.values[l].copy_(bt.api.torch.from_numpy(np.ascontiguousarray(a)))


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def interior_mask(ncells, l):
    n = 1 << l
    w = n + 1
    m = []
    for k in range(w):
        for j in range(w - k):
            for i in range(w - k - j):
                m.append(i >= 1 and j >= 1 and k >= 1 and i + j + k <= n - 1)
    return np.tile(np.array(m), ncells)


MESHES = [(bt.cube_kuhn_text(), 2, 4), (bt.cubes_mesh_text(2, 0.1, 0), 2, 4), (bt.ref_tet_text(), 2, 5)]


@pytest.mark.parametrize("text,lo,hi", MESHES)
@pytest.mark.parametrize("backward", [False, True])
def test_sweep_interior_bitwise(text, lo, hi, backward):
    g = bt.Grid(text, lo, hi)
    h = bt.make_hierarchy(g, bt.FormId.diffusion(), bt.KernelKind.Stencil)
    r = Reference(text, lo, hi)
    r.make_hierarchy(form=0, kernel=1)
    o = Oracle(text, lo, hi)
    o.make_hierarchy(0, None, 1)
    l = hi
    rhs, x = bt.allocate(bt.p1_space(), g, l, l), bt.allocate(bt.p1_space(), g, l, l)
    bt.random_fill(rhs, l, 3)
    bt.random_fill(x, l, 4)
    rh, x0 = host(rhs, l), host(x, l)
    direction = bt.SweepDirection.Backward if backward else bt.SweepDirection.Forward
    bt.smooth(h, GS, rhs, x, l, 1, direction)
    xr = r.smooth(l, GS.as_array(), rh, x0, sweeps=1, backward=backward)
    xo = o.smooth(l, GS.as_array(), rh, x0, sweeps=1, backward=backward)
    mask = interior_mask(g.n_cells(), l)
    xg = host(x, l)
    assert np.array_equal(xg[mask], xr[mask])  # wavefronts = the sequential order, bit for bit
    assert rel(xg, xr) <= REL and rel(xg, xo) <= REL
    # the table-level entry point is the same sweep
    y = bt.allocate(bt.p1_space(), g, l, l)
    upload(y, l, x0)
    bt.gauss_seidel_sweep(bt.compute_stencil(bt.FormId.diffusion(), g, l), rhs, y, l, direction)
    assert np.array_equal(host(y, l), xg)


@pytest.mark.parametrize("text,lo,hi", MESHES[:2])
def test_vcycle_default_smoother(text, lo, hi):
    """V(1,1) with the default (Gauss-Seidel) smoother: forward pre-, backward post-smoothing."""
    g = bt.Grid(text, lo, hi)
    h = bt.make_hierarchy(g, bt.FormId.diffusion())
    r = Reference(text, lo, hi)
    r.make_hierarchy(form=0, kernel=1)
    l = hi
    rhs, x = bt.allocate(bt.p1_space(), g), bt.allocate(bt.p1_space(), g)
    bt.random_fill(rhs, l, 0)
    bt.zero_dirichlet(rhs, l)
    mg = bt.MultigridConfig(coarse_level=lo, coarse_tol=1e-14, coarse_maxit=50)
    res = bt.allocate(bt.p1_space(), g, l, l)
    hist = []
    for _ in range(4):
        bt.v_cycle(h, l, rhs, x, GS, mg)
        bt.hierarchy_apply(h, x, res, l)
        res.values[l].mul_(-1.0).add_(rhs.values[l])
        hist.append(bt.norm2(res, l) / bt.norm2(rhs, l))
    rh = host(rhs, l)
    xr, hr = r.vcycles(l, GS.as_array(), rh, np.zeros_like(rh), 4, lo, 1e-14, 50)
    assert rel(hist, hr[1:]) <= REL
    assert rel(host(x, l), xr) <= REL
    assert hist[-1] < 0.1 * hist[0]


def test_fmg_default_smoother_matches_reference():
    """The reference tests' FMG (test_solvers.cpp 'full multigrid runs the documented cycle budget')."""
    text, lo, hi = bt.cube_kuhn_text(), 2, 4
    U = bt.Coefficient.sin_product(0.0, 1.0, math.pi)
    F = bt.Coefficient.sin_product(0.0, 3.0 * math.pi ** 2, math.pi)
    g = bt.Grid(text, lo, hi)
    h = bt.make_hierarchy(g, bt.FormId.diffusion())
    rhs = []
    for l in range(lo, hi + 1):
        f, b = bt.allocate(bt.p1_space(), g, l, l), bt.allocate(bt.p1_space(), g, l, l)
        bt.interpolate(f, l, F)
        bt.apply_elementwise(bt.FormId.mass(), f, b, l)
        bt.zero_dirichlet(b, l)
        rhs.append(b)
    x = bt.allocate(bt.p1_space(), g, hi, hi)
    mg = bt.MultigridConfig()
    rep = bt.fmg(h, hi, rhs, x, GS, mg, exact=U)
    assert rep.iterations == 5 * (hi - lo) and len(rep.rows) == 1 + 5 * (hi - lo)
    r = Reference(text, lo, hi)
    r.make_hierarchy(form=0, kernel=1)
    rows, xr = r.fmg(hi, GS.as_array(), [host(b, lo + i) for i, b in enumerate(rhs)], lo, mg.cycles,
                     mg.coarse_tol, mg.coarse_maxit, fp=(U.kind,) + tuple(U.c))
    for a, b in zip(rep.rows, rows):
        assert a.residual == pytest.approx(b[2], rel=1e-8, abs=1e-15)
        assert a.error == pytest.approx(b[3], rel=1e-10)
    assert rel(host(x, hi), xr) <= 1e-10
    err = {row.level: row.error for row in rep.rows}
    assert 2.8 <= err[2] / err[3] <= 4.7 and 3.4 <= err[3] / err[4] <= 4.6


def test_gauss_seidel_needs_a_stencil_table():
    g = bt.Grid(bt.cube_kuhn_text(), 2, 3)
    h = bt.make_hierarchy(g, bt.FormId.div_k_grad(bt.Coefficient.sin_product()), bt.KernelKind.Elementwise)
    x, rhs = bt.allocate(bt.p1_space(), g), bt.allocate(bt.p1_space(), g)
    with pytest.raises(bt.InvalidArgument):
        bt.smooth(h, GS, rhs, x, 3, 1)


def test_vcycle_level_guards():
    """test_solvers.cpp 'level guards': a coarse level below the grid's, or a V-cycle below the coarse level."""
    g = bt.Grid(bt.cube_kuhn_text(), 2, 4)
    h = bt.make_hierarchy(g, bt.FormId.diffusion())
    x, rhs = bt.allocate(bt.p1_space(), g), bt.allocate(bt.p1_space(), g)
    low = bt.MultigridConfig(coarse_level=1)
    with pytest.raises(bt.InvalidArgument):
        bt.v_cycle(h, 3, rhs, x, GS, low)
    with pytest.raises((bt.InvalidArgument, bt.OutOfRange)):
        bt.v_cycle(h, 1, rhs, x, GS, bt.MultigridConfig())
    bad = bt.SmootherConfig.jacobi(1.5)  # omega outside (0, 1]
    with pytest.raises(bt.InvalidArgument):
        bt.smooth(h, bad, rhs, x, 4, 1)
