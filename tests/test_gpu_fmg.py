"""Full multigrid, interpolation and the L2 error on the
device, against the compiled reference (oracle/_ref: interpolate
fe_function.hpp:454, l2_error solvers.hpp:613, fmg solvers.hpp:547) and the
reference tests' properties (test_solvers.cpp "full multigrid runs the
documented cycle budget", "one-level full multigrid is the coarse solve",
acceptance.cpp criterion 7). The reference's fields are std::function
callbacks; both sides here evaluate the same device-evaluable field kinds.
Device sin differs from glibc's by ulps, so interpolated values and errors are
compared within tolerance, not bitwise."""
import math

import numpy as np
import pytest
import torch

import paper_2308_01792_b200 as bt
from pyoracle import Reference

pytestmark = pytest.mark.gpu

U = bt.Coefficient.sin_product(0.0, 1.0, math.pi)                 # u = sin(pi x) sin(pi y) sin(pi z)
F = bt.Coefficient.sin_product(0.0, 3.0 * math.pi ** 2, math.pi)  # -lap u
LIN = bt.Coefficient.affine(0.5, -1.0, 2.0, 0.25)


def fp(c):
    return (c.kind,) + tuple(c.c)


def host(fn, l):
    return fn.values[l].cpu().numpy()


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def poisson_rhs(g, l):
    """weak rhs of the model problem (test_solvers.cpp poisson_rhs): mass x interpolated f, zero Dirichlet"""
    f = bt.allocate(bt.p1_space(), g, l, l)
    bt.interpolate(f, l, F)
    b = bt.allocate(bt.p1_space(), g, l, l)
    bt.apply_elementwise(bt.FormId.mass(), f, b, l)
    bt.zero_dirichlet(b, l)
    return b


@pytest.mark.parametrize("text", [bt.cube_kuhn_text(), bt.cubes_mesh_text(2, 0.1, 0)])
def test_interpolate_and_l2_error_match_reference(text):
    g = bt.Grid(text, 2, 4)
    r = Reference(text, 2, 4)
    for l in (2, 3, 4):
        for f in (U, LIN):
            x = bt.allocate(bt.p1_space(), g, l, l)
            bt.interpolate(x, l, f)
            xr = r.interpolate(l, fp(f))
            assert rel(host(x, l), xr) <= 1e-14
            # replicas are broadcast from the owner: bitwise consistent
            y = bt.allocate(bt.p1_space(), g, l, l)
            y.values[l].copy_(x.values[l])
            bt.sync_broadcast(y, l)
            assert torch.equal(x.values[l], y.values[l])
            e = bt.l2_error(x, l, U)
            assert e == pytest.approx(r.l2_error(l, host(x, l), fp(U)), rel=1e-12)
    # interpolation of a linear field is exact; constant 1 against 0 integrates the volume
    x = bt.allocate(bt.p1_space(), g, 2, 2)
    bt.interpolate(x, 2, LIN)
    assert bt.l2_error(x, 2, LIN) <= 1e-13
    bt.assign(x, 2, 1.0)
    vol = r.l2_error(2, host(x, 2), (0, 0.0, 0, 0, 0)) ** 2
    assert bt.l2_error(x, 2, bt.Coefficient.constant(0.0)) ** 2 == pytest.approx(vol, rel=1e-12)


def test_l2_error_orders():
    g = bt.Grid(bt.cube_kuhn_text(), 2, 4)
    errs = []
    for l in (2, 3, 4):
        x = bt.allocate(bt.p1_space(), g, l, l)
        bt.interpolate(x, l, U)
        errs.append(bt.l2_error(x, l, U))
    assert errs[0] / errs[1] == pytest.approx(4.0, abs=1.0)
    assert errs[1] / errs[2] == pytest.approx(4.0, abs=1.0)


@pytest.mark.parametrize("kernel,text,hi", [(bt.KernelKind.Stencil, bt.cube_kuhn_text(), 5),
                                            (bt.KernelKind.Elementwise, bt.cubes_mesh_text(2, 0.1, 0), 4)])
def test_fmg_matches_reference(kernel, text, hi):
    lo = 2
    g = bt.Grid(text, lo, hi)
    form = bt.FormId.diffusion()
    h = bt.make_hierarchy(g, form, kernel)
    sm = bt.SmootherConfig.chebyshev(2)
    sm.nu1 = sm.nu2 = 2
    mg = bt.MultigridConfig(coarse_level=lo, cycles=5, coarse_tol=1e-12, coarse_maxit=4000)
    rhs = [poisson_rhs(g, l) for l in range(lo, hi + 1)]
    x = bt.allocate(bt.p1_space(), g, hi, hi)
    rep = bt.fmg(h, hi, rhs, x, sm, mg, exact=U)
    assert rep.iterations == 5 * (hi - lo) and len(rep.rows) == 1 + 5 * (hi - lo) and rep.converged

    r = Reference(text, lo, hi)
    r.make_hierarchy(form=0, kernel=1 if kernel == bt.KernelKind.Stencil else 0)
    rows, xr = r.fmg(hi, sm.as_array(), [host(b, lo + i) for i, b in enumerate(rhs)], lo, 5, fp=fp(U))
    assert len(rows) == len(rep.rows)
    for a, b in zip(rep.rows, rows):
        assert (a.level, a.cycle) == (int(b[0]), int(b[1]))
        assert a.residual == pytest.approx(b[2], rel=1e-8, abs=1e-15)
        assert a.error == pytest.approx(b[3], rel=1e-10)
    assert rel(host(x, hi), xr) <= 1e-10

    # reference-test properties: second-order errors per level, and the FMG
    # error tracks a tightly solved discrete error
    last = {row.level: row.error for row in rep.rows}
    if hi >= 4:
        assert 2.8 <= last[lo] / last[lo + 1] <= 4.7
        assert 3.4 <= last[hi - 1] / last[hi] <= 4.6
    tight = bt.allocate(bt.p1_space(), g, hi, hi)
    bt.impose_dirichlet(rhs[-1], tight, hi)
    bt.cg(h, rhs[-1], tight, hi, 1e-12, 20000)
    e_cg = bt.l2_error(tight, hi, U)
    assert abs(last[hi] - e_cg) <= 0.05 * e_cg


def test_one_level_fmg_is_the_coarse_solve():
    g = bt.Grid(bt.cube_kuhn_text(), 2, 2)
    h = bt.make_hierarchy(g, bt.FormId.diffusion())
    rhs = [poisson_rhs(g, 2)]
    x = bt.allocate(bt.p1_space(), g, 2, 2)
    mg = bt.MultigridConfig(coarse_level=2, cycles=5, coarse_tol=1e-12, coarse_maxit=4000)
    rep = bt.fmg(h, 2, rhs, x, bt.SmootherConfig.chebyshev(2), mg)
    assert len(rep.rows) == 1 and rep.rows[0].error == 0.0
    direct = bt.allocate(bt.p1_space(), g, 2, 2)
    bt.impose_dirichlet(rhs[0], direct, 2)
    bt.cg(h, rhs[0], direct, 2, 1e-12, 4000)
    assert float((x.values[2] - direct.values[2]).abs().max()) <= 1e-14


def test_fmg_argument_errors():
    g = bt.Grid(bt.cube_kuhn_text(), 2, 3)
    h = bt.make_hierarchy(g, bt.FormId.diffusion())
    x = bt.allocate(bt.p1_space(), g, 3, 3)
    mg = bt.MultigridConfig(coarse_level=2, cycles=1)
    with pytest.raises(bt.InvalidArgument):
        bt.fmg(h, 3, [poisson_rhs(g, 2)], x, bt.SmootherConfig.chebyshev(2), mg)  # one rhs per level
    with pytest.raises(bt.InvalidArgument):
        bt.fmg(h, 1, [], x, bt.SmootherConfig.chebyshev(2), mg)  # finest below coarse


@pytest.mark.parametrize("kernel", [bt.KernelKind.Stencil, bt.KernelKind.Elementwise])
def test_vcycle_graph_replay_matches_eager(kernel):
    """A V-cycle (coarse CG included: no host polls inside a capture) recorded
    into a CUDA graph replays bitwise like eager V-cycles."""
    text, lo, hi = bt.cubes_mesh_text(2, 0.1, 0), 2, 4
    g = bt.Grid(text, lo, hi)
    form = bt.FormId.diffusion() if kernel == bt.KernelKind.Stencil else \
        bt.FormId.div_k_grad(bt.Coefficient.sin_product(1.0, 0.5, 2 * math.pi))
    h = bt.make_hierarchy(g, form, kernel)
    sm = bt.SmootherConfig.chebyshev(2)
    mg = bt.MultigridConfig(coarse_level=lo, coarse_tol=0.0, coarse_maxit=30)
    rhs = bt.allocate(bt.p1_space(), g)
    bt.random_fill(rhs, hi, 0)
    bt.zero_dirichlet(rhs, hi)
    xe = bt.allocate(bt.p1_space(), g)
    xg = bt.allocate(bt.p1_space(), g)
    bt.v_cycle(h, hi, rhs, xe, sm, mg)  # warm-up: spectral estimates, buffers
    xg.values[hi].copy_(xe.values[hi])
    for _ in range(3):
        bt.v_cycle(h, hi, rhs, xe, sm, mg)
    graph = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            bt.v_cycle(h, hi, rhs, xg, sm, mg)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(xg.values[hi], xe.values[hi])
