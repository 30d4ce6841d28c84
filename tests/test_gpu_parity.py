"""Parity of the CUDA product path (libbt_b200.so through its C ABI) with the
oracle (C restatement pinned bit-for-bit to the reference, see
test_oracle_vs_ref.py / test_oracle_golden.py).

Bars (BASELINE.json north_star): index maps, DoF layouts, masks, groups,
random inputs and transfers are bit-exact; fp64 operator applies, diagonals
and V-cycle residual histories within relative L2 1e-12 (REL below).
"""
import math
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2308_01792_b200 as bt  # noqa: E402
from pyoracle import Oracle, TWO_TETS, cube_kuhn_text, cubes_mesh_text, kparams, ref_tet_text  # noqa: E402

REL = 1e-12
G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))

MESHES = {
    "ref_tet": (ref_tet_text(), 2, 4),
    "kuhn": (cube_kuhn_text(), 2, 4),
    "two_tets": (TWO_TETS, 2, 3),
    "cubes2": (cubes_mesh_text(2, 0.1, 0), 2, 4),
    "released": (cube_kuhn_text() + "boundary 2\n0 1 3 0\n0 2 3 0\n", 2, 3),
}
SIN = bt.Coefficient.sin_product(1.0, 0.5, 2 * np.pi)
COEFFS = {
    "sin": (SIN, kparams(1, 1.0, 0.5, 2 * np.pi)),
    "affine": (bt.Coefficient.affine(1.0, 1.0, 0.5, 0.0), kparams(2, 1.0, 1.0, 0.5, 0.0)),
    "const2": (bt.Coefficient.constant(2.0), kparams(0, 2.0)),
}


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def host(fn, l):
    torch.cuda.synchronize()
    return fn.values[l].cpu().numpy()


def upload(fn, l, arr):
    fn.values[l].copy_(torch.from_numpy(np.ascontiguousarray(arr)))


@pytest.fixture(scope="module", params=list(MESHES))
def setup(request):
    text, lo, hi = MESHES[request.param]
    return bt.Grid(text, lo, hi), Oracle(text, lo, hi), lo, hi


def test_masks_and_groups_bit_exact(setup):
    g, o, lo, hi = setup
    for l in range(lo, hi + 1):
        for c in range(g.n_cells()):
            for s in range(8):
                a, b = g.masks(l, c, s), o.masks(l, c, s)
                assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        # P1 groups: the oracle's groups restricted to vertex members
        off, cell, sg, t = o.groups(l)
        ref = set()
        for q in range(len(off) - 1):
            mem = tuple((int(cell[m]), int(t[m])) for m in range(off[q], off[q + 1]) if sg[m] == 0)
            if len(mem) >= 2:
                ref.add(mem)
        off, cell, sg, t = g.groups(l)
        got = {tuple((int(cell[m]), int(t[m])) for m in range(off[q], off[q + 1])) for q in range(len(off) - 1)}
        assert got == ref


def test_vectors(setup):
    g, o, lo, hi = setup
    rng = np.random.default_rng(3)
    for l in range(lo, hi + 1):
        x = bt.allocate(bt.p1_space(), g, l, l)
        bt.random_fill(x, l, 17 + l)
        assert np.array_equal(host(x, l), o.random_fill(l, 17 + l))
        v = rng.standard_normal(o.size(0, l))
        upload(x, l, v)
        bt.sync_additive(x, l)
        assert np.array_equal(host(x, l), o.sync(l, v))
        upload(x, l, v)
        bt.sync_broadcast(x, l)
        assert np.array_equal(host(x, l), o.sync(l, v, broadcast=True))
        w = rng.standard_normal(o.size(0, l))
        y = bt.allocate(bt.p1_space(), g, l, l)
        upload(x, l, v)
        upload(y, l, w)
        assert bt.dot(x, y, l) == pytest.approx(o.dot(l, v, w), rel=1e-13)
        assert bt.owned_dof_count(x, l) == o.owned_count(l)
        bt.zero_dirichlet(x, l)
        assert np.array_equal(host(x, l), o.zero_dirichlet(l, v))
        bt.axpy(y, 0.75, x, l)
        assert np.array_equal(host(y, l), w + 0.75 * o.zero_dirichlet(l, v))


@pytest.mark.parametrize("form", ["diffusion", "mass"])
def test_apply_stencil(setup, form):
    g, o, lo, hi = setup
    fid = bt.FormId.diffusion() if form == "diffusion" else bt.FormId.mass()
    fk = 0 if form == "diffusion" else 1
    for l in range(lo, hi + 1):
        table = bt.compute_stencil(fid, g, l)
        rows, diag = o.stencil_rows(fk, l)
        assert np.array_equal(table.rows, rows)                      # compute_stencil rows: bit-exact
        assert np.array_equal(table.diagonal().cpu().numpy(), diag)   # assembled diagonal: bit-exact
        x = bt.allocate(bt.p1_space(), g, l, l)
        y = bt.allocate(bt.p1_space(), g, l, l)
        for seed in (1, 977):
            bt.random_fill(x, l, seed)
            xh = host(x, l)
            for bc in (bt.BC.None_, bt.BC.DirichletIdentity):
                bt.apply_stencil(table, x, y, l, bc)
                assert rel(host(y, l), o.apply_stencil(l, xh, int(bc), fk)) <= REL


@pytest.mark.parametrize("coeff", list(COEFFS))
def test_apply_elementwise(setup, coeff):
    g, o, lo, hi = setup
    cf, kp = COEFFS[coeff]
    forms = [(bt.FormId.div_k_grad(cf), 2, kp), (bt.FormId.diffusion(), 0, None), (bt.FormId.mass(), 1, None)]
    for l in range(lo, hi + 1):
        x = bt.allocate(bt.p1_space(), g, l, l)
        y = bt.allocate(bt.p1_space(), g, l, l)
        d = bt.allocate(bt.p1_space(), g, l, l)
        bt.random_fill(x, l, 5 * l)
        xh = host(x, l)
        for fid, fk, fkp in forms:
            for bc in (bt.BC.None_, bt.BC.DirichletIdentity):
                bt.apply_elementwise(fid, x, y, l, bt.ApplyMode.Replace, bc)
                ref = o.apply_elementwise(l, xh, fk, fkp, int(bc))
                assert rel(host(y, l), ref) <= REL
                before = host(y, l)
                bt.apply_elementwise(fid, x, y, l, bt.ApplyMode.Add, bc)
                assert rel(host(y, l), o.apply_elementwise(l, xh, fk, fkp, int(bc), y=before, add=True)) <= REL
            bt.extract_diagonal(fid, d, l)
            assert rel(host(d, l), o.extract_diagonal(l, fk, fkp)) <= REL


def test_transfers_bit_exact(setup):
    g, o, lo, hi = setup
    for l in range(lo + 1, hi + 1):
        c = bt.allocate(bt.p1_space(), g, l - 1, l)
        f = bt.allocate(bt.p1_space(), g, l - 1, l)
        bt.random_fill(c, l - 1, 7 * l)
        bt.random_fill(f, l, 7 * l + 1)
        ch, fh = host(c, l - 1), host(f, l)
        bt.prolongate_p1(c, f, l)
        assert np.array_equal(host(f, l), o.prolongate(l, ch))
        upload(f, l, fh)
        bt.restrict_p1(f, c, l)
        assert np.array_equal(host(c, l - 1), o.restrict(l, fh))
        # prolongate-and-add (v_cycle's axpy(x, 1, ef) fused)
        upload(f, l, fh)
        bt.prolongate_p1(c, f, l, add=True)
        assert np.array_equal(host(f, l), fh + o.prolongate(l, host(c, l - 1)))


SMOOTHERS = [("cheb", bt.SmootherConfig.chebyshev(2)), ("jacobi", bt.SmootherConfig.jacobi(0.8))]


@pytest.mark.parametrize("kernel", ["stencil", "elementwise"])
def test_hierarchy_smoothers_vcycle(setup, kernel):
    g, o, lo, hi = setup
    if kernel == "stencil":
        fid, fk, kern = bt.FormId.diffusion(), 0, bt.KernelKind.Stencil
    else:
        fid, fk, kern = bt.FormId.div_k_grad(SIN), 2, bt.KernelKind.Elementwise
    h = bt.make_hierarchy(g, fid, kern)
    o.make_hierarchy(fk, kparams(), 1 if kernel == "stencil" else 0)
    l = hi
    assert rel(h.diagonal(l).cpu().numpy(), o.hier_diag(l)) <= REL
    assert bt.spectral_estimate(h, l) == pytest.approx(o.lambda_max(l), rel=1e-12)
    rhs = bt.allocate(bt.p1_space(), g)
    x = bt.allocate(bt.p1_space(), g)
    bt.random_fill(rhs, l, 0)
    bt.zero_dirichlet(rhs, l)
    rh = host(rhs, l)
    for name, sm in SMOOTHERS:
        sm.nu1 = sm.nu2 = 2
        bt.assign(x, l, 0.0)
        bt.smooth(h, sm, rhs, x, l, 1)
        assert rel(host(x, l), o.smooth(l, sm.as_array(), rh, np.zeros_like(rh))) <= REL
        bt.assign(x, l, 0.0)
        mg = bt.MultigridConfig(coarse_level=lo, coarse_tol=1e-14, coarse_maxit=20)
        hist = []
        for _ in range(3):
            bt.v_cycle(h, l, rhs, x, sm, mg)
            r = bt.allocate(bt.p1_space(), g, l, l)
            bt.hierarchy_apply(h, x, r, l)
            bt.scale(r, l, -1.0)
            tmp = bt.allocate(bt.p1_space(), g, l, l)
            upload(tmp, l, rh)
            bt.axpy(r, 1.0, tmp, l)
            hist.append(bt.norm2(r, l) / bt.norm2(tmp, l))
        xo, ho = o.vcycles(l, sm.as_array(), rh, np.zeros_like(rh), 3, lo, 1e-14, 20)
        assert rel(hist, ho[1:]) <= REL
        assert rel(host(x, l), xo) <= REL
    b = bt.allocate(bt.p1_space(), g, lo, lo)
    xc = bt.allocate(bt.p1_space(), g, lo, lo)
    bt.random_fill(b, lo, 9)
    rep = bt.cg(h, b, xc, lo, 1e-10, 100)
    xo, ho = o.cg(lo, host(b, lo), np.zeros(o.size(0, lo)), 1e-10, 100)
    assert rep.iterations == len(ho)
    assert rel(rep.residuals, ho) <= 1e-9  # relative residuals near 1e-10 carry round-off
    assert rel(host(xc, lo), xo) <= REL


def test_config1_golden_and_repeat_bitwise():
    """Config 1: ref-tet L6, seed 0, zero Dirichlet, 1 + 10 applies."""
    g = bt.Grid(ref_tet_text(), 6, 6)
    table = bt.compute_stencil(bt.FormId.diffusion(), g, 6)
    assert np.array_equal(table.rows, G["cfg1_rows"])
    x = bt.allocate(bt.p1_space(), g)
    y = bt.allocate(bt.p1_space(), g)
    bt.random_fill(x, 6, 0)
    bt.zero_dirichlet(x, 6)
    bt.apply_stencil(table, x, y, 6, bt.BC.DirichletIdentity)
    y0 = host(y, 6)
    idx = G["cfg1_idx"]
    assert np.array_equal(host(x, 6)[idx], G["cfg1_x_sample"])
    assert rel(y0[idx], G["cfg1_y_sample"]) <= REL
    s, nrm = G["cfg1_y_sum_norm"]
    assert abs(np.sum(y0) - s) <= 1e-12 * nrm and abs(np.linalg.norm(y0) - nrm) <= 1e-12 * nrm
    for _ in range(10):
        bt.apply_stencil(table, x, y, 6, bt.BC.DirichletIdentity)
        assert np.array_equal(host(y, 6), y0)


def test_config2_full_size_against_oracle():
    """Config 2 at full size (cube-kuhn L8, 17.2 M slots): direct parity with
    the oracle plus size-independent properties."""
    text = cube_kuhn_text()
    g = bt.Grid(text, 8, 8)
    o = Oracle(text, 8, 8, with_edges=False)
    table = bt.compute_stencil(bt.FormId.diffusion(), g, 8)
    x = bt.allocate(bt.p1_space(), g)
    y = bt.allocate(bt.p1_space(), g)
    bt.random_fill(x, 8, 0)
    xh = host(x, 8)
    assert np.array_equal(xh, o.random_fill(8, 0))
    for bc in (0, 1):
        bt.apply_stencil(table, x, y, 8, bc)
        assert rel(host(y, 8), o.apply_stencil(8, xh, bc)) <= REL
    # A 1 = 0 without boundary rows
    bt.assign(x, 8, 1.0)
    bt.apply_stencil(table, x, y, 8)
    assert np.max(np.abs(host(y, 8))) <= 1e-11 * table.rows[0][0]
    # symmetry in the owned inner product and stencil == elementwise
    u = bt.allocate(bt.p1_space(), g)
    v = bt.allocate(bt.p1_space(), g)
    au = bt.allocate(bt.p1_space(), g)
    av = bt.allocate(bt.p1_space(), g)
    bt.random_fill(u, 8, 1)
    bt.random_fill(v, 8, 2)
    bt.apply_stencil(table, u, au, 8)
    bt.apply_stencil(table, v, av, 8)
    a, b = bt.dot(u, av, 8), bt.dot(v, au, 8)
    assert abs(a - b) <= 1e-12 * max(abs(a), 1.0)
    bt.apply_elementwise(bt.FormId.diffusion(), u, av, 8)
    assert rel(host(av, 8), host(au, 8)) <= REL


def test_config3_small_and_properties():
    """Config 3 family (perturbed 4^3 x 6 Kuhn tets, div(k grad), k = 1 +
    0.5 sin sin sin): oracle parity at L3, properties at L6 (full size)."""
    text = cubes_mesh_text(4, 0.1, 0)
    g = bt.Grid(text, 3, 6)
    o = Oracle(text, 3, 3, with_edges=False)
    f = bt.FormId.div_k_grad(SIN)
    x = bt.allocate(bt.p1_space(), g)
    y = bt.allocate(bt.p1_space(), g)
    bt.random_fill(x, 3, 0)
    bt.apply_elementwise(f, x, y, 3, bc=bt.BC.DirichletIdentity)
    assert rel(host(y, 3), o.apply_elementwise(3, host(x, 3), 2, kparams(), 1)) <= REL
    # L6: symmetry and k = 2 scaling of diffusion
    u, v, au, av = (bt.allocate(bt.p1_space(), g, 6, 6) for _ in range(4))
    bt.random_fill(u, 6, 11)
    bt.random_fill(v, 6, 12)
    bt.apply_elementwise(f, u, au, 6)
    bt.apply_elementwise(f, v, av, 6)
    a, b = bt.dot(u, av, 6), bt.dot(v, au, 6)
    assert abs(a - b) <= 1e-12 * max(abs(a), 1.0)
    bt.apply_elementwise(bt.FormId.div_k_grad(bt.Coefficient.constant(2.0)), u, au, 6)
    bt.apply_elementwise(bt.FormId.diffusion(), u, av, 6)
    assert rel(host(au, 6), 2.0 * host(av, 6)) <= REL


def test_config3_full_size_against_reference():
    """Config 3 at full size (384 perturbed tets, L6, div(k grad) with the sin
    product coefficient; 18.4 M slots): the elementwise apply (kbar once per
    micro-cell, on the fly) against
    the compiled reference, plus symmetry in the owned inner product."""
    from pyoracle import Reference
    text, l = cubes_mesh_text(4, 0.1, 0), 6
    g = bt.Grid(text, l, l)
    form = bt.FormId.div_k_grad(SIN)
    x = bt.allocate(bt.p1_space(), g)
    y = bt.allocate(bt.p1_space(), g)
    bt.random_fill(x, l, 0)
    bt.apply_elementwise(form, x, y, l)
    r = Reference(text, l, l)
    ref = r.apply_elementwise(l, host(x, l), form=2, kp=kparams(), threads=os.cpu_count() or 1)
    assert rel(host(y, l), ref) <= REL
    u, v, au, av = (bt.allocate(bt.p1_space(), g) for _ in range(4))
    bt.random_fill(u, l, 1)
    bt.random_fill(v, l, 2)
    bt.apply_elementwise(form, u, au, l)
    bt.apply_elementwise(form, v, av, l)
    a, b = bt.dot(u, av, l), bt.dot(v, au, l)
    assert abs(a - b) <= 1e-12 * max(abs(a), 1.0)


@pytest.mark.parametrize("l", [7])
def test_elementwise_column_tiles_against_reference(l):
    """Config-5 family (2x2x2 perturbed Kuhn cubes) at level 7, where rows are
    longer than one 64-column tile of the elementwise kernel: the apply (both
    BCs) and the assembled diagonal against the compiled reference, for the
    sin-product and an affine coefficient."""
    from pyoracle import Reference
    text = cubes_mesh_text(2, 0.1, 0)
    g = bt.Grid(text, l, l)
    r = Reference(text, l, l)
    x = bt.allocate(bt.p1_space(), g)
    y = bt.allocate(bt.p1_space(), g)
    d = bt.allocate(bt.p1_space(), g)
    bt.random_fill(x, l, 3)
    xh = host(x, l)
    aff = bt.Coefficient.affine(2.0, 0.3, -0.2, 0.1)
    for coeff, kp in ((SIN, kparams()), (aff, kparams(2, 2.0, 0.3, -0.2, 0.1))):
        form = bt.FormId.div_k_grad(coeff)
        for bc in (bt.BC.None_, bt.BC.DirichletIdentity):
            bt.apply_elementwise(form, x, y, l, bc=bc)
            ref = r.apply_elementwise(l, xh, form=2, kp=kp, bc=int(bc), threads=os.cpu_count() or 1)
            assert rel(host(y, l), ref) <= REL
        bt.extract_diagonal(form, d, l)
        assert rel(host(d, l), r.extract_diagonal(l, form=2, kp=kp)) <= REL


def test_div_k_grad_coefficient_must_be_positive():
    """local_matrix raises invalid_argument when k <= 0 at a quadrature point
    (forms.hpp:114); sin product with c0 <= |c1| is checked point by point."""
    g = bt.Grid(cube_kuhn_text(), 3, 3)
    x = bt.allocate(bt.p1_space(), g)
    y = bt.allocate(bt.p1_space(), g)
    with pytest.raises(bt.InvalidArgument):
        bt.apply_elementwise(bt.FormId.div_k_grad(bt.Coefficient.sin_product(0.2, 1.0, 2 * math.pi)), x, y, 3)
    with pytest.raises(bt.InvalidArgument):
        bt.apply_elementwise(bt.FormId.div_k_grad(bt.Coefficient.affine(0.5, -1.0, 0.0, 0.0)), x, y, 3)
    # positive on the mesh although c0 <= |c1|: accepted (k = 1.5 + 2 sin(pi x/8) ... > 0 on [0,1]^3)
    bt.apply_elementwise(bt.FormId.div_k_grad(bt.Coefficient.sin_product(1.5, 2.0, math.pi / 8)), x, y, 3)
