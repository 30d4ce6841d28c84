"""Pins the C restatement (oracle/bt_oracle.c) to the compiled reference
(oracle/_ref/libbtref.so): bit-for-bit on every hot-path function."""
import numpy as np
import pytest

from conftest import requires_reference
from pyoracle import Oracle, Reference, TWO_TETS, cube_kuhn_text, cubes_mesh_text, kparams, ref_tet_text

pytestmark = requires_reference

MESHES = {
    "ref_tet": (ref_tet_text(), 2, 4),
    "kuhn": (cube_kuhn_text(), 2, 4),
    "two_tets": (TWO_TETS, 2, 3),
    "cubes2_perturbed": (cubes_mesh_text(2, 0.1, 0), 2, 3),
    "released_faces": (cube_kuhn_text() + "boundary 2\n0 1 3 0\n0 2 3 0\n", 2, 3),
}
SMOOTHERS = {"cheb": [2, 0.8, 2, 0.25, 1.1, 2, 2], "jacobi": [0, 0.8, 2, 0.25, 1.1, 1, 1],
             "gs": [1, 0.8, 2, 0.25, 1.1, 1, 1]}


@pytest.fixture(scope="module", params=list(MESHES))
def pair(request):
    text, lo, hi = MESHES[request.param]
    return Oracle(text, lo, hi), Reference(text, lo, hi)


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape
    assert np.array_equal(a, b), f"max diff {np.max(np.abs(a - b)) if a.size else 0}"


def test_mesh_and_grid(pair):
    o, r = pair
    same(o.mesh_cells()[0], r.mesh_cells())
    for l in range(o.lo, o.hi + 1):
        for c in range(o.ncells):
            for g in range(8):
                a, b = o.masks(l, c, g), r.masks(l, c, g)
                same(a[0], b[0])
                same(a[1], b[1])
        for u, v in zip(o.groups(l), r.groups(l)):
            same(u, v)


def test_vectors(pair):
    o, r = pair
    rng = np.random.default_rng(1)
    for l in range(o.lo, o.hi + 1):
        for sp in (0, 1, 2):
            assert o.size(sp, l) == r.size(sp, l)
            same(o.random_fill(l, 7, sp), r.random_fill(l, 7, sp))
            v = rng.standard_normal(o.size(sp, l))
            same(o.sync(l, v, False, sp), r.sync(l, v, False, sp))
            same(o.sync(l, v, True, sp), r.sync(l, v, True, sp))
            assert o.dot(l, v, v, sp) == r.dot(l, v, v, sp)
            assert o.owned_count(l, sp) == r.owned_count(l, sp)


def test_operators(pair):
    o, r = pair
    for l in range(o.lo, o.hi + 1):
        x = o.random_fill(l, 3)
        for form in (0, 1):
            ro, do = o.stencil_rows(form, l)
            rr, dr = r.stencil_rows(form, l)
            same(ro, rr)
            same(do, dr)
            for c in range(o.ncells):
                same(o.class_matrices(form, l, c), r.class_matrices(form, l, c))
            for bc in (0, 1):
                same(o.apply_stencil(l, x, bc, form), r.apply_stencil(l, x, bc, form))
                same(o.apply_elementwise(l, x, form, None, bc), r.apply_elementwise(l, x, form, None, bc))
        for kp in (kparams(), kparams(2, 1.0, 1.0, 0.5, 0.0), kparams(0, 2.0)):
            for bc in (0, 1):
                same(o.apply_elementwise(l, x, 2, kp, bc), r.apply_elementwise(l, x, 2, kp, bc))
                same(o.apply_elementwise(l, x, 2, kp, bc, y=x, add=True),
                     r.apply_elementwise(l, x, 2, kp, bc, y=x, add=True))
            same(o.extract_diagonal(l, 2, kp), r.extract_diagonal(l, 2, kp))
        if l > o.lo:
            xc = o.random_fill(l - 1, 5)
            same(o.prolongate(l, xc), r.prolongate(l, xc))
            same(o.restrict(l, x), r.restrict(l, x))


@pytest.mark.parametrize("form,kernel", [(0, 1), (2, 0), (1, 1)])
def test_solvers(pair, form, kernel):
    o, r = pair
    o.make_hierarchy(form, kparams(), kernel)
    r.make_hierarchy(form, kparams(), kernel)
    l = o.hi
    same(o.hier_diag(l), r.hier_diag(l))
    assert o.lambda_max(l) == r.lambda_max(l)
    rhs = o.zero_dirichlet(l, o.random_fill(l, 0))
    x0 = np.zeros_like(rhs)
    for name, sm in SMOOTHERS.items():
        if name == "gs" and kernel == 0:
            continue
        same(o.smooth(l, sm, rhs, x0), r.smooth(l, sm, rhs, x0))
        same(o.smooth(l, sm, rhs, x0, backward=True), r.smooth(l, sm, rhs, x0, backward=True))
        xa, ha = o.vcycles(l, sm, rhs, x0, 3, o.lo, 1e-14, 20)
        xb, hb = r.vcycles(l, sm, rhs, x0, 3, o.lo, 1e-14, 20)
        same(ha, hb)
        same(xa, xb)
    b = o.random_fill(o.lo, 9)
    xa, ha = o.cg(o.lo, b, np.zeros_like(b), 1e-10, 100)
    xb, hb = r.cg(o.lo, b, np.zeros_like(b), 1e-10, 100)
    same(ha, hb)
    same(xa, xb)


def test_level7_cells_build():
    """Lifted level guard: the reference builds level 7 on a copy; the oracle agrees."""
    o, r = Oracle(ref_tet_text(), 7, 7, with_edges=False), Reference(ref_tet_text(), 7, 7)
    x = o.random_fill(7, 0)
    same(x, r.random_fill(7, 0))
    same(o.apply_stencil(7, x, 1), r.apply_stencil(7, x, 1))
