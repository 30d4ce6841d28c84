"""N1E1 curl-curl + mass on the GPU against the N1E1 restatement in the
oracle (parity UNPINNED against the reference, which has no such operator;
the restatement is self-pinned in test_n1e1_oracle.py)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2308_01792_b200 as bt  # noqa: E402
from pyoracle import Oracle, cube_kuhn_text, cubes_mesh_text, ref_tet_text  # noqa: E402

REL = 1e-12
MESHES = {"ref_tet": ref_tet_text(), "kuhn": cube_kuhn_text(), "cubes2": cubes_mesh_text(2, 0.1, 0)}


def host(fn, l):
    torch.cuda.synchronize()
    return fn.values[l].cpu().numpy()


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("mesh", list(MESHES))
@pytest.mark.parametrize("l", [2, 3])
def test_n1e1_parity(mesh, l):
    g = bt.Grid(MESHES[mesh], l, l)
    o = Oracle(MESHES[mesh], l, l)
    x = bt.allocate(bt.edge_space(), g)
    y = bt.allocate(bt.edge_space(), g)
    bt.random_fill(x, l, 11)
    xh = host(x, l)
    assert np.array_equal(xh, o.n1e1_random_fill(l, 11))          # signed-broadcast fill, bit-exact
    v = np.random.default_rng(2).standard_normal(o.size(2, l))
    y.values[l].copy_(torch.from_numpy(v))
    bt.sync_additive(y, l)
    assert np.array_equal(host(y, l), o.n1e1_sync(l, v))          # signed replica sum, bit-exact
    assert bt.dot(x, x, l) == pytest.approx(o.dot(l, xh, xh, space=2), rel=1e-13)
    for alpha, beta in ((1.0, 1.0), (1.0, 0.0), (0.0, 1.0), (2.5, 0.5)):
        op = bt.N1E1Operator(g, l, alpha, beta)
        for bc in (bt.BC.None_, bt.BC.DirichletIdentity):
            bt.apply_n1e1(op, x, y, l, bc)
            assert rel(host(y, l), o.n1e1_apply(l, xh, alpha, beta, int(bc))) <= REL


@pytest.mark.parametrize("l", [5, 6])
def test_n1e1_parity_several_column_blocks(l):
    """Levels 5 and 6: the staged kernel's rows span 2 or 3 column blocks of 30 (and layer 0 and the diagonal end
    fall into blocks b >= 1)."""
    text = cube_kuhn_text()
    g = bt.Grid(text, l, l)
    o = Oracle(text, l, l)
    x = bt.allocate(bt.edge_space(), g)
    y = bt.allocate(bt.edge_space(), g)
    bt.random_fill(x, l, 5)
    xh = host(x, l)
    op = bt.N1E1Operator(g, l, 1.0, 1.0)
    for bc in (bt.BC.None_, bt.BC.DirichletIdentity):
        bt.apply_n1e1(op, x, y, l, bc)
        assert rel(host(y, l), o.n1e1_apply(l, xh, 1.0, 1.0, int(bc))) <= REL


def test_n1e1_config4_family_properties():
    """Config 4 family (perturbed Kuhn cubes, tangential Dirichlet): curl grad
    = 0 and symmetry at level 5 on 48 macro-tets, oracle parity at level 3."""
    text = cubes_mesh_text(2, 0.1, 0)
    l = 5
    g = bt.Grid(text, l, l)
    o = Oracle(text, l, l, with_edges=True)
    phi = o.random_fill(l, 3)
    u = bt.allocate(bt.edge_space(), g)
    u.values[l].copy_(torch.from_numpy(o.n1e1_gradient(l, phi)))
    ku = bt.allocate(bt.edge_space(), g)
    bt.apply_n1e1(bt.N1E1Operator(g, l, 1.0, 0.0), u, ku, l, bt.BC.None_)
    assert np.max(np.abs(host(ku, l))) <= 1e-11 * (1 << l) * np.max(np.abs(host(u, l)))
    op = bt.N1E1Operator(g, l, 1.0, 1.0)
    a, b, aa, ab = (bt.allocate(bt.edge_space(), g) for _ in range(4))
    bt.random_fill(a, l, 1)
    bt.random_fill(b, l, 2)
    bt.apply_n1e1(op, a, aa, l, bt.BC.None_)
    bt.apply_n1e1(op, b, ab, l, bt.BC.None_)
    s1, s2 = bt.dot(a, ab, l), bt.dot(b, aa, l)
    assert abs(s1 - s2) <= 1e-12 * abs(s1)
    assert rel(host(aa, l), o.n1e1_apply(l, host(a, l), 1.0, 1.0, 0)) <= REL


def test_n1e1_config4_full_size_properties():
    """Config 4 at full size (384 perturbed tets, L7, 958 M edge slots; no
    reference N1E1 exists and the CPU oracle is too slow at this size):
    symmetry of alpha K + beta M in the owned inner product, and bitwise
    repeatability of the apply."""
    text, l = cubes_mesh_text(4, 0.1, 0), 7
    g = bt.Grid(text, l, l)
    op = bt.N1E1Operator(g, l)
    u, v, au, av = (bt.allocate(bt.edge_space(), g, l, l) for _ in range(4))
    bt.random_fill(u, l, 1)
    bt.random_fill(v, l, 2)
    bt.apply_n1e1(op, u, au, l, bt.BC.None_)
    bt.apply_n1e1(op, v, av, l, bt.BC.None_)
    a, b = bt.dot(u, av, l), bt.dot(v, au, l)
    assert abs(a - b) <= 1e-11 * max(abs(a), 1.0)
    first = au.values[l].clone()
    bt.apply_n1e1(op, u, au, l, bt.BC.None_)
    assert torch.equal(au.values[l], first)


@pytest.mark.parametrize("l", [3, 4])
def test_n1e1_config4_mesh_against_oracle(l):
    """The config-4 mesh itself (4x4x4 perturbed Kuhn cubes, 384 macro-tets)
    at levels 3 and 4 against the N1E1 restatement: random fill (bitwise),
    signed replica sync (bitwise) and the apply with both boundary conditions
    (tangential Dirichlet identity rows) within 1e-12."""
    text = cubes_mesh_text(4, 0.1, 0)
    g = bt.Grid(text, l, l)
    o = Oracle(text, l, l)
    x = bt.allocate(bt.edge_space(), g)
    y = bt.allocate(bt.edge_space(), g)
    bt.random_fill(x, l, 0)
    xh = host(x, l)
    assert np.array_equal(xh, o.n1e1_random_fill(l, 0))
    v = np.random.default_rng(4).standard_normal(o.size(2, l))
    y.values[l].copy_(torch.from_numpy(v))
    bt.sync_additive(y, l)
    assert np.array_equal(host(y, l), o.n1e1_sync(l, v))
    op = bt.N1E1Operator(g, l, 1.0, 1.0)
    for bc in (bt.BC.None_, bt.BC.DirichletIdentity):
        bt.apply_n1e1(op, x, y, l, bc)
        assert rel(host(y, l), o.n1e1_apply(l, xh, 1.0, 1.0, int(bc))) <= REL
