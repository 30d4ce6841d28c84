"""Self-pinning of the N1E1 restatement (oracle/bt_oracle_n1e1.c). The
reference has no curl-curl operator, so parity is UNPINNED
against the reference; the restatement is pinned by identities:
Whitney duality and quadrature of the element matrices, curl grad = 0,
symmetry, u^T M u = |c|^2 |Omega| and K u = 0 for constant fields, and
consistency of the signed replica sync."""
import numpy as np
import pytest

from pyoracle import Oracle, cube_kuhn_text, cubes_mesh_text, n_tet, ref_tet_text, width_formula

LOC = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]


def whitney(X):
    """barycentric gradients and the basis evaluator on a tet with corners X"""
    J = np.stack([X[1] - X[0], X[2] - X[0], X[3] - X[0]], axis=1)
    inv = np.linalg.inv(J)
    g = np.zeros((4, 3))
    g[1:] = inv
    g[0] = -g[1:].sum(axis=0)

    def w(e, lam):
        a, b = LOC[e]
        return lam[a] * g[b] - lam[b] * g[a]

    return g, w, abs(np.linalg.det(J)) / 6


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_element_matrix_by_quadrature(seed):
    rng = np.random.default_rng(seed)
    X = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float) + 0.2 * rng.standard_normal((4, 3))
    o = Oracle(ref_tet_text(), 2, 2)
    M = o.n1e1_local(X, 0.0, 1.0)
    K = o.n1e1_local(X, 1.0, 0.0)
    g, w, vol = whitney(X)
    a, b = (5 + 3 * np.sqrt(5)) / 20, (5 - np.sqrt(5)) / 20
    Mq = np.zeros((6, 6))
    for q in range(4):
        lam = np.full(4, b)
        lam[q] = a
        for e in range(6):
            for f in range(6):
                Mq[e, f] += vol / 4 * w(e, lam) @ w(f, lam)
    assert np.allclose(M, Mq, rtol=1e-13, atol=1e-15)
    curl = np.array([2 * np.cross(g[LOC[e][0]], g[LOC[e][1]]) for e in range(6)])
    assert np.allclose(K, vol * curl @ curl.T, rtol=1e-13, atol=1e-15)
    # Whitney duality: the tangential integral of w_f along edge e is delta_ef
    t, wts = np.polynomial.legendre.leggauss(4)
    t, wts = 0.5 * (t + 1), 0.5 * wts
    for e, (p, q) in enumerate(LOC):
        for f in range(6):
            s = 0.0
            for ti, wi in zip(t, wts):
                lam = np.zeros(4)
                lam[p], lam[q] = 1 - ti, ti
                s += wi * w(f, lam) @ (X[q] - X[p])
            assert s == pytest.approx(1.0 if e == f else 0.0, abs=1e-13)
    assert np.all(np.linalg.eigvalsh(M) > 0)
    assert np.allclose(K, K.T) and np.allclose(M, M.T)


MESHES = [(ref_tet_text(), 1.0 / 6), (cube_kuhn_text(), 1.0), (cubes_mesh_text(2, 0.1, 0), 1.0)]


@pytest.mark.parametrize("mesh,volume", MESHES)
def test_global_identities(mesh, volume):
    l = 3
    o = Oracle(mesh, 2, l)
    phi = o.random_fill(l, 4)
    u = o.n1e1_gradient(l, phi)
    ku = o.n1e1_apply(l, u, 1.0, 0.0, 0)
    assert np.max(np.abs(ku)) <= 1e-12 * (1 << l) * np.max(np.abs(u))   # curl grad = 0
    x = o.n1e1_random_fill(l, 1)
    y = o.n1e1_random_fill(l, 2)
    ax, ay = o.n1e1_apply(l, x, 1.0, 1.0, 0), o.n1e1_apply(l, y, 1.0, 1.0, 0)
    assert o.dot(l, x, ay, 2) == pytest.approx(o.dot(l, y, ax, 2), rel=1e-12)   # symmetry
    c = np.array([0.3, -1.2, 0.7])
    uc = o.n1e1_constant_field(l, c)
    assert o.dot(l, uc, o.n1e1_apply(l, uc, 0.0, 1.0, 0), 2) == pytest.approx(c @ c * volume, rel=1e-12)
    assert np.max(np.abs(o.n1e1_apply(l, uc, 1.0, 0.0, 0))) <= 1e-12 * (1 << l)
    assert o.dot(l, x, ax, 2) > 0                                               # SPD on the free space


def test_signed_sync_consistency():
    """After the signed additive sync every replica equals sigma times the
    group sum; a signed broadcast of a consistent field is a no-op."""
    l = 3
    o = Oracle(cubes_mesh_text(2, 0.1, 0), 2, l)
    off, cell, g, t = o.groups(l)
    sign = o.n1e1_signs(l)
    assert set(np.unique(sign[g > 0])) == {-1, 1}   # opposite orientations occur across faces
    v = np.random.default_rng(0).standard_normal(o.size(2, l))
    s = o.n1e1_sync(l, v)
    sizes = [sum(n_tet(width_formula(q, l)) for q in range(1, q0)) for q0 in range(1, 9)]
    cs = sizes[-1]
    x = o.n1e1_random_fill(l, 5)
    for q in range(len(off) - 1):
        mem = [m for m in range(off[q], off[q + 1]) if g[m] > 0]
        if len(mem) < 2:
            continue
        slot = [cs * cell[m] + sizes[g[m] - 1] + t[m] for m in mem]
        vals = [s[k] * sign[m] for k, m in zip(slot, mem)]
        assert max(vals) == min(vals)
        raw = sum(v[k] * sign[m] for k, m in zip(slot, mem))
        assert vals[0] == pytest.approx(raw, rel=1e-14, abs=1e-14)
        # the signed-broadcast random fill is orientation-consistent
        assert len({x[k] * sign[m] for k, m in zip(slot, mem)}) == 1
