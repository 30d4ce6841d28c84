"""Partitioned grids through the public API: every P1 entry
point — apply_stencil, apply_elementwise, extract_diagonal, dot, transfers,
hierarchies, Chebyshev smoothing, coarse CG and the V-cycle — runs as a
collective on memory-sharded vectors, with the library calling the grid's
allreduce hook itself.

One process plays R ranks as R host threads on one GPU. The hook syncs the
device, then the threads meet at a barrier and sum the buffers: no kernel
ever waits on another rank's kernel. Every rank's slice must equal the
single-handle result bitwise, and every dot / residual norm must be equal
bitwise (replica sums in member order; dots as per-cell partials summed in
cell order)."""
import math
import threading

import pytest
import torch

import paper_2308_01792_b200 as bt

pytestmark = pytest.mark.gpu


class VirtualComm:
    def __init__(self, nranks):
        self.n = nranks
        self.bar = threading.Barrier(nranks, timeout=300)
        self.bufs = [None] * nranks

    def hook(self, r):
        def allreduce(t):
            torch.cuda.synchronize()
            self.bufs[r] = t
            self.bar.wait()
            total = self.bufs[0].clone()
            for q in range(1, self.n):
                total += self.bufs[q]
            torch.cuda.synchronize()
            self.bar.wait()  # every rank has read every buffer
            t.copy_(total)
            torch.cuda.synchronize()
        return allreduce


def run_ranks(nranks, body):
    """body(rank, grid_setup) on nranks threads; grid_setup(g) partitions g."""
    comm = VirtualComm(nranks)
    results, errors = [None] * nranks, []

    def worker(r):
        try:
            results[r] = body(lambda g: g.set_partition(r, nranks, allreduce=comm.hook(r)))
        except BaseException as e:  # noqa: BLE001 - reraised below
            errors.append(e)
            comm.bar.abort()

    threads = [threading.Thread(target=worker, args=(r,)) for r in range(nranks)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return results


def var_form():
    return bt.FormId.div_k_grad(bt.Coefficient.sin_product(1.0, 0.5, 2 * math.pi))


def operators_body(text, L):
    def body(setup):
        g = bt.Grid(text, 2, L)
        setup(g)
        out = {"part": g.partition()}
        x = bt.allocate(bt.p1_space(), g)
        y = bt.allocate(bt.p1_space(), g)
        bt.random_fill(x, L, 7)
        out["x"] = x.values[L].clone()
        t = bt.compute_stencil(bt.FormId.diffusion(), g, L)
        for bc in (bt.BC.None_, bt.BC.DirichletIdentity):
            bt.apply_stencil(t, x, y, L, bc)
            out[f"stencil{int(bc)}"] = y.values[L].clone()
        bt.apply_elementwise(var_form(), x, y, L, bc=bt.BC.DirichletIdentity)
        out["elementwise"] = y.values[L].clone()
        out["dot"] = bt.dot(x, y, L)
        d = bt.allocate(bt.p1_space(), g)
        bt.extract_diagonal(var_form(), d, L)
        out["diag_ew"] = d.values[L].clone()
        bt.extract_diagonal(t, d, L)
        out["diag_stencil"] = d.values[L].clone()
        c = bt.allocate(bt.p1_space(), g)
        bt.restrict_p1(x, c, L)
        out["restrict"] = c.values[L - 1].clone()
        f = bt.allocate(bt.p1_space(), g)
        bt.prolongate_p1(c, f, L)
        out["prolongate"] = f.values[L].clone()
        bt.sync_additive(f, L)
        out["sync"] = f.values[L].clone()
        torch.cuda.synchronize()
        return out
    return body


def check_slices(full, ranks, L, keys_fine, keys_coarse):
    cs = {L: bt.n_tet((1 << L) + 1), L - 1: bt.n_tet((1 << (L - 1)) + 1)}
    for out in ranks:
        _, _, b, e = out["part"]
        for k in keys_fine:
            assert torch.equal(out[k], full[k][b * cs[L]:e * cs[L]]), k
        for k in keys_coarse:
            assert torch.equal(out[k], full[k][b * cs[L - 1]:e * cs[L - 1]]), k


@pytest.mark.parametrize("text,L,nranks", [(bt.cube_kuhn_text(), 5, 2), (bt.cube_kuhn_text(), 4, 4),
                                           (bt.cubes_mesh_text(2, 0.1, 0), 4, 3)])
def test_partitioned_operators(text, L, nranks):
    body = operators_body(text, L)
    full = body(lambda g: None)
    ranks = run_ranks(nranks, body)
    check_slices(full, ranks, L, ["x", "stencil0", "stencil1", "elementwise", "diag_ew", "diag_stencil",
                                  "prolongate", "sync"], ["restrict"])
    for out in ranks:
        assert out["dot"] == full["dot"]


def vcycle_body(text, lo, hi, kernel):
    def body(setup):
        g = bt.Grid(text, lo, hi)
        setup(g)
        form = var_form() if kernel == bt.KernelKind.Elementwise else bt.FormId.diffusion()
        h = bt.make_hierarchy(g, form, kernel)
        rhs = bt.allocate(bt.p1_space(), g)
        x = bt.allocate(bt.p1_space(), g)
        r = bt.allocate(bt.p1_space(), g, hi, hi)
        bt.random_fill(rhs, hi, 0)
        bt.zero_dirichlet(rhs, hi)
        sm = bt.SmootherConfig.chebyshev(2)
        sm.nu1 = sm.nu2 = 2
        mg = bt.MultigridConfig(coarse_level=lo, cycles=1, coarse_tol=0.0, coarse_maxit=20)
        hist = []
        for _ in range(2):
            bt.v_cycle(h, hi, rhs, x, sm, mg)
            bt.hierarchy_apply(h, x, r, hi)
            r.values[hi].mul_(-1.0).add_(rhs.values[hi])
            hist.append(bt.norm2(r, hi))
        rep = bt.cg(h, rhs, x, hi, 0.0, 5)
        torch.cuda.synchronize()
        return {"part": g.partition(), "x": x.values[hi].clone(), "hist": hist, "cg": list(rep.residuals)}
    return body


@pytest.mark.parametrize("kernel,text,lo,hi,nranks", [
    (bt.KernelKind.Elementwise, bt.cubes_mesh_text(2, 0.1, 0), 2, 4, 3),
    (bt.KernelKind.Stencil, bt.cube_kuhn_text(), 2, 5, 2),
])
def test_partitioned_vcycle(kernel, text, lo, hi, nranks):
    body = vcycle_body(text, lo, hi, kernel)
    full = body(lambda g: None)
    assert full["hist"][1] < full["hist"][0]
    ranks = run_ranks(nranks, body)
    cs = bt.n_tet((1 << hi) + 1)
    for out in ranks:
        _, _, b, e = out["part"]
        assert torch.equal(out["x"], full["x"][b * cs:e * cs])
        assert out["hist"] == full["hist"]
        assert out["cg"] == full["cg"]


def test_partitioned_without_hook_raises():
    g = bt.Grid(bt.cube_kuhn_text(), 2, 3)
    bt.api._check(bt.api._L.bt_grid_set_partition(g.handle, 0, 2))  # no allreduce hook
    x = bt.allocate(bt.p1_space(), g, 3, 3)
    with pytest.raises(bt.LogicError):
        bt.sync_additive(x, 3)
    with pytest.raises(bt.LogicError):
        bt.dot(x, x, 3)


def fmg_body(text, lo, hi):
    U = bt.Coefficient.sin_product(0.0, 1.0, math.pi)
    F = bt.Coefficient.sin_product(0.0, 3.0 * math.pi ** 2, math.pi)

    def body(setup):
        g = bt.Grid(text, lo, hi)
        setup(g)
        h = bt.make_hierarchy(g, bt.FormId.diffusion(), bt.KernelKind.Elementwise)
        rhs = []
        for l in range(lo, hi + 1):
            f = bt.allocate(bt.p1_space(), g, l, l)
            bt.interpolate(f, l, F)
            b = bt.allocate(bt.p1_space(), g, l, l)
            bt.apply_elementwise(bt.FormId.mass(), f, b, l)
            bt.zero_dirichlet(b, l)
            rhs.append(b)
        x = bt.allocate(bt.p1_space(), g, hi, hi)
        sm = bt.SmootherConfig.chebyshev(2)
        sm.nu1 = sm.nu2 = 2
        mg = bt.MultigridConfig(coarse_level=lo, cycles=2, coarse_tol=0.0, coarse_maxit=30)
        rep = bt.fmg(h, hi, rhs, x, sm, mg, exact=U)
        torch.cuda.synchronize()
        return {"part": g.partition(), "x": x.values[hi].clone(),
                "rows": [(r.level, r.cycle, r.residual, r.error) for r in rep.rows]}
    return body


def test_partitioned_fmg():
    text, lo, hi = bt.cubes_mesh_text(2, 0.1, 0), 2, 4
    body = fmg_body(text, lo, hi)
    full = body(lambda g: None)
    ranks = run_ranks(3, body)
    cs = bt.n_tet((1 << hi) + 1)
    for out in ranks:
        _, _, b, e = out["part"]
        assert torch.equal(out["x"], full["x"][b * cs:e * cs])
        assert out["rows"] == full["rows"]  # residuals and L2 errors bitwise


def n1e1_body(text, L):
    def body(setup):
        g = bt.Grid(text, 2, L)
        setup(g)
        op = bt.N1E1Operator(g, L)
        x = bt.allocate(bt.edge_space(), g, L, L)
        y = bt.allocate(bt.edge_space(), g, L, L)
        bt.random_fill(x, L, 5)
        out = {"part": g.partition(), "x": x.values[L].clone()}
        for bc in (bt.BC.None_, bt.BC.DirichletIdentity):
            bt.apply_n1e1(op, x, y, L, bc)
            out[f"y{int(bc)}"] = y.values[L].clone()
        out["dot"] = bt.dot(x, y, L)
        bt.sync_additive(x, L)
        out["sync"] = x.values[L].clone()
        torch.cuda.synchronize()
        return out
    return body


@pytest.mark.parametrize("text,L,nranks", [(bt.cube_kuhn_text(), 4, 2), (bt.cubes_mesh_text(2, 0.1, 0), 3, 3)])
def test_partitioned_n1e1(text, L, nranks):
    body = n1e1_body(text, L)
    full = body(lambda g: None)
    ranks = run_ranks(nranks, body)
    g = bt.Grid(text, 2, L)
    cs = g.space_size(2, L) // g.n_cells()
    for out in ranks:
        _, _, b, e = out["part"]
        for k in ("x", "y0", "y1", "sync"):
            assert torch.equal(out[k], full[k][b * cs:e * cs]), k
        assert out["dot"] == full["dot"]


def test_more_ranks_than_cells():
    """8 ranks on 6 cells: two ranks hold no cell and still take part in every collective."""
    text, L = bt.cube_kuhn_text(), 4
    body = operators_body(text, L)
    full = body(lambda g: None)
    ranks = run_ranks(8, body)
    assert any(out["part"][2] == out["part"][3] for out in ranks)  # an empty block
    check_slices(full, ranks, L, ["x", "stencil0", "stencil1", "elementwise", "diag_ew", "diag_stencil",
                                  "prolongate", "sync"], ["restrict"])
    for out in ranks:
        assert out["dot"] == full["dot"]
    vb = vcycle_body(text, 2, 4, bt.KernelKind.Stencil)
    vfull = vb(lambda g: None)
    cs = bt.n_tet((1 << 4) + 1)
    for out in run_ranks(8, vb):
        _, _, b, e = out["part"]
        assert torch.equal(out["x"], vfull["x"][b * cs:e * cs])
        assert out["hist"] == vfull["hist"] and out["cg"] == vfull["cg"]


def test_more_ranks_than_cells_n1e1_and_fmg():
    text = bt.cube_kuhn_text()
    nb = n1e1_body(text, 3)
    full = nb(lambda g: None)
    g = bt.Grid(text, 2, 3)
    cs = g.space_size(2, 3) // g.n_cells()
    for out in run_ranks(8, nb):
        _, _, b, e = out["part"]
        for k in ("x", "y0", "y1", "sync"):
            assert torch.equal(out[k], full[k][b * cs:e * cs]), k
        assert out["dot"] == full["dot"]
    fb = fmg_body(text, 2, 4)
    ffull = fb(lambda g: None)
    cs = bt.n_tet((1 << 4) + 1)
    for out in run_ranks(8, fb):
        _, _, b, e = out["part"]
        assert torch.equal(out["x"], ffull["x"][b * cs:e * cs])
        assert out["rows"] == ffull["rows"]


def gs_body(text, lo, hi):
    def body(setup):
        g = bt.Grid(text, lo, hi)
        setup(g)
        h = bt.make_hierarchy(g, bt.FormId.diffusion(), bt.KernelKind.Stencil)
        rhs = bt.allocate(bt.p1_space(), g)
        x = bt.allocate(bt.p1_space(), g)
        bt.random_fill(rhs, hi, 0)
        bt.zero_dirichlet(rhs, hi)
        gs = bt.SmootherConfig.gauss_seidel()
        bt.smooth(h, gs, rhs, x, hi, 2)
        bt.smooth(h, gs, rhs, x, hi, 1, bt.SweepDirection.Backward)
        mg = bt.MultigridConfig(coarse_level=lo, coarse_tol=0.0, coarse_maxit=20)
        for _ in range(2):
            bt.v_cycle(h, hi, rhs, x, gs, mg)  # the reference's default smoother
        torch.cuda.synchronize()
        return {"part": g.partition(), "x": x.values[hi].clone()}
    return body


@pytest.mark.parametrize("nranks", [2, 3])
def test_partitioned_gauss_seidel(nranks):
    text, lo, hi = bt.cubes_mesh_text(2, 0.1, 0), 2, 4
    body = gs_body(text, lo, hi)
    full = body(lambda g: None)
    cs = bt.n_tet((1 << hi) + 1)
    for out in run_ranks(nranks, body):
        _, _, b, e = out["part"]
        assert torch.equal(out["x"], full["x"][b * cs:e * cs])
