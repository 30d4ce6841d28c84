"""Config 5's protocol as a parity test against the compiled reference
(oracle/_ref/libbtref.so, the unmodified blocktet headers): geometric
multigrid V(2,2)-cycles with Chebyshev(2)-Jacobi smoothing (lambda_max from
estimate_lambda_max), linear transfers, a coarse level-2 CG of exactly 50
iterations (coarse_tol 0), variable-coefficient P1 elementwise operator
k = 1 + 0.5 sin(2 pi x) sin(2 pi y) sin(2 pi z), rhs = random_fill(seed 0) +
zero_dirichlet, x0 = 0, 5 cycles (solvers.hpp:140-172, 425-456, 509-541).
Reduced instance: 2x2x2 perturbed Kuhn cubes (48 macro-tets), levels 2 -> 5
(the full 3,072-tet L2 -> 8 problem holds 70 GB per vector)."""
import math

import numpy as np
import pytest
import torch

import paper_2308_01792_b200 as bt
import pyoracle

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("n,lo,hi", [(2, 2, 5)])
def test_config5_protocol_against_reference(n, lo, hi):
    text = bt.cubes_mesh_text(n, 0.1, 0)
    form = bt.FormId.div_k_grad(bt.Coefficient.sin_product(1.0, 0.5, 2 * math.pi))
    sm = bt.SmootherConfig.chebyshev(2)
    sm.nu1 = sm.nu2 = 2
    mg = bt.MultigridConfig(coarse_level=lo, cycles=5, coarse_tol=0.0, coarse_maxit=50)
    g = bt.Grid(text, lo, hi)
    h = bt.make_hierarchy(g, form, bt.KernelKind.Elementwise)
    rhs = bt.allocate(bt.p1_space(), g)
    x = bt.allocate(bt.p1_space(), g)
    r = bt.allocate(bt.p1_space(), g, hi, hi)
    bt.random_fill(rhs, hi, 0)
    bt.zero_dirichlet(rhs, hi)
    nb = bt.norm2(rhs, hi)
    hist = [1.0]
    for _ in range(5):
        bt.v_cycle(h, hi, rhs, x, sm, mg)
        bt.hierarchy_apply(h, x, r, hi)
        r.values[hi].mul_(-1.0).add_(rhs.values[hi])
        hist.append(bt.norm2(r, hi) / nb)
    torch.cuda.synchronize()
    ref = pyoracle.Reference(text, lo, hi)
    ref.make_hierarchy(form=2, kp=pyoracle.kparams(), kernel=0, threads=8)
    xr, href = ref.vcycles(hi, sm.as_array(), rhs.values[hi].cpu().numpy(),
                           np.zeros(g.space_size(0, hi)), 5, lo, 0.0, 50)
    assert hist[-1] < 1e-3 * hist[0]                       # the cycles converge
    assert rel(hist[1:], href[1:]) <= 1e-12                # residual history
    assert rel(x.values[hi].cpu().numpy(), xr) <= 1e-12    # solution after 5 cycles
