"""Generates tests/golden/golden.npz from the compiled reference
(oracle/_ref/libbtref.so = /root/reference/proj/include/blocktet built by
oracle/Makefile). Run here, where /root/reference is mounted:

    make -C oracle && python tests/golden/make_golden.py

The fixtures pin the C restatement (tests/test_oracle_golden.py) and the CUDA
path (tests/test_gpu_parity.py) on machines without the reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
from pyoracle import Reference, cube_kuhn_text, kparams, ref_tet_text, TWO_TETS  # noqa: E402

CHEB = [2, 0.8, 2, 0.25, 1.1, 2, 2]  # SmootherConfig::chebyshev(2), V(2,2)


def main():
    out = {}
    # config 1: ref-tet L6, random_fill(seed 0), zero_dirichlet, apply_stencil(DirichletIdentity)
    r = Reference(ref_tet_text(), 6, 6)
    x = r.zero_dirichlet(6, r.random_fill(6, 0))
    y = r.apply_stencil(6, x, bc=1)
    idx = np.arange(0, x.size, 97)
    out["cfg1_idx"] = idx
    out["cfg1_x_sample"] = x[idx]
    out["cfg1_y_sample"] = y[idx]
    out["cfg1_y_sum_norm"] = np.array([np.sum(y), np.linalg.norm(y)])
    out["cfg1_rows"] = r.stencil_rows(0, 6)[0]
    # Kuhn cube L2..4: fills, applies, transfers, V-cycles
    k = Reference(cube_kuhn_text(), 2, 4)
    for l in (2, 3, 4):
        xk = k.random_fill(l, 31 * l)
        out[f"kuhn{l}_x"] = xk
        out[f"kuhn{l}_stencil_bc"] = k.apply_stencil(l, xk, bc=1)
        out[f"kuhn{l}_stencil"] = k.apply_stencil(l, xk, bc=0)
        out[f"kuhn{l}_mass"] = k.apply_stencil(l, xk, bc=1, form=1)
        out[f"kuhn{l}_ew_sin"] = k.apply_elementwise(l, xk, 2, kparams(), bc=1)
        out[f"kuhn{l}_diag_sin"] = k.extract_diagonal(l, 2, kparams())
        out[f"kuhn{l}_dot"] = np.array([k.dot(l, xk, xk)])
        for g in range(8):
            o, d = k.masks(l, 1, g)
            out[f"kuhn{l}_masks_c1_g{g}"] = np.stack([o, d])
    for l in (3, 4):
        out[f"kuhn{l}_prolong"] = k.prolongate(l, out[f"kuhn{l-1}_x"])
        out[f"kuhn{l}_restrict"] = k.restrict(l, out[f"kuhn{l}_x"])
    k.make_hierarchy(2, kparams(), 0)
    rhs = k.zero_dirichlet(4, k.random_fill(4, 0))
    x0 = np.zeros_like(rhs)
    xs, hist = k.vcycles(4, CHEB, rhs, x0, 3, 2, 0.0, 50)
    out["kuhn_vcycle_rhs"] = rhs
    out["kuhn_vcycle_hist"] = hist
    out["kuhn_vcycle_x"] = xs
    out["kuhn_lambda4"] = np.array([k.lambda_max(4)])
    # two glued tets, P2 sync (edge replica bookkeeping)
    t = Reference(TWO_TETS, 2, 2)
    out["two_p2_fill"] = t.random_fill(2, 99, space=1)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
