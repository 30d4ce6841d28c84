"""Index algebra of the product (C ABI host functions of libbt_b200.so)
against the oracle and the reference KATs (test_micro_index.cpp). Runs
without a GPU: these entry points are pure host code."""
import itertools

import numpy as np
import pytest

import paper_2308_01792_b200 as bt
from pyoracle import load_oracle

ORC = load_oracle()


def test_kats():
    assert [bt.n_tri(w) for w in (0, 1, 4)] == [0, 1, 10]
    assert [bt.n_tet(w) for w in (0, 1, 3, 4)] == [0, 1, 10, 20]
    assert bt.width(0, 2) == 5 and bt.width(7, 2) == 3 and bt.width(15, 2) == 3
    assert bt.width(20, 2) == 4 and bt.width(21, 2) == 2 and bt.width(21, 3) == 6
    assert bt.width(7, 1) == 1 and bt.width(0, 0) == 2
    with pytest.raises(bt.DomainError):
        bt.width(21, 1)
    with pytest.raises(bt.DomainError):
        bt.width(7, 0)
    assert bt.linearize(3, (0, 0, 0)) == 0 and bt.linearize(3, (0, 1, 0)) == 3 and bt.linearize(3, (0, 0, 1)) == 6
    with pytest.raises(bt.OutOfRange):
        bt.linearize_checked(3, (1, 1, 1))
    with pytest.raises(bt.OutOfRange):
        bt.delinearize(3, 10)
    assert bt.index_set(2) == [(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)]


@pytest.mark.parametrize("w", list(range(1, 21)) + [65, 129, 257])
def test_linearize_bijection(w):
    pos = 0
    step = 1 if w <= 20 else 997
    pts = bt.index_set(w) if w <= 20 else None
    if pts is not None:
        for p in pts:
            assert bt.linearize(w, p) == pos == ORC.bo_linearize(w, *p)
            assert bt.delinearize(w, pos) == p
            pos += 1
        assert pos == bt.n_tet(w)
    else:
        ijk = (bt._lib.C.c_int32 * 3)()
        for t in range(0, bt.n_tet(w), step):
            p = bt.delinearize(w, t)
            assert bt.linearize(w, p) == t
            ORC.bo_delinearize(w, t, ijk)
            assert tuple(ijk) == p


def test_widths_and_offsets_match_oracle():
    for g in range(26):
        for l in range(0, 11):
            assert bt.width_formula(g, l) == ORC.bo_width_formula(g, l)
        buf = (bt._lib.C.c_int32 * 12)()
        n = ORC.bo_subgroup_offsets(g, buf)
        assert bt.subgroup_offsets(g) == [tuple(buf[3 * i:3 * i + 3]) for i in range(n)]


def test_counting_identities():
    for l in (2, 3, 4, 8):
        n = 1 << l
        edges = sum(bt.n_tet(bt.width(g, l)) for g in range(1, 8))
        faces = sum(bt.n_tet(bt.width(g, l)) for g in range(8, 20))
        cells = sum(bt.n_tet(bt.width(g, l)) for g in range(20, 26))
        verts = bt.n_tet(bt.width(0, l))
        assert edges == 6 * bt.n_tet(n) + bt.n_tet(n - 1)
        assert faces == 2 * n ** 3 + 2 * n ** 2
        assert cells == n ** 3
        assert verts - edges + faces - cells == 1


def test_row_layout_offsets():
    """The stencil kernels' row-offset formulas (bt_index.cuh row_offsets,
    SURVEY Appendix A) against linearize for every interior point, w <= 24."""
    dirs = [(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1), (1, -1, 0), (1, 0, -1), (0, 1, -1), (1, -1, 1),
            (-1, 0, 0), (0, -1, 0), (0, 0, -1), (-1, 1, 0), (-1, 0, 1), (0, -1, 1), (-1, 1, -1)]
    for w in range(5, 25):
        for (i, j, k) in bt.index_set(w):
            if not (i >= 1 and j >= 1 and k >= 1 and i + j + k <= w - 2):
                continue
            L, m = w - j - k, w - k
            U = m * (m + 1) // 2 - j
            D = -((m + 1) * (m + 2) // 2 - j)
            off = [0, 1, L, U, -L, D + 1, D + L + 1, U - L + 1, -1, -(L + 1), D, L - 1, U - 1, U - L, D + L]
            t = bt.linearize(w, (i, j, k))
            for d, (dx, dy, dz) in enumerate(dirs):
                assert bt.linearize(w, (i + dx, j + dy, k + dz)) - t == off[d]


def test_presence_rule_against_lattice():
    """The zero-set micro-cell presence table used by the kernels equals the
    reference's in_i_tet(w_s, p - o) test (operators.hpp:88) at every point."""
    O = [[(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)], [(1, 1, 0), (1, 0, 1), (0, 1, 1), (1, 1, 1)],
         [(0, 1, 0), (0, 0, 1), (1, 0, 1), (0, 1, 1)], [(1, 0, 0), (0, 1, 0), (1, 1, 0), (1, 0, 1)],
         [(1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1)], [(0, 1, 0), (1, 1, 0), (1, 0, 1), (0, 1, 1)]]
    present = [0xffffff, 0xe8cc8e, 0x962b4d, 0x80080c, 0x4d962b, 0x48840a, 0x40209, 0x8, 0x337117, 0x204006,
               0x122105, 0x4, 0x11003, 0x2, 0x1, 0x0]
    for l in (2, 3, 4):
        n = 1 << l
        for (i, j, k) in bt.index_set(n + 1):
            z = (i + j + k == n) | ((i == 0) << 1) | ((j == 0) << 2) | ((k == 0) << 3)
            for s in range(6):
                w = bt.width(20 + s, l)
                for slot in range(4):
                    a = [(i, j, k)[e] - O[s][slot][e] for e in range(3)]
                    inside = min(a) >= 0 and sum(a) < w
                    assert inside == bool(present[z] >> (4 * s + slot) & 1)
