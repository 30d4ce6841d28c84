"""Host-side pieces of the Python mirror that need no GPU: parse_mesh /
CoarseMesh (coarse_mesh.hpp:37-47, 225-308) and the checked / AoS / SoA
linearisations (micro_index.hpp:150-175), through the C ABI."""
import numpy as np
import pytest

import paper_2308_01792_b200 as bt
from pyoracle import Oracle  # noqa: F401  (oracle on the path; only the C restatement below)


def test_parse_mesh_counts_and_round_trip():
    m = bt.parse_mesh(bt.cube_kuhn_text())
    assert m.n_vertices() == 8 and m.n_cells() == 6
    again = bt.parse_mesh(m.text)
    assert np.array_equal(again.cells, m.cells) and np.array_equal(again.vertex_coords, m.vertex_coords)
    p = bt.parse_mesh(bt.cubes_mesh_text(2, 0.1, 0))
    assert p.n_cells() == 48 and p.n_vertices() == 27


def test_parse_mesh_repairs_orientation():
    # negatively oriented reference tet: local vertices 2 and 3 swap (validate_and_finalize)
    m = bt.parse_mesh("vertices 4\n0 0 0\n1 0 0\n0 0 1\n0 1 0\ncells 1\n0 1 2 3\n")
    assert list(m.cells[0]) == [0, 1, 3, 2]


def test_parse_mesh_errors():
    with pytest.raises(bt.InvalidArgument):
        bt.parse_mesh("vertices 4\n0 0 0\n1 0 0\n0 1 0\ncells 1\n0 1 2 3\n")  # truncated vertex list
    with pytest.raises(bt.InvalidArgument):
        bt.parse_mesh("vertices 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\ncells 1\n0 1 2 9\n")  # bad vertex id


def test_linearize_checked_aos_soa():
    w = 5
    assert bt.linearize_checked(w, (1, 1, 1)) == bt.linearize(w, (1, 1, 1))
    with pytest.raises(bt.OutOfRange):
        bt.linearize_checked(w, (3, 1, 1))
    for p in [(0, 0, 0), (2, 1, 1), (0, 0, 4)]:
        t = bt.linearize(w, p)
        for m in (1, 3):
            for d in range(m):
                assert bt.linearize_aos(w, m, p, d) == m * t + d
                assert bt.linearize_soa(w, m, p, d) == d * bt.n_tet(w) + t
        with pytest.raises(bt.OutOfRange):
            bt.linearize_aos(w, 2, p, 2)
        with pytest.raises(bt.OutOfRange):
            bt.linearize_soa(w, 2, p, -1)


def test_blocked_mesh_partition_blocks_are_compact():
    """bt_blocked_mesh_text numbers cubes block-major, so bt_grid_set_partition's
    contiguous cell ranges are compact blocks of cubes: 4x4x4
    cubes in 2x2x2 blocks over 8 ranks give each rank one 2x2x2 block; the
    unblocked numbering gives 4x2x1 slabs."""
    text = bt.blocked_mesh_text(4, 4, 4, (2, 2, 2), h=0.25, perturb=0.0)
    m = bt.parse_mesh(text)
    assert m.n_cells() == 384
    for r in range(8):
        b, e = bt.partition_range(384, r, 8)
        xyz = m.vertex_coords[m.cells[b:e].ravel()]
        ext = xyz.max(axis=0) - xyz.min(axis=0)
        assert np.allclose(ext, [0.5, 0.5, 0.5])
    plain = bt.parse_mesh(bt.cubes_mesh_text(4, 0.0, 0))
    b, e = bt.partition_range(384, 0, 8)
    ext = np.ptp(plain.vertex_coords[plain.cells[b:e].ravel()], axis=0)
    assert np.allclose(sorted(ext), [0.25, 0.5, 1.0])
    # the same geometry and perturbation as the unblocked generator, cells renumbered
    a = bt.parse_mesh(bt.blocked_mesh_text(4, 4, 4, (4, 4, 4), h=0.25, perturb=0.1, seed=0))
    c = bt.parse_mesh(bt.cubes_mesh_text(4, 0.1, 0))
    assert np.array_equal(a.vertex_coords, c.vertex_coords) and np.array_equal(a.cells, c.cells)
