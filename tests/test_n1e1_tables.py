"""CPU: the committed N1E1 coupling header (csrc/bt_n1e1_tables.cuh) is what
scripts/gen_n1e1_tables.py generates, and its structure matches the oracle's
coupling counts (13 / 19 coupled edges, 31 distinct x rows in 16 streams,
33 + 33 corrections). The library re-checks it against build_static at
operator creation on the GPU."""
import os
import runpy
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "paper_2308_01792_b200", "csrc", "bt_n1e1_tables.cuh")


def generated(tmp_path):
    gen = runpy.run_path(os.path.join(ROOT, "scripts", "gen_n1e1_tables.py"))
    out = tmp_path / "t.cuh"
    gen["OUT"] = str(out)
    gen["main"].__globals__["OUT"] = str(out)
    gen["main"]()
    return out.read_text()


def test_header_is_generated(tmp_path):
    with open(HEADER) as f:
        assert f.read() == generated(tmp_path)


def test_coupling_structure():
    gen = runpy.run_path(os.path.join(ROOT, "scripts", "gen_n1e1_tables.py"))
    nb, inc = gen["coupling"]()
    assert [len(nb[g]) for g in range(1, 8)] == [19, 13, 19, 19, 13, 19, 13]
    assert [len(inc[g]) for g in range(1, 8)] == [6, 4, 6, 6, 4, 6, 4]
    rows = {(g, dy, dz) for G in nb for (g, dx, dy, dz) in nb[G]}
    streams = {(g, dz) for (g, dy, dz) in rows}
    assert len(rows) == 31 and len(streams) == 16
    c0, c1 = gen["corrections"](inc)
    assert len(c0) == 33 and len(c1) == 33
    assert all(dx in (-1, 0, 1) and dy in (-1, 0, 1) and dz in (-1, 0, 1)
               for G in nb for (g, dx, dy, dz) in nb[G])
