"""CPU: the compiled reference's interpolate / l2_error / fmg through the
oracle shim (oracle/ref_driver.cpp), which the GPU FMG tests compare against,
checked against the reference tests' own statements (test_solvers.cpp 'l2 error
measures interpolation quality', 'full multigrid runs the documented cycle
budget')."""
import math

import numpy as np
import pytest

from pyoracle import Reference, cube_kuhn_text

U = (1, 0.0, 1.0, math.pi, 0.0)              # sin(pi x) sin(pi y) sin(pi z)
F = (1, 0.0, 3.0 * math.pi ** 2, math.pi, 0.0)
LIN = (2, 0.5, -1.0, 2.0, 0.25)
GS = [1, 0.8, 2, 0.25, 1.1, 1, 1]


@pytest.fixture(scope="module")
def ref():
    return Reference(cube_kuhn_text(), 2, 4)


def test_l2_error_known_answers(ref):
    x = ref.interpolate(2, LIN)
    assert ref.l2_error(2, x, LIN) <= 1e-13                      # linear fields are interpolated exactly
    one = np.ones(ref.size(0, 2))
    assert ref.l2_error(2, one, (0, 0.0, 0, 0, 0)) == pytest.approx(1.0, abs=1e-12)  # unit cube volume
    e = [ref.l2_error(l, ref.interpolate(l, U), U) for l in (2, 3, 4)]
    assert e[0] / e[1] == pytest.approx(4.0, abs=1.0) and e[1] / e[2] == pytest.approx(4.0, abs=1.0)


def test_fmg_cycle_budget_and_orders(ref):
    ref.make_hierarchy(form=0, kernel=1)
    rhs = [ref.zero_dirichlet(l, ref.apply_elementwise(l, ref.interpolate(l, F), form=1)) for l in (2, 3, 4)]
    rows, x = ref.fmg(4, GS, rhs, 2, 5, fp=U)
    assert len(rows) == 1 + 5 * 2
    assert [int(r[0]) for r in rows] == [2] + [3] * 5 + [4] * 5
    err = {int(r[0]): r[3] for r in rows}
    assert 2.8 <= err[2] / err[3] <= 4.7 and 3.4 <= err[3] / err[4] <= 4.6
    rows2, x2 = ref.fmg(4, GS, rhs, 2, 5, fp=U)                     # deterministic
    assert np.array_equal(rows, rows2) and np.array_equal(x, x2)
