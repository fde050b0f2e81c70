"""Box-column locality order (plan_colperm) on the GPU (-m gpu).

When the long rows of G gather strided box columns (Fisher's supply rows over a
buyer-major X), libpdcs stores the box columns in the order of their longest
row.  The order is internal: every x-side array that crosses the C ABI
(get/set_iterate, get/set_state, get_scaling) is in the caller's order, so the
oracle comparisons below are the same as for an unpermuted context.
"""
import numpy as np
import pytest

import oracle as O
from instances import gen_fisher

pytestmark = pytest.mark.gpu
TOL = 1e-9


@pytest.fixture(scope="module")
def P():
    from paper_2505_00311_b200 import build
    build.build()
    import paper_2505_00311_b200 as P
    return P


def rel(a, b):
    return np.max(np.abs(a - b)) / (1.0 + np.max(np.abs(b)))


def test_colperm_is_chosen_and_invisible_at_the_boundary(P, monkeypatch):
    prog = gen_fisher(1200, 40, seed=3)            # 40 supply rows of 1200 strided entries
    g = P.PdcsSolver(prog)
    assert g.scalars()["colperm"] == 1.0
    monkeypatch.setenv("PDCS_COLPERM", "0")
    g0 = P.PdcsSolver(prog)
    assert g0.scalars()["colperm"] == 0.0
    o = O.OracleSolver(prog)
    ro, qo = o.get_scaling()
    for h in (g, g0):                              # scaling in the caller's order
        rg, qg = h.get_scaling()
        np.testing.assert_allclose(qg, qo, rtol=1e-13)
        np.testing.assert_allclose(rg, ro, rtol=1e-13)
    # one Eq. 5 step from random original-space points (set_iterate / get_iterate)
    rng = np.random.default_rng(1)
    for _ in range(3):
        x, y = rng.standard_normal(prog.n), rng.standard_normal(prog.m)
        g.set_iterate(x, y)
        o.set_iterate(x * qo, y * ro)
        g.iterate(1)
        o.iterate(1)
        xg, yg = g.get_iterate(P.PDHG_OUT)
        xo, yo = o.get_iterate(1)
        assert max(rel(xg, xo), rel(yg, yo)) <= 1e-12
        xg1, _ = g.get_iterate(P.PDHG_OUT, P.ORIGINAL)
        assert rel(xg1, xo / qo) <= 1e-12
    # checkpoint shadowing through get_state / set_state (x, x0, xsum permuted inside)
    o = O.OracleSolver(prog)
    g = P.PdcsSolver(prog)
    worst = 0.0
    for _ in range(12):
        st = o.get_state()
        g.set_state(st)
        g.iterate(10)
        o.iterate(10)
        sg, so = g.get_state(), o.get_state()
        assert np.array_equal(sg["sc"][9:], so["sc"][9:])
        for k in ("x", "x0"):
            worst = max(worst, rel(sg[k], so[k]))
        if so["sc"][4] > 0:
            worst = max(worst, rel(sg["xsum"] / sg["sc"][4], so["xsum"] / so["sc"][4]))
    assert worst <= TOL, worst


def test_colperm_free_running_matches_identity_order(P, monkeypatch):
    """The same trajectory with and without the locality order over the first
    120 iterations (only summation orders differ), and the same solve."""
    prog = gen_fisher(1200, 40, seed=4)
    a = P.PdcsSolver(prog, tol=1e-4, max_iters=400000)
    monkeypatch.setenv("PDCS_COLPERM", "0")
    b = P.PdcsSolver(prog, tol=1e-4, max_iters=400000)
    a.iterate(120)
    b.iterate(120)
    xa, ya = a.get_iterate(P.CURRENT)
    xb, yb = b.get_iterate(P.CURRENT)
    assert max(rel(xa, xb), rel(ya, yb)) <= TOL
    ra, rb = a.solve(), b.solve()
    assert ra["status"] == rb["status"] == "OPTIMAL"
    assert abs(ra["pobj"] - rb["pobj"]) <= 1e-3 * (1 + abs(rb["pobj"]))
