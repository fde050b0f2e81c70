"""L2 column panels of the SpMV sweeps (panels.cuh) on the GPU.

The setup autotune keeps panels only when the gathered vector exceeds L2
(configs[4] at its stated size); PDCS_PANELS=P forces P panels so that the
panelled sweeps (K x^ with the fused dual trial, K^T y+ with the fused Halpern
step, the check's product stores) are checked against the oracle at test
sizes: one Eq. 5 step from random points at 1e-12 and checkpoint shadowing at
the north_star tolerance, as tests/test_gpu_parity.py does for the CSR and
tiled paths.
"""
import numpy as np
import pytest

import oracle as O
from instances import gen_fisher, gen_lasso, gen_mixed

pytestmark = pytest.mark.gpu
TOL = 1e-9
STOL = 1e-6


@pytest.fixture(scope="module")
def P():
    from paper_2505_00311_b200 import build
    build.build()
    import paper_2505_00311_b200 as P
    return P


def rel(a, b):
    return np.max(np.abs(a - b)) / (1.0 + np.max(np.abs(b)))


CASES = {
    "mixed": lambda: gen_mixed(600, 80, 300, seed=9, soc_dims=(3, 100), scale_spread=1.5),
    "lasso": lambda: gen_lasso(400, 60, 0.3, seed=2),
    "fisher": lambda: gen_fisher(1200, 40, seed=5),
}


@pytest.mark.parametrize("panels", ["1", "3", "7"])
@pytest.mark.parametrize("name", sorted(CASES))
def test_panelled_sweeps_match_oracle(P, name, panels, monkeypatch):
    monkeypatch.setenv("PDCS_TILED", "0")
    monkeypatch.setenv("PDCS_PANELS", panels)
    prog = CASES[name]()
    g = P.PdcsSolver(prog)
    sc = g.scalars()
    assert sc["panels_K"] == int(panels) and sc["panels_KT"] == int(panels)
    o = O.OracleSolver(prog)
    ro, qo = o.get_scaling()
    rng = np.random.default_rng(3)
    for _ in range(2):
        x, y = rng.standard_normal(prog.n) * 2, rng.standard_normal(prog.m) * 2
        g.set_iterate(x, y)
        o.set_iterate(x * qo, y * ro)
        g.iterate(1)
        o.iterate(1)
        xg, yg = g.get_iterate(P.PDHG_OUT)
        xo, yo = o.get_iterate(1)
        assert max(rel(xg, xo), rel(yg, yo)) <= 1e-12
        # the accepted step's K^T y+ (panelled, fused Halpern) and Eq. 9 at this point
        kg, ko = g.kkt(P.CURRENT), o.kkt(0)
        for k in ("err_p", "err_d", "err_gap"):
            assert abs(kg[k] - ko[k]) <= 1e-12 * (1 + abs(ko[k]))
    g = P.PdcsSolver(prog)
    o = O.OracleSolver(prog)
    worst = 0.0
    for s in range(0, 160, 10):
        g.set_state(o.get_state())
        g.iterate(10)
        o.iterate(10)
        sg, so = g.get_state(), o.get_state()
        assert np.array_equal(sg["sc"][9:], so["sc"][9:]), (s, sg["sc"], so["sc"])
        for i in (0, 2, 4):
            assert abs(sg["sc"][i] - so["sc"][i]) <= STOL * abs(so["sc"][i])
        worst = max(worst, rel(sg["x"], so["x"]), rel(sg["y"], so["y"]))
    assert worst <= TOL, worst


def test_panels_not_kept_when_the_vector_fits_in_l2(P):
    """Autotune gating: below 64 MB of gathered vector no panels are built."""
    g = P.PdcsSolver(CASES["mixed"]())
    sc = g.scalars()
    assert sc["panels_K"] == 0 and sc["panels_KT"] == 0
