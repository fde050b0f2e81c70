"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (graph path, setup autotune: the tiled sweeps on Lasso, CSR elsewhere).

At these sizes the CPU oracle still runs a whole PDHG step in about a second
(setup with its own Ruiz / Pock-Chambolle scaling: 10-25 s), so the comparison
is over every coordinate, not a sample.  No value of the CUDA path enters the
oracle: both get the same seeded random point in the ORIGINAL space (the
oracle scales it with its own r, q).

Tolerances.  One Eq. 5 step from a random point: 1e-10 relative.  The longest
sums are the 1e4-term K^T rows of Lasso and the 1e6-term norms of its RSOC
multiplier equation (Thm 1); summed in a different order, their worst-case
rounding difference is d * eps = 1e6 * 1.1e-16 = 1.1e-10 relative (typical
sqrt(d) eps ~ 1e-13).  A few accepted PDCS steps after it: north_star's 1e-9
per iterate, with equal trial and restart counts.
"""
import numpy as np
import pytest

import oracle as O
from instances import CONFIGS

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    from paper_2505_00311_b200 import build
    build.build()
    import paper_2505_00311_b200 as P
    return P


def rel(a, b):
    return np.max(np.abs(a - b)) / (1.0 + np.max(np.abs(b))) if a.size else 0.0


def parity(xg, yg, xo, yo):
    return max(rel(xg, xo), rel(yg, yo))


@pytest.mark.parametrize("config", ["lasso", "fisher", "mpo", "mixed"])
def test_full_size_step_parity(P, config):
    prog = CONFIGS[config](0)
    g = P.PdcsSolver(prog)
    o = O.OracleSolver(prog)
    ro, qo = o.get_scaling()
    rg, qg = g.get_scaling()
    assert rel(rg, ro) <= 1e-12 and rel(qg, qo) <= 1e-12
    rng = np.random.default_rng(7)
    x = rng.standard_normal(prog.n)
    y = rng.standard_normal(prog.m)
    g.set_iterate(x, y)                 # original space
    o.set_iterate(x * qo, y * ro)       # the oracle's own scaling
    g.iterate(1)
    o.iterate(1)
    one = parity(*g.get_iterate(P.PDHG_OUT), *o.get_iterate(1))
    assert one <= 1e-10, (config, one)
    rg3 = g.iterate(3)
    o.iterate(3)
    so = o.scalars()
    assert rg3["trials"] == so["trials"] and rg3["restarts"] == so["restarts"], (rg3, so)
    more = parity(*g.get_iterate(P.CURRENT), *o.get_iterate(0))
    assert more <= 1e-9, (config, more)
    g.close()
