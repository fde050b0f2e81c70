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
sqrt(d) eps ~ 1e-13).  The one step is also checked per coordinate against
each coordinate's own rounding scale (block-maximised over cone blocks).  A
few accepted PDCS steps after it: north_star's 1e-9 per iterate, with equal
trial and restart counts.
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


def block_max(a, n_head, kinds, dims):
    """a with every cone block (SOC/RSOC/exp) replaced by its block maximum: a
    projection mixes the coordinates of its block, so their rounding scale is
    the block's.  The first n_head coordinates (box / elementwise) are kept."""
    out = a.copy()
    off = n_head + np.concatenate([[0], np.cumsum(dims)[:-1]]).astype(np.int64)
    big = np.asarray(kinds) >= 2
    if big.any():
        seg = np.maximum.reduceat(a[n_head:], off - n_head) if len(dims) else np.zeros(0)
        for o, d, v in zip(off[big], np.asarray(dims)[big], seg[big]):
            out[o:o + d] = v
    return out


def per_coordinate_scales(prog, o, state, tau, sigma, xh):
    """Rounding scale of every coordinate of one Eq. 5 step in the scaled space:
    x^_j: |x_j| + tau(|c~_j| + (|K~|^T |y|)_j); y^_i: |y_i| + sigma(|h~_i| +
    (|K~| (2|x^| + |x|))_i), block-maximised over cone blocks."""
    import scipy.sparse as sp
    r, q = o.get_scaling()
    A = sp.csr_matrix((np.abs(prog.vals), prog.col_idx, prog.row_ptr), shape=(prog.m, prog.n))
    A = sp.diags(1.0 / r) @ A @ sp.diags(1.0 / q)
    x, y = state["x"], state["y"]
    ax = np.abs(x) + tau * (np.abs(prog.c / q) + A.T @ np.abs(y))
    ay = np.abs(y) + sigma * (np.abs(prog.h / r) + A @ (2 * np.abs(xh) + np.abs(x)))
    return block_max(ax, prog.n1, prog.pk, prog.pdim), block_max(ay, 0, prog.rk, prog.rdim)


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
    st0, sc0 = o.get_state(), o.scalars()
    g.iterate(1)
    o.iterate(1)
    xg, yg = g.get_iterate(P.PDHG_OUT)
    xo, yo = o.get_iterate(1)
    one = parity(xg, yg, xo, yo)
    assert one <= 1e-10, (config, one)
    # per coordinate, each against its own rounding scale (the vector-max
    # normalisation above would hide a wrong coordinate far below the maximum
    # on instances whose values span many decades, as mixed cfg 5 does)
    tau, sigma = sc0["eta"] / sc0["omega"], sc0["eta"] * sc0["omega"]
    ax, ay = per_coordinate_scales(prog, o, st0, tau, sigma, xo)
    ex = np.abs(xg - xo) / (ax + 1e-300)
    ey = np.abs(yg - yo) / (ay + 1e-300)
    assert ex.max() <= 1e-10 and ey.max() <= 1e-10, (config, ex.max(), int(ex.argmax()), ey.max(),
                                                       int(ey.argmax()))
    rg3 = g.iterate(3)
    o.iterate(3)
    so = o.scalars()
    assert rg3["trials"] == so["trials"] and rg3["restarts"] == so["restarts"], (rg3, so)
    more = parity(*g.get_iterate(P.CURRENT), *o.get_iterate(0))
    assert more <= 1e-9, (config, more)
    g.close()
