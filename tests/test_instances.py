"""Input generators (instances/): recipe properties and planted optima.

The planted mixed-cone instance of SURVEY §8(d) cfg 5 must be an exact KKT
point of Eq. 1-2: Eq. 9 at (x*, y*), evaluated by the
oracle, is zero up to rounding, and c^T x* is the optimal value.
"""
import numpy as np
import pytest

import oracle as O
from instances import gen_mixed_large, ZERO, NONNEG, SOC, RSOC, EXP, DUAL_EXP


@pytest.mark.parametrize("seed", [0, 3])
def test_cfg5_recipe_and_planted_kkt(seed):
    p = gen_mixed_large(0.0003, seed=seed)
    assert p.m == 6000 and p.n == 3000 and p.n1 == 1200
    lens = np.diff(p.row_ptr)
    assert lens.min() >= 20 and lens.max() <= 180
    for i in range(0, p.m, 97):                                 # distinct sorted columns per row
        c = p.col_idx[p.row_ptr[i]:p.row_ptr[i + 1]]
        assert np.all(np.diff(c) > 0)
    assert p.rdim.sum() == p.m and p.pdim.sum() == p.n - p.n1
    share = np.bincount(np.repeat(p.rk, p.rdim), minlength=6) / p.m
    assert np.allclose(share, [.30, .30, .25, .05, .075, .025], atol=0.002)
    pshare = np.bincount(np.repeat(p.pk, p.pdim), minlength=6) / (p.n - p.n1)
    assert np.allclose(pshare, [.01, .20, .40, .15, .20, .04], atol=0.003)
    assert np.all(p.rdim[(p.rk == EXP) | (p.rk == DUAL_EXP)] == 3)
    assert np.all(p.rdim[p.rk == SOC] >= 2) and np.all(p.rdim[p.rk == RSOC] >= 3)
    e = O.OracleSolver(p).kkt_point(p.x_star, p.y_star)
    assert e["err_p"] < 1e-13 and e["err_d"] < 1e-13 and e["err_gap"] < 1e-12
    assert abs(e["pobj"] - p.obj_star) <= 1e-12 * max(1.0, abs(p.obj_star))


def test_lasso_balanced_form_is_the_same_problem():
    """Reading P9: the balanced Lasso SOCP stores the RSOC leading pair as
    (S w, r / S), an automorphism of the rotated cone.  Solved by the oracle,
    both forms reach the same optimal value (the Lasso objective, FISTA-free:
    the two are checked against each other), the balanced solution mapped back
    by to_literal satisfies the literal form's Eq. 9, and the balanced form
    needs far fewer iterations on a tall instance (PDCS on the literal form
    stalls there, P8)."""
    import oracle as O
    from instances import gen_lasso
    bal = gen_lasso(120, 40, 0.3, seed=4)
    lit = gen_lasso(120, 40, 0.3, seed=4, balance=False)
    assert bal.lasso_S == max(1.0, (float(bal.lasso_b @ bal.lasso_b) / 2.0) ** 0.5) and lit.lasso_S == 1.0
    lb = bal.literal()                                  # derived literal form == generated literal form
    for f in ("row_ptr", "col_idx", "vals", "c", "h", "l", "u", "pk", "pdim", "rk", "rdim"):
        assert np.array_equal(getattr(lb, f), getattr(lit, f)), f
    assert lb.name == lit.name
    rb = O.OracleSolver(bal, tol=1e-8, max_iters=200000).solve()
    rl = O.OracleSolver(lit, tol=1e-8, max_iters=200000).solve()
    assert rb.status == 0 and rl.status == 0
    assert abs(rb.kkt.pobj - rl.kkt.pobj) <= 1e-6 * (1 + abs(rl.kkt.pobj))
    ob = O.OracleSolver(bal, tol=1e-8, max_iters=200000)
    ob.solve()
    x, y = ob.get_iterate(0, 1)
    k = O.OracleSolver(lit).kkt_point(bal.to_literal(x), y)
    assert max(k["err_p"], k["err_d"], k["err_gap"]) <= 1e-7, k
    tall_b = O.OracleSolver(gen_lasso(4000, 200, 0.05, seed=1), tol=1e-4, max_iters=20000).solve()
    tall_l = O.OracleSolver(gen_lasso(4000, 200, 0.05, seed=1, balance=False), tol=1e-4, max_iters=20000).solve()
    assert tall_b.status == 0 and tall_b.iters < tall_l.iters / 3, (tall_b.iters, tall_l.iters, tall_l.status)
