"""Pins for the oracle's Alg. 1 rules that have no closed form (-m "not gpu").

Each rule is pinned to its statement (PAPER.md / SPEC.md passage, or the
DESIGN.md §3 reading) by hand-evaluated values, or by checking the oracle's
observable state step by step against that statement.  Every pin is chosen
so that a plausible slip fails it (named in each docstring).
"""
import math

import numpy as np
import pytest

import oracle as O
from instances import ConicProgram, csr_from_coo, gen_mixed, ZERO, NONNEG, RSOC, SOC

INF = np.inf


def tiny(G_, c, h, l, u, rk, rdim, pk=(), pdim=()):
    A = np.asarray(G_, float)
    r, cc = np.nonzero(A)
    m, n = A.shape
    ptr, col, val = csr_from_coo(m, n, r, cc, A[r, cc])
    return ConicProgram(m=m, n=n, n1=len(l), row_ptr=ptr, col_idx=col, vals=val,
                        c=np.asarray(c, float), h=np.asarray(h, float), l=np.asarray(l, float),
                        u=np.asarray(u, float), pk=np.array(pk, np.int32),
                        pdim=np.array(pdim, np.int64), rk=np.array(rk, np.int32),
                        rdim=np.array(rdim, np.int64))


def box_lp(seed, m=12, n=9):
    """Random LP: box columns of all four kinds, NonNeg rows (P is a clip on both sides)."""
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, n)) * (rng.uniform(size=(m, n)) < 0.6)
    A[np.arange(m), np.arange(m) % n] += 1.0
    l = np.where(np.arange(n) % 4 < 2, 0.0, -INF)
    u = np.where(np.isin(np.arange(n) % 4, [1, 2]), 2.0, INF)
    return tiny(A, rng.standard_normal(n), rng.standard_normal(m), l, u, [NONNEG], [m])


# ------------------------------------------------------------------ reflection parameter (A9)
def _beta_seq(res, W, beta=1.0):
    rs = 0.0
    out = []
    for k, r in enumerate(res):
        beta, rs = O.reflection_beta(k, W, r, rs, beta)
        out.append(beta)
    return out


def test_reflection_beta_window_rule_hand_sequences():
    """SPEC.md:366-368 examples and reading A9 (non-overlapping windows of W).

    Fails for: halving on a decrease, halving before the window's end, a
    sliding window, comparing with the previous window's start, halving twice.
    """
    # empty history -> beta_max
    assert O.reflection_beta(0, 4, 1.0, 0.0, 1.0)[0] == 1.0
    # monotonically decreasing window keeps beta_max
    assert _beta_seq([8, 7, 6, 5, 4, 3, 2, 1], 4) == [1.0] * 8
    # residual rose over the window -> halved at the window's last iteration only
    assert _beta_seq([1.0, 0.5, 0.5, 1.5], 4) == [1.0, 1.0, 1.0, 0.5]
    # a rise inside the window that ends below its start does not halve
    assert _beta_seq([1.0, 5.0, 5.0, 0.9], 4) == [1.0] * 4
    # sliding-window counterexample: r(5) > r(2) but each non-overlapping window decreases
    assert _beta_seq([1, 0.9, 0.8, 0.7, 0.6, 0.95, 0.5, 0.4], 4) == [1.0] * 8
    # the second window compares with its own start (0.1), not the first window's (1.0)
    assert _beta_seq([1.0, 0.9, 0.8, 0.7, 0.1, 0.1, 0.1, 0.2], 4)[-1] == 0.5
    # two rising windows halve twice; equality does not halve
    assert _beta_seq([1, 1, 1, 2, 1, 1, 1, 1.5, 3, 3, 3, 3], 4) == [1] * 3 + [0.5] * 4 + [0.25] * 5


def _step_states(S, nsteps):
    """Per accepted step: (scalars before, state before, scalars after, state after, PDHG out)."""
    rows = []
    for _ in range(nsteps):
        sb, gb = S.scalars(), S.get_state()
        S.iterate(1)
        sa, ga = S.scalars(), S.get_state()
        rows.append((sb, gb, sa, ga, S.get_iterate(1)))
    return rows


def test_reflection_beta_in_the_solver():
    """Alg. 1 line 5 as wired in the oracle: the residual is ||z^ - z||_omega
    (SPEC.md:434 with the omega-norm of SPEC.md:437) of each accepted step,
    windows of refl_window, reset to beta_max at a restart."""
    p = gen_mixed(80, 10, 30, seed=5)
    W = 5
    S = O.OracleSolver(p, refl_window=W, check_interval=15)
    rstart = None
    halvings = 0
    for sb, gb, sa, ga, (xh, yh) in _step_states(S, 300):
        k = int(sb["k"])
        om = sb["omega"]
        dx, dy = xh - gb["x"], yh - gb["y"]
        num = om * (dx @ dx) + (dy @ dy) / om
        assert abs(sa["last_num"] - num) <= 1e-12 * num
        res = math.sqrt(sa["last_num"])
        if k % W == 0:
            rstart = res
        expect = sb["beta"] * (0.5 if (k % W == W - 1 and res > rstart) else 1.0)
        if sa["restarts"] > sb["restarts"]:
            assert sa["beta"] == 1.0 and sa["k"] == 0
        else:
            assert sa["beta"] == expect
        halvings += expect != sb["beta"]
    assert halvings >= 2        # the rule fired on this trajectory


# ------------------------------------------------------------------ step-weighted average (A8)
def test_average_weights_are_the_steps_that_produced_the_points():
    """Alg. 1 line 7: zbar = sum eta^i z^i / sum eta^i, eta^i the step
    with which z^i was produced (reading A8).

    Fails for: weighting by the grown step min(1.05 eta, eta_bar), by the
    pre-rejection step, summing z^ instead of z, or a uniform average.
    """
    p = gen_mixed(80, 10, 30, seed=6)
    S = O.OracleSolver(p, eta0=5.0)          # large start: the first steps reject
    seen_reject = seen_grow = 0
    for sb, gb, sa, ga, _ in _step_states(S, 120):
        if sa["restarts"] > sb["restarts"]:
            assert sa["W"] == 0.0 and np.all(ga["xsum"] == 0)
            continue
        rejects = int(sa["trials"] - sb["trials"]) - 1
        eta_used = sb["eta"] * 0.5 ** rejects
        seen_reject += rejects > 0
        seen_grow += sa["eta"] != eta_used
        assert sa["W"] == sb["W"] + eta_used
        assert np.array_equal(ga["xsum"], gb["xsum"] + eta_used * ga["x"])
        assert np.array_equal(ga["ysum"], gb["ysum"] + eta_used * ga["y"])
    assert seen_reject and seen_grow


def test_average_candidate_is_the_projected_weighted_mean():
    """The average candidate is P(sum eta z / sum eta) (Alg. 1 lines 7-8, reading A10);
    on a box LP with NonNeg rows P is a clip.  Fails for: an unprojected average,
    an unnormalised sum, the candidate taken from the wrong side of the tie."""
    took_avg = took_cur = 0
    for seed in range(8):
        p = box_lp(seed)
        S = O.OracleSolver(p, check_interval=10, restart_art=10.0, restart_suff=0.0,
                           restart_nec=0.0)
        S.iterate(10)                          # 10 accepted steps, then the check
        g, sc = S.get_state(), S.scalars()
        _, q_ = S.get_scaling()
        x_mean = np.clip(g["xsum"] / sc["W"], p.l * q_, p.u * q_)
        y_mean = np.maximum(g["ysum"] / sc["W"], 0.0)
        xc, yc = S.get_iterate(4)
        if list(S.trace())[-2] == 11:
            took_avg += 1
            assert np.array_equal(xc, x_mean) and np.array_equal(yc, y_mean)
        else:
            took_cur += 1
            xh, yh = S.get_iterate(1)
            assert np.array_equal(xc, xh) and np.array_equal(yc, yh)
    assert took_avg and took_cur


# ------------------------------------------------------------------ restart candidate (A14)
def test_candidate_tie_goes_to_the_average():
    """the smaller aggregate Eq. 9 error wins, a tie favours the average.
    Fails for: a strict '<' (tie -> current), the reversed comparison."""
    assert O.candidate_is_average(1.0, 1.0)
    assert O.candidate_is_average(1.0, 0.5)
    assert not O.candidate_is_average(0.5, 1.0)
    assert O.candidate_is_average(0.0, 0.0)


def test_candidate_choice_in_the_solver_follows_the_errors():
    """At every check the trace's candidate code (10 current, 11 average) is the
    argmin of max(err_p, err_d, err_gap) of the two candidates (reading A14)."""
    p = gen_mixed(80, 10, 30, seed=7)
    S = O.OracleSolver(p, check_interval=10)
    both = set()
    for _ in range(40):
        S.iterate(10)
        sc = S.scalars()
        ec = max(sc["cur_err_p"], sc["cur_err_d"], sc["cur_err_gap"])
        ea = max(sc["avg_err_p"], sc["avg_err_d"], sc["avg_err_gap"])
        code = [t for t in S.trace() if t in (10, 11)][-1]
        assert code == (11 if ea <= ec else 10)
        both.add(code)
    assert both == {10, 11}


# ------------------------------------------------------------------ Pock-Chambolle and RSOC pair
def test_pock_chambolle_pass_hand_values():
    """one Pock-Chambolle pass with exponent 1 divides rows and
    columns by the square root of their 1-norms of |G|.
    Fails for: inf-norms, dropped sqrt, squared entries, PC before Ruiz."""
    p = tiny([[1.0, 3.0], [0.0, -4.0]], [0, 0], [0, 0], [-INF] * 2, [INF] * 2, [ZERO], [2])
    r, q = O.ruiz(p, 0, 1)
    np.testing.assert_allclose(r, [2.0, 2.0], rtol=1e-15)                 # sqrt(1+3), sqrt(4)
    np.testing.assert_allclose(q, [1.0, math.sqrt(7.0)], rtol=1e-15)      # sqrt(1), sqrt(3+4)
    # one Ruiz round, then PC on the Ruiz-scaled matrix (hand-evaluated):
    # Ruiz: r = (sqrt 3, 2), q = (1, 2); |K| = [[1/sqrt3, sqrt3/2], [0, 1]]
    r, q = O.ruiz(p, 1, 1)
    s3 = math.sqrt(3.0)
    np.testing.assert_allclose(r, [s3 * math.sqrt(1 / s3 + s3 / 2), 2.0], rtol=1e-15)
    np.testing.assert_allclose(q, [math.sqrt(1 / s3), 2.0 * math.sqrt(s3 / 2 + 1.0)], rtol=1e-15)


def test_rsoc_leading_pair_geometric_mean():
    """SPEC.md:306 (reading A21): the two leading scalings of every RSOC block are
    replaced by their geometric mean, after Ruiz and PC, on both sides.
    Fails for: arithmetic mean, max, leaving them unequal, averaging before PC."""
    G = np.diag([1.0, 9.0, 4.0])
    # primal RSOC block over columns 0..2; Ruiz round: r = q = (1, 3, 2); PC then sees I
    p = tiny(G, [0, 0, 0], [0, 0, 0], [], [], [ZERO], [3], [RSOC], [3])
    for pc in (0, 1):
        r, q = O.ruiz(p, 1, pc)
        np.testing.assert_allclose(q, [math.sqrt(3.0), math.sqrt(3.0), 2.0], rtol=1e-15)
        np.testing.assert_allclose(r, [1.0, 3.0, 2.0], rtol=1e-15)
    # row-side RSOC block
    p = tiny(G, [0, 0, 0], [0, 0, 0], [], [], [RSOC], [3], [SOC], [3])
    r, q = O.ruiz(p, 1, 1)
    np.testing.assert_allclose(r, [math.sqrt(3.0), math.sqrt(3.0), 2.0], rtol=1e-15)
    np.testing.assert_allclose(q, [1.0, 3.0, 2.0], rtol=1e-15)
    # order: with a matrix where PC changes the scalings, the mean is taken last
    p = tiny([[1.0, 2.0, 0.0], [0.0, 4.0, 0.0], [0.0, 0.0, 1.0]], [0] * 3, [0] * 3, [], [],
             [ZERO], [3], [RSOC], [3])
    r, q = O.ruiz(p, 0, 1)
    # PC alone: column 1-norms (1, 6, 1) -> (1, sqrt6, 1); mean of the pair sqrt(sqrt 6)
    np.testing.assert_allclose(q, [6 ** 0.25, 6 ** 0.25, 1.0], rtol=1e-15)
    np.testing.assert_allclose(r, [math.sqrt(3.0), 2.0, 1.0], rtol=1e-15)


# ------------------------------------------------------------------ Eq. 9 normalisers
def _kkt_problem():
    # columns: 0 box [0.25, inf) (Lambda = R+), 1 box (-inf, 2] (Lambda = R-), 2 NonNeg cone
    return tiny([[1.0, 2.0, 0.0], [0.0, 1.0, 3.0]], [1.0, -1.0, 2.0], [1.0, 1.0],
                [0.25, -INF], [INF, 2.0], [ZERO], [2], [NONNEG], [1])


def test_eq9_err_d_normaliser_hand_values():
    """err_d = max(|lam1 - P_Lambda lam1|inf, |lam2 - P_Kp* lam2|inf)
    / (1 + max(|c|inf, |G^T y|inf)), lam = c - G^T y.
    Fails for: a denominator without |G^T y| or without |c|, a missing 1+,
    a wrong Lambda orientation, the cone part dropped."""
    p = _kkt_problem()
    S = O.OracleSolver(p, ruiz_iters=0, pock_chambolle=0)
    x = np.array([0.5, 1.0, 0.2])
    # y = (2, -1): G^T y = (2, 3, -3), lam = (-1, -4, 5): col 0 off R+ by 1; |G^T y| = 3 > |c| = 2
    assert S.kkt_point(x, np.array([2.0, -1.0]))["err_d"] == 1.0 / 4.0
    # y = (1.05, -0.5): G^T y = (1.05, 1.6, -1.5), lam = (-0.05, -2.6, 3.5); |c| = 2 > 1.6
    assert abs(S.kkt_point(x, np.array([1.05, -0.5]))["err_d"] - 0.05 / 3.0) <= 1e-16
    # y = (0, 1): G^T y = (0, 1, 3), lam = (1, -2, -1): cone part off R+ by 1
    assert S.kkt_point(x, np.array([0.0, 1.0]))["err_d"] == 1.0 / 4.0
    # y = (-1, 0): lam = (2, 1, 2): column 1 (Lambda = R-) off by 1; |G^T y| = 2 = |c|
    assert S.kkt_point(x, np.array([-1.0, 0.0]))["err_d"] == 1.0 / 3.0


def test_eq9_err_gap_and_err_p_hand_values():
    """err_gap = |c.x - (y.h + l.lam1+ - u.lam1-)| /
    (1 + max(|c.x|, |dual obj|)), lam1 taken as P_Lambda(lam1) (reading A13);
    err_p = |(Gx-h) - P(Gx-h)|inf / (1 + max(|h|, |Gx|, |P(Gx-h)|)).
    Fails for: dropping the bound terms, a sign slip in u.lam1-, a sum instead of
    max in the denominator, a missing 1+."""
    p = _kkt_problem()
    S = O.OracleSolver(p, ruiz_iters=0, pock_chambolle=0)
    x = np.array([0.5, 1.0, 0.2])
    # y = (0, 1): lam1 = (1, -2): dual obj = 1 + 0.25*1 - 2*2 = -2.75; c.x = -0.1
    k = S.kkt_point(x, np.array([0.0, 1.0]))
    assert k["pobj"] == 0.5 - 1.0 + 0.4 and k["dobj"] == -2.75
    assert abs(k["err_gap"] - 2.65 / 3.75) <= 1e-15
    # y = (2, -1): lam1 = (-1, -4) -> P_Lambda = (0, -4): dual obj = 1 - 8 = -7
    k = S.kkt_point(x, np.array([2.0, -1.0]))
    assert k["dobj"] == -7.0 and abs(k["err_gap"] - 6.9 / 8.0) <= 1e-15
    # err_p: Gx = (2.5, 1.6), Zero rows: residual (1.5, 0.6), P = 0
    assert abs(k["err_p"] - 1.5 / 3.5) <= 1e-16


# ------------------------------------------------------------------ eta0 / omega0 / power iteration
def test_initial_step_and_primal_weight_hand_values():
    """Reading A5 eta0 = 1/||K~||inf (max row 1-norm) and A6 omega0 = ||c~||inf/||h~||inf
    clipped to [1e-4, 1e4], 1 when either is 0.
    Fails for: a column norm, a 2-norm, the inverse ratio, no clip."""
    G = [[1.0, -2.0], [3.0, 0.5]]
    for c, h, om in [([2.0, -6.0], [3.0, 1.0], 2.0), ([2e5, 1.0], [1.0, -1.0], 1e4),
                     ([1e-5, 0.0], [1.0, 1.0], 1e-4), ([0.0, 0.0], [1.0, 1.0], 1.0),
                     ([1.0, 1.0], [0.0, 0.0], 1.0), ([1.0, 0.5], [-4.0, 2.0], 0.25)]:
        p = tiny(G, c, h, [-INF] * 2, [INF] * 2, [ZERO], [2])
        sc = O.OracleSolver(p, ruiz_iters=0, pock_chambolle=0).scalars()
        assert sc["eta0"] == 1.0 / 3.5 and sc["eta"] == 1.0 / 3.5
        assert sc["omega"] == om
    # with Ruiz + PC the same definitions hold in the scaled space
    p = gen_mixed(60, 8, 20, seed=2)
    S = O.OracleSolver(p)
    r, q = S.get_scaling()
    K = p.dense() / r[:, None] / q[None, :]
    sc = S.scalars()
    assert abs(sc["eta0"] - 1.0 / np.abs(K).sum(axis=1).max()) <= 1e-14 * sc["eta0"]
    cn, hn = np.abs(p.c / q).max(), np.abs(p.h / r).max()
    assert abs(sc["omega"] - min(max(cn / hn, 1e-4), 1e4)) <= 1e-14 * sc["omega"]


@pytest.mark.parametrize("G,norm", [([[3.0, 0.0], [0.0, 1.0]], 3.0),
                                    ([[1.0, 2.0], [0.0, 2.0]], math.sqrt((9 + math.sqrt(65)) / 2)),
                                    ([[1.0, 1.0, 1.0]], math.sqrt(3.0))])
def test_vanilla_step_uses_the_spectral_norm(G, norm):
    """Vanilla PDHG: tau = sigma = 0.9/||G||_2 by power iteration.
    The test matrices separate ||G||_2 from ||G||_F, ||G||inf and ||G||_2^2."""
    m, n = np.asarray(G).shape
    p = tiny(G, [1.0] * n, [0.0] * m, [-INF] * n, [INF] * n, [ZERO], [m])
    sc = O.OracleSolver(p, vanilla_pdhg=1).scalars()
    assert abs(0.9 / sc["eta"] - norm) <= 2e-4 * norm
    assert sc["omega"] == 1.0


# ------------------------------------------------------------------ restart bookkeeping (A11, A12)
def test_restart_moves_anchor_and_updates_primal_weight():
    """Alg. 1 line 11: at a restart z^{t+1,0} = z_c and
    omega <- PrimalWeightUpdate(z^{t+1,0}, z^{t,0}, omega) with the anchor gaps
    ||x_new - x_old||, ||y_new - y_old||; the epoch restarts at
    k = 0 with beta = beta_max and an empty average.  Also: the restart decision
    at each check is restart_rule(e, e_anchor, e_prev, k, total) with e the
    chosen candidate's error (reading A11).
    Fails for: swapped gaps (omega moves the wrong way), gaps to the current
    iterate instead of the old anchor, omega not updated, the anchor left in place."""
    p = gen_mixed(80, 10, 30, seed=8)
    S = O.OracleSolver(p, check_interval=10)
    n_restart = n_check = 0
    for _ in range(400):
        sb, gb = S.scalars(), S.get_state()
        S.iterate(1)
        sa, ga = S.scalars(), S.get_state()
        if (int(sb["k"]) + 1) % 10 != 0:
            continue
        # a check ran after this step
        n_check += 1
        ec = max(sa["cur_err_p"], sa["cur_err_d"], sa["cur_err_gap"])
        ea = max(sa["avg_err_p"], sa["avg_err_d"], sa["avg_err_gap"])
        e = min(ec, ea)
        did = sa["restarts"] > sb["restarts"]
        assert did == O.restart_rule(e, sb["e_anchor"], sb["e_prev"], int(sb["k"]) + 1,
                                     int(sb["total"]) + 1)
        if not did:
            assert sa["e_prev"] == e
            continue
        n_restart += 1
        xc, yc = S.get_iterate(4)
        assert np.array_equal(ga["x0"], xc) and np.array_equal(ga["y0"], yc)
        assert np.array_equal(ga["x"], xc) and np.array_equal(ga["y"], yc)
        dxn = np.sqrt(((xc - gb["x0"]) ** 2).sum())
        dyn = np.sqrt(((yc - gb["y0"]) ** 2).sum())
        om = O.primal_weight(dxn, dyn, sb["omega"])
        assert abs(sa["omega"] - om) <= 1e-13 * om
        assert abs(om - math.sqrt(dyn / dxn * sb["omega"])) <= 1e-12 * om   # theta = 1/2
        assert sa["e_anchor"] == e and sa["k"] == 0 and sa["W"] == 0.0 and sa["beta"] == 1.0
    assert n_restart >= 2 and n_check > n_restart


def test_start_point_is_the_projection_of_zero():
    """Reading A4: z^{0,0} = (P_X(0), 0) in the scaled space; for bounds
    l = 0.5 > 0 and u = -1 < 0 the start sits on the bound (q-scaled, reading A2)."""
    p = tiny([[1.0, 1.0, 2.0], [0.0, 1.0, -1.0]], [1.0, 1.0, 1.0], [1.0, 2.0],
             [0.5, -INF, -INF], [INF, -1.0, INF], [NONNEG], [2])
    S = O.OracleSolver(p)
    _, q = S.get_scaling()
    x, y = S.get_iterate(0)
    assert np.array_equal(x, [0.5 * q[0], -1.0 * q[1], 0.0]) and np.all(y == 0)
