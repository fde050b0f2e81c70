"""GPU parity: the CUDA path (C ABI, libpdcs.so) vs the CPU oracle (-m gpu).

Tolerance (BASELINE.json north_star): per iterate, on scaled iterates,
    max(|x_g - x_o|_inf / (1 + |x_o|_inf), |y_g - y_o|_inf / (1 + |y_o|_inf)) <= 1e-9
(fp64; reduction order, FMA contraction and the root-finder method differ).
"""
import numpy as np
import pytest

import oracle as O
from instances import gen_fisher, gen_lasso, gen_mixed, gen_mpo, EXP, DUAL_EXP, SOC, RSOC

pytestmark = pytest.mark.gpu

TOL = 1e-9
# eta, omega, W are functions of differences dz = z^ - z; near convergence
# |dz|/|z| ~ 1e-5, so a 1e-14 iterate difference moves them by ~1e-9 relative
# (condition number |z|/|dz|).  They are compared at STOL (reading P2).
STOL = 1e-6


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


def mixed(seed, m=300, n1=60, n2=150, **kw):
    return gen_mixed(m, n1, n2, seed=seed, **kw)


# ------------------------------------------------------------------ setup parity
@pytest.mark.parametrize("make", [lambda: gen_lasso(100, 50, 1.0, dense=True),
                                  lambda: mixed(1), lambda: gen_fisher(30, 20, seed=1),
                                  lambda: gen_mpo(2, 15, seed=1)])
def test_scaling_parity(P, make):
    prog = make()
    g = P.PdcsSolver(prog)
    o = O.OracleSolver(prog)
    rg, qg = g.get_scaling()
    ro, qo = o.get_scaling()
    np.testing.assert_allclose(rg, ro, rtol=1e-13)
    np.testing.assert_allclose(qg, qo, rtol=1e-13)


# ------------------------------------------------------------------ one step from random points
@pytest.mark.parametrize("seed", range(4))
def test_one_step_random_point_all_cones(P, seed):
    """One Eq. 5 step from a random point: exercises every projection kernel
    (box, R+, zero, rescaled SOC/RSOC, exp, dual exp; thread/warp/CTA teams)."""
    prog = mixed(seed, m=600, n1=80, n2=400, soc_dims=(3, 300), scale_spread=1.5)
    rng = np.random.default_rng(seed)
    g = P.PdcsSolver(prog)
    o = O.OracleSolver(prog)
    ro, qo = o.get_scaling()
    for _ in range(3):
        x = rng.standard_normal(prog.n) * 3
        y = rng.standard_normal(prog.m) * 3
        g.set_iterate(x, y)               # original space
        o.set_iterate(x * qo, y * ro)     # oracle takes scaled space
        g.iterate(1)
        o.iterate(1)
        xg, yg = g.get_iterate(P.PDHG_OUT)
        xo, yo = o.get_iterate(1)
        assert parity(xg, yg, xo, yo) <= 1e-12, parity(xg, yg, xo, yo)


# ------------------------------------------------------------------ multi-step parity
@pytest.mark.parametrize("name,make,steps", [
    ("tiny_lasso", lambda: gen_lasso(100, 50, 1.0, dense=True), 500),
    ("mixed", lambda: mixed(5), 400),
    ("fisher", lambda: gen_fisher(40, 30, seed=2), 400),
])
def test_vanilla_parity(P, name, make, steps):
    """Vanilla PDHG (decision-free) per-iterate parity."""
    prog = make()
    g = P.PdcsSolver(prog, vanilla_pdhg=1)
    o = O.OracleSolver(prog, vanilla_pdhg=1)
    worst = 0.0
    for chunk in range(steps // 100):
        g.iterate(100)
        o.iterate(100)
        xg, yg = g.get_iterate(P.CURRENT)
        xo, yo = o.get_iterate(0)
        worst = max(worst, parity(xg, yg, xo, yo))
    assert worst <= TOL, worst


def _free_running(P, prog, steps, every=40):
    """Both implementations from the same start, no resets."""
    g = P.PdcsSolver(prog)
    o = O.OracleSolver(prog)
    worst = []
    for done in range(0, steps, every):
        rg = g.iterate(every)
        o.iterate(every)
        xg, yg = g.get_iterate(P.CURRENT)
        xo, yo = o.get_iterate(0)
        worst.append(parity(xg, yg, xo, yo))
        so = o.scalars()
        assert rg["restarts"] == so["restarts"] and rg["trials"] == so["trials"], (done, rg, so)
    return worst


def _shadow(P, prog, steps, seg=10, floor=None):
    """Checkpoint shadowing: at every check-interval
    boundary of the oracle's trajectory (every `seg` accepted iterations; every
    4th segment ends on an Eq. 9 check, restart and primal-weight decision) the
    GPU is loaded with the oracle's exact state (pdcs_set_state) and both run one
    segment.  Every segment must agree to TOL."""
    g = P.PdcsSolver(prog)
    o = O.OracleSolver(prog)
    worst = 0.0
    for s in range(0, steps, seg):
        st = o.get_state()
        if floor is not None and st["sc"][8] < floor:
            return worst, s       # solved to the rounding floor: the rest is noise
        g.set_state(st)
        g.iterate(seg)
        o.iterate(seg)
        xg, yg = g.get_iterate(P.CURRENT)
        xo, yo = o.get_iterate(0)
        worst = max(worst, parity(xg, yg, xo, yo))
        sg, so = g.get_state(), o.get_state()
        # decisions exact (k, total, trials, restarts, beta); eta/omega/W to STOL
        assert np.array_equal(sg["sc"][9:], so["sc"][9:]), (s, sg["sc"], so["sc"])
        assert sg["sc"][3] == so["sc"][3], (s, sg["sc"], so["sc"])
        # near the optimum eta-bar = ||dz||^2 / (2 |<dy, K dx>|) is a ratio of
        # differences of size e |z| (e = the best Eq. 9 error so far), so its
        # rounding error grows like 1/e: the tolerance widens below e = 1e-5
        # (measured on configs[0]: 4.9e-6 relative at e = 1e-7, 8.5e-2 at e = 2.4e-11)
        stol = STOL * max(1.0, 1e-5 / max(st["sc"][8], 1e-12))
        for i in (0, 2, 4):
            assert abs(sg["sc"][i] - so["sc"][i]) <= stol * abs(so["sc"][i]), (s, i, stol, sg["sc"], so["sc"])
        worst = max(worst, rel(sg["x0"], so["x0"]), rel(sg["y0"], so["y0"]))
        if so["sc"][4] > 0:   # the average z = sum eta z / sum eta (Alg. 1 line 7)
            worst = max(worst, rel(sg["xsum"] / sg["sc"][4], so["xsum"] / so["sc"][4]),
                        rel(sg["ysum"] / sg["sc"][4], so["ysum"] / so["sc"][4]))
    return (worst, steps) if floor is not None else worst


def test_pdcs_parity_tiny_lasso_2000(P):
    """BASELINE configs[0]: tiny Lasso SOCP 100x50 dense, fixed 2000 accepted PDHG
    iterations.  PDCS amplifies rounding (tests/test_sensitivity.py), so the
    2000-step comparison is made segment by segment from the oracle's state; the
    free-running comparison is held to TOL over the first 200 iterations."""
    prog = gen_lasso(100, 50, 1.0, seed=0, dense=True)
    # the balanced form (P9) is solved to Eq. 9 ~ 1e-13 by iteration ~600;
    # past the 1e-10 floor the step and restart decisions are taken on
    # rounding noise (P5), so the shadow stops there ...
    worst, stop = _shadow(P, prog, 2000, floor=1e-10)
    assert worst <= TOL and 300 <= stop < 2000, (worst, stop)
    free = _free_running(P, prog, 200)
    assert max(free) <= TOL, free
    # ... and the full 2000 iterations, free-running, end at the same optimum
    g = P.PdcsSolver(prog)
    o = O.OracleSolver(prog)
    g.iterate(2000)
    o.iterate(2000)
    xg, yg = g.get_iterate(P.CURRENT)
    xo, yo = o.get_iterate(0)
    assert parity(xg, yg, xo, yo) <= 1e-8, parity(xg, yg, xo, yo)


def test_pdcs_parity_tiny_lasso_2000_literal_form(P):
    """configs[0] in the literal form of PAPER.md:1641-1659 (balance=False,
    reading P9): the trajectory that stalls far from the optimum, 2000 steps
    segment by segment."""
    prog = gen_lasso(100, 50, 1.0, seed=0, dense=True, balance=False)
    worst = _shadow(P, prog, 2000)
    assert worst <= TOL, worst


@pytest.mark.parametrize("name,make,steps", [
    ("mixed", lambda: mixed(7), 800),
    ("mixed_big_soc", lambda: mixed(8, m=800, n1=50, n2=600, soc_dims=(30, 400)), 400),
    ("fisher", lambda: gen_fisher(40, 30, seed=3), 800),
    ("mpo", lambda: gen_mpo(3, 20, seed=3), 800),
])
def test_pdcs_parity(P, name, make, steps):
    prog = make()
    worst = _shadow(P, prog, steps)
    assert worst <= TOL, worst
    free = _free_running(P, prog, 120)
    assert max(free) <= TOL, free


# ------------------------------------------------------------------ Eq. 9
@pytest.mark.parametrize("seed", range(2))
def test_kkt_parity_same_point(P, seed):
    prog = mixed(20 + seed)
    g = P.PdcsSolver(prog)
    o = O.OracleSolver(prog)
    rng = np.random.default_rng(seed)
    ro, qo = o.get_scaling()
    x = prog.x_star + 0.01 * rng.standard_normal(prog.n)
    y = prog.y_star + 0.01 * rng.standard_normal(prog.m)
    g.set_iterate(x, y)
    o.set_iterate(x * qo, y * ro)
    kg = g.kkt(P.CURRENT)
    ko = o.kkt(0)
    for key in ("err_p", "err_d", "err_gap", "pobj", "dobj"):
        assert abs(kg[key] - ko[key]) <= 1e-12 * (1 + abs(ko[key])), (key, kg, ko)
    # at the planted optimum all three vanish
    g.set_iterate(prog.x_star, prog.y_star)
    k = g.kkt(P.CURRENT)
    assert max(k["err_p"], k["err_d"], k["err_gap"]) < 1e-12


# ------------------------------------------------------------------ solve
def test_solve_tiny_lasso(P):
    prog = gen_lasso(100, 50, 1.0, seed=0, dense=True)
    g = P.PdcsSolver(prog, tol=1e-6)
    r = g.solve()
    assert r["status"] == "OPTIMAL"
    assert max(r["err_p"], r["err_d"], r["err_gap"]) <= 1e-6
    ro = O.OracleSolver(prog, tol=1e-6).solve()
    assert abs(r["pobj"] - ro.kkt.pobj) <= 1e-5 * abs(ro.kkt.pobj)


@pytest.mark.parametrize("seed", range(2))
def test_solve_planted_mixed(P, seed):
    prog = mixed(30 + seed, m=400, n1=60, n2=200)
    g = P.PdcsSolver(prog, tol=1e-8, max_iters=200000)
    r = g.solve()
    assert r["status"] == "OPTIMAL"
    assert abs(r["pobj"] - prog.obj_star) <= 1e-6 * (1 + abs(prog.obj_star))


def test_solve_fisher_and_mpo(P):
    for prog, tol in ((gen_fisher(50, 40, seed=4), 1e-6), (gen_mpo(3, 30, seed=4), 1e-6)):
        g = P.PdcsSolver(prog, tol=tol, max_iters=200000)
        r = g.solve()
        assert r["status"] == "OPTIMAL", r
        assert max(r["err_p"], r["err_d"], r["err_gap"]) <= tol


def test_set_tolerance_continues_trajectory(P):
    """Solve to 1e-3, pdcs_set_tolerance(1e-6), solve again: the continued run
    is the same trajectory as one solve straight to 1e-6 (stops land on Eq. 9
    checks, the state is kept), so the iteration count and iterate bits match."""
    prog = gen_lasso(100, 50, 1.0, seed=0, dense=True)
    g = P.PdcsSolver(prog, tol=1e-3)
    r1 = g.solve()
    assert r1["status"] == "OPTIMAL" and max(r1["err_p"], r1["err_d"], r1["err_gap"]) <= 1e-3
    g.set_tolerance(1e-6)
    r2 = g.solve()
    assert r2["status"] == "OPTIMAL" and max(r2["err_p"], r2["err_d"], r2["err_gap"]) <= 1e-6
    h = P.PdcsSolver(prog, tol=1e-6)
    r3 = h.solve()
    assert r2["iters"] == r3["iters"] and r2["restarts"] == r3["restarts"]
    x2, y2 = g.get_iterate(P.BEST)
    x3, y3 = h.get_iterate(P.BEST)
    assert np.array_equal(x2, x3) and np.array_equal(y2, y3)
    with pytest.raises(P.PdcsError):
        g.set_tolerance(-1.0)


# ------------------------------------------------------------------ boundary errors
def test_create_errors(P):
    prog = gen_lasso(10, 5, 1.0, dense=True)
    bad = prog.vals.copy()
    bad[3] = np.nan
    import copy
    p2 = copy.copy(prog)
    p2.vals = bad
    with pytest.raises(P.PdcsError) as e:
        P.PdcsSolver(p2)
    assert e.value.code == 4
    p3 = copy.copy(prog)
    p3.l = prog.l.copy()
    p3.u = prog.u.copy()
    p3.l[0], p3.u[0] = 1.0, 0.0
    with pytest.raises(P.PdcsError) as e:
        P.PdcsSolver(p3)
    assert e.value.code == 3
    p4 = copy.copy(prog)
    p4.pdim = prog.pdim + 1
    with pytest.raises(P.PdcsError) as e:
        P.PdcsSolver(p4)
    assert e.value.code == 5
    p5 = copy.copy(prog)
    p5.pk = np.array([EXP], np.int32)
    with pytest.raises(P.PdcsError) as e:
        P.PdcsSolver(p5)
    assert e.value.code == 5


def test_empty_and_degenerate(P):
    """Zero-nnz rows / columns, and an instance whose optimum is the origin."""
    from instances import ConicProgram, ZERO, NONNEG
    prog = ConicProgram(m=3, n=3, n1=3, row_ptr=np.array([0, 0, 1, 1], np.int64),
                        col_idx=np.array([1], np.int32), vals=np.array([2.0]), c=np.array([1.0, 1.0, 0.0]),
                        h=np.array([0.0, 0.0, 0.0]), l=np.zeros(3), u=np.full(3, np.inf),
                        pk=np.zeros(0, np.int32), pdim=np.zeros(0, np.int64),
                        rk=np.array([NONNEG], np.int32), rdim=np.array([3], np.int64))
    g = P.PdcsSolver(prog, tol=1e-8)
    r = g.solve()
    assert r["status"] == "OPTIMAL" and abs(r["pobj"]) < 1e-8


# ------------------------------------------------------------------ tiled SpMV path forced
@pytest.fixture
def tiled_env(monkeypatch):
    """Force the column-tiled SpMV (tiled.cuh) regardless of the setup autotune."""
    monkeypatch.setenv("PDCS_TILED", "1")
    monkeypatch.setenv("PDCS_TILE_KB", "1")        # tiny tiles -> many staged segments
    yield


@pytest.mark.parametrize("seed", range(2))
def test_tiled_one_step_and_shadow(P, tiled_env, seed):
    prog = mixed(40 + seed, m=900, n1=120, n2=500, soc_dims=(3, 120), row_len=(20, 90))
    rng = np.random.default_rng(seed)
    g = P.PdcsSolver(prog)
    sc = g.scalars()
    assert sc["tiled_K"] == 1.0 and sc["tiled_KT"] == 1.0
    o = O.OracleSolver(prog)
    ro, qo = o.get_scaling()
    x = rng.standard_normal(prog.n) * 3
    y = rng.standard_normal(prog.m) * 3
    g.set_iterate(x, y)
    o.set_iterate(x * qo, y * ro)
    g.iterate(1)
    o.iterate(1)
    xg, yg = g.get_iterate(P.PDHG_OUT)
    xo, yo = o.get_iterate(1)
    assert parity(xg, yg, xo, yo) <= 1e-12
    worst = _shadow(P, prog, 200)
    assert worst <= TOL, worst


def test_tiled_tma_pipeline_parity(P, tiled_env, monkeypatch):
    """The TMA-pipelined tiled kernel (cp.async.bulk + mbarrier ring, opt-in)."""
    monkeypatch.setenv("PDCS_TMA", "1")
    prog = mixed(45, m=900, n1=120, n2=500, soc_dims=(3, 120), row_len=(20, 90))
    worst = _shadow(P, prog, 120)
    assert worst <= TOL, worst
    prog = gen_lasso(400, 300, 0.2, seed=6)
    g = P.PdcsSolver(prog, vanilla_pdhg=1)
    o = O.OracleSolver(prog, vanilla_pdhg=1)
    g.iterate(200)
    o.iterate(200)
    xg, yg = g.get_iterate(P.CURRENT)
    xo, yo = o.get_iterate(0)
    assert parity(xg, yg, xo, yo) <= TOL


def test_tiled_lasso_vanilla_parity(P, tiled_env):
    prog = gen_lasso(400, 300, 0.2, seed=5)
    g = P.PdcsSolver(prog, vanilla_pdhg=1)
    assert g.scalars()["tiled_K"] == 1.0
    o = O.OracleSolver(prog, vanilla_pdhg=1)
    g.iterate(300)
    o.iterate(300)
    xg, yg = g.get_iterate(P.CURRENT)
    xo, yo = o.get_iterate(0)
    assert parity(xg, yg, xo, yo) <= TOL


def test_tiled_build_threads_and_bank_balance(P, tiled_env, monkeypatch):
    """The tiled format is built on host threads (one contiguous chunk range
    each) and concatenated: the result must not depend on the thread count
    (bit-identical iterates).  Bank balancing only permutes entries within a
    row, so it changes nothing but the summation order."""
    monkeypatch.setenv("PDCS_TILE_KB", "4")
    prog = gen_lasso(12000, 400, 0.05, seed=8)
    runs = {}
    for key, env in {"t1": {"PDCS_BUILD_THREADS": "1"}, "t5": {"PDCS_BUILD_THREADS": "5"},
                     "nobal": {"PDCS_BUILD_THREADS": "3", "PDCS_TILE_BALANCE": "0"}}.items():
        for k in ("PDCS_BUILD_THREADS", "PDCS_TILE_BALANCE"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        g = P.PdcsSolver(prog, vanilla_pdhg=1)
        assert g.scalars()["tiled_K"] == 1.0 and g.scalars()["tiled_KT"] == 1.0
        g.iterate(60)
        runs[key] = g.get_iterate(P.CURRENT)
        g.close()
    assert np.array_equal(runs["t1"][0], runs["t5"][0]) and np.array_equal(runs["t1"][1], runs["t5"][1])
    assert parity(*runs["t1"], *runs["nobal"]) <= 1e-12
    o = O.OracleSolver(prog, vanilla_pdhg=1)
    o.iterate(60)
    assert parity(*runs["t1"], *o.get_iterate(0)) <= TOL


def test_fused_combine_matches_partial_plus_combine(P, tiled_env, monkeypatch):
    """The fused combine (the last work item of a chunk sums the chunk's group
    partials and runs the epilogue, tiled.cuh k_tiled_sliced<ELEM, Epi>) adds
    the same partials in the same order as k_tiled_combine: with fixed steps
    (vanilla PDHG) the iterates are bit-identical; with the line search only
    the epilogue's accumulator order differs (per chunk instead of per combine
    CTA).  Chunks of one and of many work items (TILE_GROUP) both occur."""
    monkeypatch.setenv("PDCS_TILE_KB", "2")
    prog = gen_lasso(5000, 400, 0.05, seed=9)
    for vanilla in (1, 0):
        runs = {}
        for fused in ("1", "0"):
            for grp in ("4000", "1000000"):
                monkeypatch.setenv("PDCS_FUSED_COMBINE", fused)
                monkeypatch.setenv("PDCS_TILE_GROUP", grp)
                g = P.PdcsSolver(prog, vanilla_pdhg=vanilla)
                assert g.scalars()["tiled_K"] == 1.0 and g.scalars()["tiled_KT"] == 1.0
                g.iterate(80)
                runs[(fused, grp)] = g.get_iterate(P.CURRENT)
                g.close()
        for grp in ("4000", "1000000"):
            a, b = runs[("1", grp)], runs[("0", grp)]
            if vanilla:
                assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
            else:
                assert parity(*a, *b) <= 1e-11


def test_warm_started_soc_multipliers(P, monkeypatch):
    """The trial projections start each SOC/RSOC Newton iteration from 90% of
    the block's previous multiplier (soc_team, PDCS_WARM).  The root is the
    same one as from a cold start, so 60 PDCS iterations with and without the
    warm start agree to rounding, and checkpoint shadowing against the oracle
    (the GPU reloaded with the oracle's state every 10 iterations, its warm
    values left from other points) holds at TOL."""
    prog = mixed(17, m=900, n1=120, n2=500, soc_dims=(3, 200))
    runs = {}
    for warm in ("1", "0"):
        monkeypatch.setenv("PDCS_WARM", warm)
        g = P.PdcsSolver(prog)
        g.iterate(60)
        runs[warm] = g.get_iterate(P.CURRENT)
        g.close()
    assert parity(*runs["1"], *runs["0"]) <= 1e-10
    monkeypatch.setenv("PDCS_WARM", "1")
    worst = _shadow(P, prog, 120)
    assert worst <= TOL, worst


def test_memory_pool_reuse_gives_the_same_bits(P):
    """Device buffers come from the library's memory pool (pdcs.cu dev_alloc):
    later contexts reuse the memory earlier ones freed, including setup
    scratch.  Five create / iterate / destroy rounds of the same instance (the
    tiled formats forced, so the device structure build and its scratch run)
    give the first round's bits every time."""
    import os
    os.environ["PDCS_TILED"] = "1"
    try:
        prog = gen_lasso(3000, 400, 0.05, seed=12)
        ref = None
        for _ in range(5):
            g = P.PdcsSolver(prog)
            assert g.scalars()["tiled_K"] == 1.0
            g.iterate(50)
            xy = g.get_iterate(P.CURRENT)
            g.close()
            if ref is None:
                ref = xy
            assert np.array_equal(ref[0], xy[0]) and np.array_equal(ref[1], xy[1])
        assert P.pdcs_trim_memory() > 0            # every context is gone: their memory goes back
        g = P.PdcsSolver(prog)                     # and a context after the trim still gives the bits
        g.iterate(50)
        xy = g.get_iterate(P.CURRENT)
        g.close()
        assert np.array_equal(ref[0], xy[0]) and np.array_equal(ref[1], xy[1])
    finally:
        del os.environ["PDCS_TILED"]


def test_cfg5_recipe_parity(P):
    """SURVEY §8(d) cfg 5 recipe (row lengths 20..180, values over 8 decades,
    all six cone kinds, log-uniform SOC dims up to 4096 -> thread/warp/CTA
    teams, planted optimum) at a size the oracle runs in seconds: one Eq. 5
    step from random points at 1e-12, then checkpoint shadowing."""
    from instances import gen_mixed_large
    prog = gen_mixed_large(0.0003, seed=4)
    rng = np.random.default_rng(4)
    g = P.PdcsSolver(prog)
    o = O.OracleSolver(prog)
    ro, qo = o.get_scaling()
    rg, qg = g.get_scaling()
    np.testing.assert_allclose(rg, ro, rtol=1e-13)
    np.testing.assert_allclose(qg, qo, rtol=1e-13)
    for _ in range(2):
        x = rng.standard_normal(prog.n) * 3
        y = rng.standard_normal(prog.m) * 3
        g.set_iterate(x, y)
        o.set_iterate(x * qo, y * ro)
        g.iterate(1)
        o.iterate(1)
        assert parity(*g.get_iterate(P.PDHG_OUT), *o.get_iterate(1)) <= 1e-12
    g.close()
    worst = _shadow(P, prog, 120)
    assert worst <= TOL, worst


def test_cta_and_grid_teams_one_step(P):
    """Rescaled SOC / RSOC blocks on the CTA team (513..4096 entries), the
    thread-block-cluster team (4097..131072, DSMEM reductions) and the
    whole-grid cooperative team (> 131072): one Eq. 5 step from random points
    against the oracle's projection (Thm 1)."""
    prog = gen_mixed(3000, 100, 150000, seed=11, soc_dims=(600, 2000), scale_spread=1.5,
                     col_mix=[(SOC, 1.0)], row_len=(3, 12))
    assert prog.pdim.max() > 131072 or (prog.rdim.max() > 512)
    big = [d for k, d in zip(prog.pk, prog.pdim) if k == SOC]
    prog2 = gen_mixed(3000, 100, 150000, seed=12, soc_dims=(140000, 150000), scale_spread=1.5,
                      col_mix=[(SOC, 1.0)], row_len=(3, 12))
    assert max(d for k, d in zip(prog2.pk, prog2.pdim) if k == SOC) > 131072
    assert max(big) > 512
    prog3 = gen_mixed(3000, 100, 150000, seed=13, soc_dims=(5000, 40000), scale_spread=1.5,
                      col_mix=[(SOC, 0.7), (RSOC, 0.3)], row_len=(3, 12))
    assert any(4096 < d <= 131072 for d in prog3.pdim)            # cluster team
    for pr in (prog, prog2, prog3):
        rng = np.random.default_rng(7)
        g = P.PdcsSolver(pr)
        o = O.OracleSolver(pr)
        ro, qo = o.get_scaling()
        for _ in range(2):
            x = rng.standard_normal(pr.n) * 3
            y = rng.standard_normal(pr.m) * 3
            g.set_iterate(x, y)
            o.set_iterate(x * qo, y * ro)
            g.iterate(1)
            o.iterate(1)
            assert parity(*g.get_iterate(P.PDHG_OUT), *o.get_iterate(1)) <= 1e-12
        g.close()


@pytest.mark.parametrize("fuse", ["0", "1"])
def test_fused_y_update_bit_identical(P, monkeypatch, fuse):
    """The y-side Halpern update folded into k_decide (m <= 2048) computes the
    same formula in the same order as k_halpern_y: 300 iterations with and
    without it give the same bits, and both match the oracle."""
    prog = mixed(11, m=500, n1=60, n2=200)
    monkeypatch.setenv("PDCS_FUSE_Y", "1")
    a = P.PdcsSolver(prog)
    a.iterate(300)
    monkeypatch.setenv("PDCS_FUSE_Y", fuse)
    b = P.PdcsSolver(prog)
    b.iterate(300)
    xa, ya = a.get_iterate(P.CURRENT)
    xb, yb = b.get_iterate(P.CURRENT)
    assert np.array_equal(xa, xb) and np.array_equal(ya, yb)
    o = O.OracleSolver(prog)
    o.iterate(120)
    c = P.PdcsSolver(prog)
    c.iterate(120)
    xc, yc = c.get_iterate(P.CURRENT)
    xo, yo = o.get_iterate(0)
    assert parity(xc, yc, xo, yo) <= TOL


def test_set_iterate_mid_run_starts_new_epoch(P):
    """pdcs_set_iterate after some iterations starts a new epoch at the point
    (include/pdcs.h): the oracle's set_iterate does the same, so the two agree
    on the steps that follow (k, W, sums, beta reset; eta, omega, counters kept)."""
    prog = mixed(13, m=400, n1=60, n2=200)
    g = P.PdcsSolver(prog)
    o = O.OracleSolver(prog)
    ro, qo = o.get_scaling()
    g.iterate(60)
    o.iterate(60)
    rng = np.random.default_rng(13)
    x, y = rng.standard_normal(prog.n), rng.standard_normal(prog.m)
    # eta / omega carry over and differ by rounding after 60 steps: hand the
    # GPU the oracle's exact state first, then restart both at the point
    g.set_state(o.get_state())
    g.set_iterate(x, y)
    o.set_iterate(x * qo, y * ro)
    sg, so = g.get_state(), o.get_state()
    assert np.array_equal(sg["sc"][9:], so["sc"][9:]) and sg["sc"][3] == so["sc"][3], (sg["sc"], so["sc"])
    assert sg["sc"][4] == 0.0 and so["sc"][4] == 0.0
    g.iterate(40)
    o.iterate(40)
    assert parity(*g.get_iterate(P.CURRENT), *o.get_iterate(0)) <= TOL


@pytest.mark.parametrize("make", [lambda: gen_lasso(100, 50, 1.0, seed=0, dense=True),
                                  lambda: gen_mixed(200, 30, 80, seed=4, soc_dims=(3, 20))])
def test_set_tolerance_continuation_against_oracle(P, make):
    """pdcs_set_tolerance on the GPU against the oracle (not only GPU against GPU):
    solve to 1e-3, continue to 1e-6.  At each stage the returned point is
    certified by the ORACLE's Eq. 9 at that point (<= the stage's tolerance), and
    its objective agrees with the oracle's own solve to the same tolerance."""
    prog = make()
    g = P.PdcsSolver(prog, tol=1e-3, max_iters=400000)
    o_check = O.OracleSolver(prog)
    for tol, otol in ((1e-3, 5e-3), (1e-6, 1e-5)):
        if tol < 1e-3:
            g.set_tolerance(tol)
        r = g.solve()
        assert r["status"] == "OPTIMAL", r
        xb, yb = g.get_iterate(P.BEST, P.ORIGINAL)
        k = o_check.kkt_point(xb, yb)
        assert max(k["err_p"], k["err_d"], k["err_gap"]) <= tol * (1 + 1e-9), (tol, k)
        ro = O.OracleSolver(prog, tol=tol, max_iters=400000).solve()
        assert ro.status == 0
        assert abs(r["pobj"] - ro.kkt.pobj) <= otol * (1 + abs(ro.kkt.pobj)), (tol, r["pobj"], ro.kkt.pobj)


def test_caller_allocator(P):
    """pdcs_set_allocator: every device buffer of a context comes from the
    caller's allocator (here torch's caching allocator through ctypes
    callbacks), all of it is returned at destroy, and the iterates are the
    default allocator's bits."""
    import torch
    live = {}
    stats = {"alloc": 0, "free": 0}

    def alloc(nbytes):
        p = torch.cuda.caching_allocator_alloc(nbytes)
        live[p] = nbytes
        stats["alloc"] += 1
        return p

    def free(ptr):
        live.pop(ptr)
        torch.cuda.caching_allocator_delete(ptr)
        stats["free"] += 1

    prog = mixed(6)
    P.pdcs_set_allocator(alloc, free)
    try:
        g = P.PdcsSolver(prog)
        g.iterate(100)
        xa, ya = g.get_iterate(P.CURRENT)
        assert stats["alloc"] > 20 and live
        g.close()
        assert not live and stats["free"] == stats["alloc"]
    finally:
        P.pdcs_set_allocator(None, None)
    g = P.PdcsSolver(prog)
    g.iterate(100)
    xb, yb = g.get_iterate(P.CURRENT)
    assert np.array_equal(xa, xb) and np.array_equal(ya, yb)


def test_balanced_lasso_solves_to_1e4_and_maps_to_the_literal_form(P):
    """Reading P9 at a size the oracle still solves in seconds (2e4 x 2e3 at 1%,
    the tall P8 proxy): the GPU solves the balanced form to Eq. 9 <= 1e-4; its
    best point, mapped back (w = w'/S, r = S r'), scores <= 1e-4 on the
    LITERAL form's Eq. 9 in a second GPU context; its objective is the Lasso
    objective ||A x - b||^2 + lam ||x||_1 evaluated directly from (A, b) at
    x = x+ - x- (PAPER.md:1641-1659), and agrees with the oracle's solve of
    the same balanced program to the accuracy both stop at."""
    prog = gen_lasso(20000, 2000, 0.01, seed=0)
    g = P.PdcsSolver(prog, tol=1e-4)
    r = g.solve()
    assert r["status"] == "OPTIMAL", r
    x, y = g.get_iterate(P.BEST, P.ORIGINAL)
    g.close()
    lit = P.PdcsSolver(prog.literal())
    lit.set_iterate(prog.to_literal(x), y)
    k = lit.kkt(P.CURRENT)
    lit.close()
    assert max(k["err_p"], k["err_d"], k["err_gap"]) <= 1e-4, k
    arow, acol, aval, m, nf = prog.lasso_A
    xf = x[:nf] - x[nf:2 * nf]
    resid = np.bincount(arow, weights=aval * xf[acol], minlength=m) - prog.lasso_b
    f = float(resid @ resid) + prog.lasso_lam * float(np.abs(xf).sum())
    assert abs(k["pobj"] - f) <= 1e-3 * f, (k["pobj"], f)
    ro = O.OracleSolver(prog, tol=1e-4, max_iters=20000).solve()
    assert ro.status == 0
    assert abs(k["pobj"] - ro.kkt.pobj) <= 1e-3 * abs(ro.kkt.pobj), (k["pobj"], ro.kkt.pobj)
