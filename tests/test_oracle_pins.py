"""Pins for the CPU oracle against what the paper and mathematics fix (-m "not gpu").

Each pin is independent of the oracle's own formulas: printed examples
(tests/golden/spec_examples.json), closed forms, certificates that
characterise a projection uniquely (Moreau, Lemma 2),
50-digit mpmath solutions of the paper's literal equations, dense brute force,
and planted KKT pairs whose optimum is known exactly.
"""
import json
import math
import os

import mpmath as mp
import numpy as np
import pytest

import oracle as O
from instances import (ConicProgram, gen_fisher, gen_lasso, gen_mixed, gen_mpo, ZERO, NONNEG,
                       SOC, RSOC, EXP, DUAL_EXP)

HERE = os.path.dirname(os.path.abspath(__file__))
G = json.load(open(os.path.join(HERE, "golden", "spec_examples.json")))


def csr(A):
    A = np.asarray(A, float)
    m, n = A.shape
    ptr = [0]
    col, val = [], []
    for i in range(m):
        for j in range(n):
            if A[i, j] != 0:
                col.append(j)
                val.append(A[i, j])
        ptr.append(len(col))
    return np.array(ptr, np.int64), np.array(col, np.int32), np.array(val)


# ------------------------------------------------------------------ SpMV
def test_spmv_spec_examples():
    for e in G["spmv"]:
        p, c, v = csr(e["A"])
        assert np.array_equal(O.spmv(p, c, v, e["x"]), e["Ax"]), e["cite"]
    for e in G["spmv_t"]:
        p, c, v = csr(e["A"])
        assert np.array_equal(O.spmv_t(p, c, v, e["y"], 2), e["ATy"]), e["cite"]


def test_spmv_empty_and_dense_bruteforce():
    p = np.zeros(4, np.int64)
    assert np.array_equal(O.spmv(p, np.zeros(0, np.int32), np.zeros(0), np.ones(5)), np.zeros(3))
    rng = np.random.default_rng(0)
    A = rng.standard_normal((20, 30)) * (rng.uniform(size=(20, 30)) < 0.3)
    p, c, v = csr(A)
    x, y = rng.standard_normal(30), rng.standard_normal(20)
    np.testing.assert_allclose(O.spmv(p, c, v, x), A @ x, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(O.spmv_t(p, c, v, y, 30), A.T @ y, rtol=1e-13, atol=1e-13)
    # adjoint identity
    lhs = y @ O.spmv(p, c, v, x)
    rhs = O.spmv_t(p, c, v, y, 30) @ x
    assert abs(lhs - rhs) <= 1e-12 * (1 + abs(lhs))


# ------------------------------------------------------------------ SOC
def soc_cert(v, p, D=None):
    """Moreau certificate for P_{D K_soc}: p in DK, p - v in (DK)^* = D^-1 K, <p, p-v> = 0."""
    D = np.ones(len(v)) if D is None else np.asarray(D, float)
    w = p / D
    z = (p - v) * D
    scale = 1 + np.linalg.norm(v)
    return (np.linalg.norm(w[1:]) - w[0] <= 1e-10 * scale * (1 + np.max(1 / D)),
            np.linalg.norm(z[1:]) - z[0] <= 1e-10 * scale * (1 + np.max(D)),
            abs(p @ (p - v)) <= 1e-10 * scale ** 2)


def test_soc_unit_examples_and_certificate():
    for e in G["soc_unit"]:
        np.testing.assert_allclose(O.proj_soc_unit(e["v"]), e["out"], atol=1e-15, err_msg=e["cite"])
    rng = np.random.default_rng(1)
    for _ in range(500):
        d = int(rng.integers(2, 9))
        v = rng.standard_normal(d) * 10 ** rng.uniform(-2, 2)
        assert all(soc_cert(v, O.proj_soc_unit(v)))


def mp_soc_literal(t, x, dhat, dps=50):
    """Thm 1 case (iv) literally: root of Eq. 7 at 50 digits,
    y = (I + 2 lam Dhat^-2)^-1 x, s = t/(1-2lam)."""
    mp.mp.dps = dps
    t = mp.mpf(t)
    x = [mp.mpf(a) for a in x]
    dh = [mp.mpf(a) for a in dhat]

    def f(lam):
        return sum((xi / di / (1 + 2 * lam / di ** 2)) ** 2 for xi, di in zip(x, dh)) - t ** 2 / (1 - 2 * lam) ** 2

    if t > 0:      # root in (0, 1/2): f(0+) > 0 > f(1/2-)
        a, b = mp.mpf(0), mp.mpf("0.5")
        fa = f(a)
        for _ in range(400):
            mid = (a + b) / 2
            fm = f(mid)
            if (fm > 0) == (fa > 0):
                a, fa = mid, fm
            else:
                b = mid
        lam = (a + b) / 2
    else:          # root lam > 1/2; bisect in mu = 1/(2 lam) in (0, 1)
        a, b = mp.mpf(10) ** (-45), 1 - mp.mpf(10) ** (-45)
        ga = f(1 / (2 * a))
        for _ in range(400):
            mid = (a + b) / 2
            gm = f(1 / (2 * mid))
            if (gm > 0) == (ga > 0):
                a, ga = mid, gm
            else:
                b = mid
        lam = 1 / (a + b)
    y = [xi / (1 + 2 * lam / di ** 2) for xi, di in zip(x, dh)]
    s = t / (1 - 2 * lam)
    return np.array([float(s)] + [float(v) for v in y])


def test_soc_scaled_spec_examples():
    e = G["soc_scaled_case1"][0]
    out = O.proj_soc_scaled([e["t"]] + e["x"], [1.0] + e["dhat"])
    np.testing.assert_array_equal(out, e["out"])
    e = G["soc_scaled_root"][0]
    out = O.proj_soc_scaled([e["t"]] + e["x"], [1.0] + e["dhat"])
    ref = mp_soc_literal(e["t"], e["x"], e["dhat"])
    np.testing.assert_allclose(out, ref, rtol=1e-14, atol=1e-14, err_msg=e["cite"])
    assert all(soc_cert(np.array([e["t"]] + e["x"], float), out, [1.0] + e["dhat"]))


def test_soc_scaled_unit_and_uniform_closed_forms():
    rng = np.random.default_rng(2)
    for _ in range(1000):
        d = int(rng.integers(2, 7))
        v = rng.standard_normal(d) * 10 ** rng.uniform(-1, 1)
        # unit scaling reduces Thm 1 to the textbook SOC (acceptance 3)
        np.testing.assert_allclose(O.proj_soc_scaled(v, np.ones(d)), O.proj_soc_unit(v),
                                   rtol=1e-12, atol=1e-12)
        # uniform dhat = c: D K_soc = SOC with slope 1/c; closed form
        c = 10 ** rng.uniform(-1.5, 1.5)
        t, x = v[0], v[1:]
        nx = np.linalg.norm(x)
        if nx / c <= t:
            ref = v
        elif t <= 0 and c * nx <= -t:
            ref = np.zeros(d)
        else:
            a = (t + c * nx) / (1 + c * c)
            ref = np.concatenate([[a], a * c * x / nx])
        D = np.concatenate([[1.0], np.full(d - 1, c)])
        np.testing.assert_allclose(O.proj_soc_scaled(v, D), ref, rtol=1e-11, atol=1e-11)


@pytest.mark.parametrize("seed", range(4))
def test_soc_scaled_vs_mpmath_literal_eq7(seed):
    rng = np.random.default_rng(100 + seed)
    for _ in range(25):
        d = int(rng.integers(2, 8))
        dhat = 10 ** rng.uniform(-2, 2, d - 1)
        v = rng.standard_normal(d)
        v[0] = rng.uniform(-1, 1) * np.linalg.norm(v[1:] * dhat) * 1.5
        D = np.concatenate([[1.0], dhat])
        out = O.proj_soc_scaled(v, D)
        t, x = v[0], v[1:]
        if (t <= 0 and np.linalg.norm(dhat * x) <= -t) or np.linalg.norm(x / dhat) <= t or t == 0:
            continue
        ref = mp_soc_literal(t, x, dhat)
        np.testing.assert_allclose(out, ref, rtol=1e-11, atol=1e-11 * (1 + np.linalg.norm(v)))
        assert all(soc_cert(v, out, D))


def test_soc_scaled_tiny_t_regression():
    """Reading A16: |t| << ||x|| (SPEC.md:239's bracket fails there)."""
    for t in (1e-9, -1e-13, 1e-300, -1e-300):
        v = np.array([t, 3.0, 4.0, 1e6])
        D = np.array([1.0, 2.0, 0.5, 1.0])
        out = O.proj_soc_scaled(v, D)
        assert all(soc_cert(v, out, D))


def test_rsoc_certificate():
    rng = np.random.default_rng(3)
    for _ in range(500):
        d = int(rng.integers(3, 8))
        v = rng.standard_normal(d)
        p = O.proj_rsoc_scaled(v)
        a, b, z = p[0], p[1], p[2:]
        q = p - v            # must lie in RSOC^* = RSOC (self-dual)
        assert a >= -1e-12 and b >= -1e-12 and z @ z <= 2 * a * b + 1e-10
        assert q[0] >= -1e-12 and q[1] >= -1e-12 and q[2:] @ q[2:] <= 2 * q[0] * q[1] + 1e-10
        assert abs(p @ q) <= 1e-10


def test_rsoc_scaled_equal_leading():
    rng = np.random.default_rng(4)
    for _ in range(300):
        d = int(rng.integers(3, 8))
        v = rng.standard_normal(d)
        D = 10 ** rng.uniform(-1, 1, d)
        D[1] = D[0]
        p = O.proj_rsoc_scaled(v, D)
        w = p / D          # in RSOC
        z = (p - v) * D    # in (D K)^* = D^-1 K  => D (p - v) in K
        assert w[0] >= -1e-10 and w[1] >= -1e-10 and w[2:] @ w[2:] <= 2 * w[0] * w[1] + 1e-9
        assert z[0] >= -1e-10 and z[1] >= -1e-10 and z[2:] @ z[2:] <= 2 * z[0] * z[1] + 1e-9
        assert abs(p @ (p - v)) <= 1e-10 * (1 + v @ v)


# ------------------------------------------------------------------ exponential cone
def mp_exp_reference(v, D, dps=60):
    """Independent reference for P_{D K_exp}(v): maximise <v,u>/||u|| over the
    curved boundary u(rho) = D (rho, 1, e^rho) (distance^2 = |v|^2 - F^2), compare
    with the face {s=0, r<=0, t>=0}, 0 and v itself (if inside) — Eq. 12
     parameterisation, no use of Thm 4's root function."""
    mp.mp.dps = dps
    r0, s0, t0 = (mp.mpf(a) for a in v)
    dr, ds, dt = (mp.mpf(a) for a in D)

    def F(rho):
        u = (dr * rho, ds, dt * mp.e ** rho)
        dotv = r0 * u[0] + s0 * u[1] + t0 * u[2]
        return dotv / mp.sqrt(u[0] ** 2 + u[1] ** 2 + u[2] ** 2)

    cands = []
    # inside?
    w = (r0 / dr, s0 / ds, t0 / dt)
    if (w[1] > 0 and w[2] >= w[1] * mp.e ** (w[0] / w[1])) or (w[1] == 0 and w[0] <= 0 and w[2] >= 0):
        return np.array([float(a) for a in (r0, s0, t0)])
    cands.append((mp.mpf(0), mp.mpf(0), mp.mpf(0)))
    cands.append((min(r0, 0), mp.mpf(0), max(t0, 0)))
    grid = np.concatenate([-np.logspace(5, np.log10(60), 300, endpoint=False),
                           np.linspace(-60, 40, 2001),
                           np.logspace(np.log10(40), 3, 100)[1:]])
    if s0 > 0:   # ratio r/s of v itself (where the t-raised boundary point lives)
        rho0 = float((r0 / dr) / (s0 / ds))
        grid = np.unique(np.concatenate([grid, rho0 + np.linspace(-5, 5, 101)]))
    vals = [float(F(mp.mpf(g))) for g in grid]
    i = int(np.argmax(vals))
    if vals[i] > 0:
        a, b = mp.mpf(grid[max(i - 1, 0)]), mp.mpf(grid[min(i + 1, len(grid) - 1)])
        gr = (mp.sqrt(5) - 1) / 2
        c1, c2 = b - gr * (b - a), a + gr * (b - a)
        f1, f2 = F(c1), F(c2)
        for _ in range(300):
            if f1 > f2:
                b, c2, f2 = c2, c1, f1
                c1 = b - gr * (b - a)
                f1 = F(c1)
            else:
                a, c1, f1 = c1, c2, f2
                c2 = a + gr * (b - a)
                f2 = F(c2)
        rho = (a + b) / 2
        u = (dr * rho, ds, dt * mp.e ** rho)
        uu = u[0] ** 2 + u[1] ** 2 + u[2] ** 2
        sp = (r0 * u[0] + s0 * u[1] + t0 * u[2]) / uu
        if sp > 0:
            cands.append(tuple(sp * ui for ui in u))
    best = min(cands, key=lambda p: (p[0] - r0) ** 2 + (p[1] - s0) ** 2 + (p[2] - t0) ** 2)
    return np.array([float(a) for a in best])


def exp_cert(v, p, D, tol=1e-9):
    """Moreau certificate (Lemma 2; Eq. 11):
    p in D K_exp, v - p in -D^-1 K_exp^*, <p, v - p> = 0."""
    v, p, D = (np.asarray(a, float) for a in (v, p, D))
    sc = 1 + np.linalg.norm(v)
    vd = v - p
    w = p / D
    z = -vd * D
    return (O.in_exp(w, tol * sc * (1 + np.max(1 / D))),
            O.in_exp_dual(z, tol * sc * (1 + np.max(D))),
            abs(p @ vd) <= tol * sc ** 2)


def test_exp_spec_examples():
    for e in G["exp"]:
        np.testing.assert_allclose(O.proj_exp_scaled(e["v"], e["d"]), e["out"], atol=1e-15,
                                   err_msg=e["cite"])
    for e in G["dual_exp"]:
        np.testing.assert_allclose(O.proj_dual_exp_scaled(e["v"], e["d"]), e["out"], atol=1e-15)


def test_exp_spec197_degenerate():
    """SPEC.md:197 sits on a3 = a4 (h has a pole there); the reference is the
    independent boundary maximisation at 60 digits (reading A18/A25)."""
    e = G["exp_degenerate"][0]
    out = O.proj_exp_scaled(e["v"], e["d"])
    ref = mp_exp_reference(e["v"], e["d"])
    np.testing.assert_allclose(out, ref, rtol=1e-13, atol=1e-14)
    assert all(exp_cert(e["v"], out, e["d"]))


@pytest.mark.parametrize("seed", range(4))
def test_exp_vs_independent_reference(seed):
    rng = np.random.default_rng(200 + seed)
    for _ in range(20):
        v = rng.standard_normal(3) * 10 ** rng.uniform(-1, 1)
        D = 10 ** rng.uniform(-1.5, 1.5, 3)
        out = O.proj_exp_scaled(v, D)
        ref = mp_exp_reference(v, D)
        np.testing.assert_allclose(out, ref, rtol=1e-9, atol=1e-9 * (1 + np.linalg.norm(v)))


def test_exp_moreau_certificate_all_cases():
    rng = np.random.default_rng(5)
    for _ in range(20000):
        v = rng.standard_normal(3) * 10 ** rng.uniform(-2, 2)
        D = 10 ** rng.uniform(-2, 2, 3)
        p = O.proj_exp_scaled(v, D)
        if not all(exp_cert(v, p, D)):
            # the inequality form of the certificate is ill-conditioned when the
            # dual part's (r, s) are tiny; there, match the 60-digit reference.
            ref = mp_exp_reference(v, D)
            assert np.abs(p - ref).max() <= 1e-13 * (1 + np.linalg.norm(v)), (v, D, p, ref)
    assert O.rootfail_count() == 0


def test_dual_exp_certificate():
    """P_{D K*}: p in D K_exp^*, v - p in -(D K*)^* = -D^-1 K_exp, orthogonal."""
    rng = np.random.default_rng(6)
    for _ in range(5000):
        v = rng.standard_normal(3) * 10 ** rng.uniform(-2, 2)
        D = 10 ** rng.uniform(-2, 2, 3)
        p = O.proj_dual_exp_scaled(v, D)
        sc = 1 + np.linalg.norm(v)
        ok = (O.in_exp_dual(p / D, 1e-9 * sc * (1 + np.max(1 / D)))
              and O.in_exp(-(v - p) * D, 1e-9 * sc * (1 + np.max(D)))
              and abs(p @ (v - p)) <= 1e-9 * sc ** 2)
        if not ok:   # Moreau: P_{DK*}(v) = v + P_{D^-1 K}(-v)
            ref = v + mp_exp_reference(-v, 1.0 / D)
            assert np.abs(p - ref).max() <= 1e-13 * sc, (v, D, p, ref)


def test_exp_membership_examples():
    assert O.in_exp([0, 0, 1])
    assert O.in_exp_dual([-1, 0, math.exp(-1) * (1 + 1e-6)])
    assert not O.in_exp_dual([-1, 0, math.exp(-1) * (1 - 1e-6)])


def test_projection_laws_idempotent_nonexpansive():
    """SPEC.md:227-228 (acceptance 4)."""
    rng = np.random.default_rng(7)
    for _ in range(2000):
        D = 10 ** rng.uniform(-1, 1, 3)
        a, b = rng.standard_normal(3) * 3, rng.standard_normal(3) * 3
        for f in (O.proj_exp_scaled, O.proj_dual_exp_scaled):
            pa, pb = f(a, D), f(b, D)
            np.testing.assert_allclose(f(pa, D), pa, atol=1e-10 * (1 + np.linalg.norm(a)))
            assert np.linalg.norm(pa - pb) <= np.linalg.norm(a - b) * (1 + 1e-10) + 1e-12
        d = int(rng.integers(3, 7))
        Ds = 10 ** rng.uniform(-1, 1, d)
        a, b = rng.standard_normal(d), rng.standard_normal(d)
        pa, pb = O.proj_soc_scaled(a, Ds), O.proj_soc_scaled(b, Ds)
        np.testing.assert_allclose(O.proj_soc_scaled(pa, Ds), pa, atol=1e-10)
        assert np.linalg.norm(pa - pb) <= np.linalg.norm(a - b) * (1 + 1e-10) + 1e-12


# ------------------------------------------------------------------ Alg. 1 scalar rules
def test_scalar_rules_spec_examples():
    for e in G["primal_weight"]:
        assert abs(O.primal_weight(e["dx"], e["dy"], e["omega"]) - e["out"]) <= 1e-15, e["cite"]
    for e in G["restart"]:
        assert O.restart_rule(e["e"], e["e_anchor"], -1.0, e["k"], e["total"]) == e["out"], e["cite"]
    for e in G["halpern"]:
        assert O.halpern_coef(e["k"]) == (e["a"], e["b"])
    assert O.ls_bound(1.25, -0.5) == 1.25
    assert O.ls_bound(3.0, 0.0) == math.inf
    # necessary decay + stall
    assert O.restart_rule(0.7, 1.0, 0.6, 1, 100)
    assert not O.restart_rule(0.7, 1.0, 0.75, 1, 100)
    assert not O.restart_rule(0.9, 1.0, 0.6, 1, 100)


def _tiny(G_, c, h, l, u, rk, rdim, pk=(), pdim=()):
    from instances import csr_from_coo
    A = np.asarray(G_, float)
    r, cc = np.nonzero(A)
    m, n = A.shape
    ptr, col, val = csr_from_coo(m, n, r, cc, A[r, cc])
    return ConicProgram(m=m, n=n, n1=len(l), row_ptr=ptr, col_idx=col, vals=val,
                        c=np.asarray(c, float), h=np.asarray(h, float), l=np.asarray(l, float),
                        u=np.asarray(u, float), pk=np.array(pk, np.int32), pdim=np.array(pdim, np.int64),
                        rk=np.array(rk, np.int32), rdim=np.array(rdim, np.int64))


def test_one_pdhg_spec349():
    e = G["one_pdhg"][0]
    p = _tiny(e["G"], e["c"], e["h"], e["l"], e["u"], [NONNEG], [1])
    S = O.OracleSolver(p, vanilla_pdhg=1, eta0=0.5)
    S.iterate(1)
    x, y = S.get_iterate(0)
    assert x[0] == 0.0 and y[0] == 0.0


def test_line_search_and_halpern_spec358():
    e = G["line_search"][0]
    p = _tiny(e["G"], [0.0], [0.0], [-np.inf], [np.inf], [ZERO], [1])
    S = O.OracleSolver(p, ruiz_iters=0, pock_chambolle=0, eta0=0.5, omega0=1.0)
    S.set_iterate([1.0], [1.0])
    S.iterate(1)
    xh, yh = S.get_iterate(1)
    assert xh[0] == e["xhat"] and yh[0] == e["yhat"]
    assert list(S.trace()) == [1]
    sc = S.scalars()
    assert sc["eta"] == min(1.05 * 0.5, e["bound"])
    # Halpern with beta = 1, k = 0: 1/2 (2 zh - z) + 1/2 z0
    x, y = S.get_iterate(0)
    assert x[0] == 0.5 * (2 * 1.5 - 1.0) + 0.5 * 1.0 and y[0] == 0.5 * (0.0 - 1.0) + 0.5 * 1.0
    # beta = 0: midpoint with the anchor
    S = O.OracleSolver(p, ruiz_iters=0, pock_chambolle=0, eta0=0.5, omega0=1.0, beta_max=0.0)
    S.set_iterate([1.0], [1.0])
    S.iterate(1)
    x, y = S.get_iterate(0)
    assert x[0] == 0.5 * 1.5 + 0.5 and y[0] == 0.5 * 0.0 + 0.5
    # shrink path: eta far above the bound is halved until accepted
    p = gen_mixed(60, 10, 20, seed=3)
    S = O.OracleSolver(p, ruiz_iters=0, pock_chambolle=0, eta0=100.0, omega0=1.0)
    z0x, z0y = S.get_iterate(0)
    S.iterate(1)
    tr = list(S.trace())
    assert tr[-1] == 1 and tr.count(0) >= 1
    xh, yh = S.get_iterate(1)
    eta_acc = 100.0 * 0.5 ** tr.count(0)
    dx, dy = xh - z0x, yh - z0y
    A = p.dense()
    assert eta_acc <= (dx @ dx + dy @ dy) / (2 * abs(dy @ (A @ dx)))   # accepted pair satisfies the test


def test_ruiz_spec278():
    e = G["ruiz"][0]
    p = _tiny(e["A"], [0.0, 0.0], [0.0, 0.0], [-np.inf] * 2, [np.inf] * 2, [ZERO], [2])
    r, q = O.ruiz(p, e["iters"], 0)
    np.testing.assert_allclose(r, e["r"], rtol=1e-15)
    np.testing.assert_allclose(q, e["q"], rtol=1e-15)
    r, q = O.ruiz(p, 0, 0)
    assert np.all(r == 1) and np.all(q == 1)          # SPEC.md:279 no-op


def test_ruiz_equilibrates():
    """Ruiz converges to unit row/column inf-norms (the fixed point of SPEC.md:274)."""
    p = gen_mixed(60, 20, 30, seed=3, scale_spread=2.0)
    r, q = O.ruiz(p, 40, 0)
    K = p.dense() / r[:, None] / q[None, :]
    rm = np.abs(K).max(axis=1)
    cm = np.abs(K).max(axis=0)
    assert np.all(np.abs(rm[rm > 0] - 1) < 1e-3) and np.all(np.abs(cm[cm > 0] - 1) < 1e-3)


# ------------------------------------------------------------------ Eq. 9 and the whole solver
@pytest.mark.parametrize("seed", range(3))
def test_kkt_zero_at_planted_optimum(seed):
    p = gen_mixed(120, 30, 60, seed=seed)
    S = O.OracleSolver(p)
    k = S.kkt_point(p.x_star, p.y_star)
    assert k["err_p"] < 1e-12 and k["err_d"] < 1e-12 and k["err_gap"] < 1e-12
    assert abs(k["pobj"] - p.obj_star) <= 1e-12 * (1 + abs(p.obj_star))


def test_kkt_perturbation_hand_formula():
    """x* + delta on a Zero-row instance: err_p numerator = max_i |G_ij| delta (Eq. 9)."""
    p = _tiny([[1.0, 2.0], [0.0, 3.0]], [1.0, 1.0], [1.0, 3.0], [-np.inf] * 2, [np.inf] * 2,
              [ZERO], [2])
    S = O.OracleSolver(p)
    xs = np.array([-1.0, 1.0])            # G x = h
    ys = np.linalg.solve(np.array([[1.0, 0.0], [2.0, 3.0]]), [1.0, 1.0])   # G^T y = c
    k = S.kkt_point(xs, ys)
    assert max(k["err_p"], k["err_d"], k["err_gap"]) < 1e-14
    d = 1e-3
    k = S.kkt_point(xs + [0.0, d], ys)
    Gx = np.array([-1 + 2 * (1 + d), 3 * (1 + d)])
    assert abs(k["err_p"] - (3 * d) / (1 + max(3.0, np.abs(Gx).max(), 0.0))) < 1e-15


@pytest.mark.parametrize("seed", range(3))
def test_pdhg_fixed_point_at_planted_saddle(seed):
    """SPEC acceptance 5: one Eq. 5 step from a saddle point returns it."""
    p = gen_mixed(150, 30, 60, seed=10 + seed)
    S = O.OracleSolver(p, vanilla_pdhg=1, eta0=0.05)
    S.set_iterate(p.x_star, p.y_star)
    S.iterate(1)
    x, y = S.get_iterate(0)
    assert np.max(np.abs(x - p.x_star)) <= 1e-10 * (1 + np.abs(p.x_star).max())
    assert np.max(np.abs(y - p.y_star)) <= 1e-10 * (1 + np.abs(p.y_star).max())


def test_solve_tiny_lp_and_soc():
    p = _tiny([[1.0]], [1.0], [-5.0], [0.0], [np.inf], [NONNEG], [1])
    r = O.OracleSolver(p, tol=1e-8).solve()
    assert r.status == 0 and abs(r.kkt.pobj) < 1e-7
    # min t s.t. (t, x) in SOC, x = (1, 2)  ->  t* = sqrt 5
    p = _tiny([[0.0, 1.0, 0.0], [0.0, 0.0, 1.0]], [1.0, 0.0, 0.0], [1.0, 2.0], [], [],
              [ZERO], [2], [SOC], [3])
    r = O.OracleSolver(p, tol=1e-9).solve()
    assert r.status == 0 and abs(r.kkt.pobj - math.sqrt(5)) < 1e-7


@pytest.mark.parametrize("seed", range(3))
def test_solve_planted_mixed_objective(seed):
    p = gen_mixed(200, 40, 80, seed=20 + seed)
    r = O.OracleSolver(p, tol=1e-8, max_iters=400000).solve()
    assert r.status == 0
    assert abs(r.kkt.pobj - p.obj_star) <= 1e-6 * (1 + abs(p.obj_star))


def test_solve_lasso_vs_fista():
    """SPEC acceptance 6 / SPEC.md:554: objective vs an independent FISTA oracle."""
    p = gen_lasso(100, 50, 1.0, seed=0, dense=True)
    r = O.OracleSolver(p, tol=1e-7).solve()
    assert r.status == 0
    arow, acol, aval, m, nf = p.lasso_A
    A = np.zeros((m, nf))
    A[arow, acol] = aval
    b, lam = p.lasso_b, p.lasso_lam
    L = 2 * np.linalg.norm(A, 2) ** 2
    x = np.zeros(nf)
    z, tk = x.copy(), 1.0
    for _ in range(20000):
        g = 2 * A.T @ (A @ z - b)
        xn = z - g / L
        xn = np.sign(xn) * np.maximum(np.abs(xn) - lam / L, 0)
        tn = (1 + math.sqrt(1 + 4 * tk * tk)) / 2
        z = xn + (tk - 1) / tn * (xn - x)
        x, tk = xn, tn
    f = np.sum((A @ x - b) ** 2) + lam * np.abs(x).sum()
    assert abs(r.kkt.pobj - f) <= 1e-5 * abs(f)


def test_solve_fisher_vs_proportional_response():
    """SPEC acceptance 7: Fisher equilibrium objective vs proportional-response
    dynamics (an independent market algorithm) on the original problem Eq. arrow_market."""
    p = gen_fisher(10, 20, seed=0)
    r = O.OracleSolver(p, tol=1e-8, max_iters=400000).solve()
    assert r.status == 0
    urow, ucol, uval, w, mb, ng = p.fisher
    U = np.zeros((mb, ng))
    U[urow, ucol] = uval
    bsup = np.full(ng, 0.25)
    bids = np.outer(w, np.ones(ng)) * (U > 0) / np.maximum((U > 0).sum(1, keepdims=True), 1)
    for _ in range(200000):
        price = bids.sum(0)
        X = bids / price * bsup
        util = (U * X).sum(1)
        bids = w[:, None] * U * X / util[:, None]
    obj = -np.sum(w * np.log((U * X).sum(1)))
    assert abs(r.kkt.pobj - obj) <= 1e-5 * (1 + abs(obj))


def test_solve_mpo_feasible():
    """SPEC acceptance 8: returned portfolio satisfies the MPO constraints."""
    p = gen_mpo(3, 20, seed=0)
    S = O.OracleSolver(p, tol=1e-7, max_iters=400000)
    r = S.solve()
    assert r.status == 0
    x, y = S.get_iterate(3, 1)
    G = p.dense()
    s = G @ x - p.h
    off = 0
    for k, d in zip(p.rk, p.rdim):
        blk = s[off:off + d]
        if k == ZERO:
            assert np.abs(blk).max() < 1e-5
        elif k == NONNEG:
            assert blk.min() > -1e-5
        elif k == SOC:
            assert np.linalg.norm(blk[1:]) - blk[0] < 1e-5
        off += d
    assert x[p.l > -np.inf].min() >= -1e-12


def test_determinism():
    """SPEC acceptance 12: bit-identical runs."""
    p = gen_mixed(100, 20, 40, seed=4)
    a = O.OracleSolver(p)
    b = O.OracleSolver(p)
    a.iterate(300)
    b.iterate(300)
    xa, ya = a.get_iterate(0)
    xb, yb = b.get_iterate(0)
    assert np.array_equal(xa, xb) and np.array_equal(ya, yb)


def test_exp_nearest_candidate_when_distances_tie_to_the_ulp():
    """Reading P7.  A point far below the cone (t0 << 0) next to the s = 0 face:
    the root point and the t-raised point are at squared distances that agree
    to one ulp of t0^2, yet differ in r, s at 1e-6 relative.  "Nearest" is
    decided by <p - q, p + q - 2 v0>.  The first case is a primal exp block of
    the mixed cfg 5 bench instance (seed 0, block 33696, first trial from the
    seeded random point of tests/test_full_size.py); the rest are random
    points of the same shape.  All are checked against the 60-digit
    reference."""
    cases = [(np.array([-53.848289446000855, 5.317878561776792, -533.0367249585]),
              np.array([25.540130991958577, 59.559580156562696, 414.0600653716415]))]
    rng = np.random.default_rng(11)
    for _ in range(12):
        D = 10 ** rng.uniform(-1, 2.5, 3)
        cases.append((np.array([-rng.uniform(5, 80), rng.uniform(0.5, 8), -rng.uniform(100, 5000)]), D))
    for v, D in cases:
        ref = mp_exp_reference(v, D)
        got = O.proj_exp_scaled(v, D)
        assert np.max(np.abs(got - ref)) <= 1e-13 * (1 + np.max(np.abs(v))), (v, D, got, ref)
