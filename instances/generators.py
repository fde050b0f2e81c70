"""Seeded synthetic instance generators (shared by the oracle and the CUDA path).

This module builds INPUT DATA ONLY: it contains none of the method's
arithmetic (no projections, no PDHG, no scaling).  Every random number comes
from ``numpy.random.Generator(Philox(seed))``.  Recipes:

* Lasso SOCP   — PAPER.md:1625-1664 (App. B.2); rotated-SOC reading A22.
* Fisher market — PAPER.md:1577-1623 (App. B.1, Eq. pro:fisher_cp).
* MPO SOCP     — PAPER.md:1668-1706 (App. B.3, Eq. pro:MPO_SOCP); synthetic
                 covariance per SURVEY §8(c) A24.
* Mixed planted — SURVEY §8(d) cfg 5: all cone kinds with a planted KKT pair
                 (x*, y*) so that c^T x* is the exact optimum.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

from .program import (ConicProgram, csr_from_coo, ZERO, NONNEG, SOC, RSOC, EXP,
                      DUAL_EXP)

INF = np.inf


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(seed))


def bernoulli_positions(rng: np.random.Generator, total: int, p: float) -> np.ndarray:
    """Sorted positions in [0, total) of an i.i.d. Bernoulli(p) mask.

    Drawn with geometric gaps, so every position is independently selected with
    probability p (row counts are exactly Binomial) and the result is sorted and
    duplicate-free.
    """
    if p >= 1.0:
        return np.arange(total, dtype=np.int64)
    out = []
    pos = -1
    while True:
        need = int((total - pos) * p * 1.02) + 1024
        gaps = rng.geometric(p, size=need).astype(np.int64)
        idx = pos + np.cumsum(gaps)
        cut = np.searchsorted(idx, total)
        out.append(idx[:cut])
        if cut < need:
            break
        pos = int(idx[-1])
    return np.concatenate(out) if out else np.zeros(0, np.int64)


# --------------------------------------------------------------------------
# Lasso as SOCP (variables ordered (x+, x-, w, r, y), A22)
# --------------------------------------------------------------------------
def gen_lasso(m: int, nfeat: int, density: float, seed: int = 0,
              dense: bool = False, balance: bool = True) -> ConicProgram:
    """min ||A x - b||^2 + lam ||x||_1 as the conic program of PAPER.md:1641-1659.

    Variables x = (x+ [nfeat], x- [nfeat] | w, r, y [m]); n1 = 2 nfeat with
    bounds [0, inf); one primal RSOC block (w, r, y): ||y||^2 <= 2 w r
    (PAPER.md:1657 is exactly the rotated SOC, reading A22).  Rows: w = 1;
    y - A x+ + A x- = -b (all Zero cones).  Data recipe PAPER.md:1663-1664:
    A_ij ~ U[0,1] at the given density, x~ ~ N(0,1) with half zeroed,
    b = A x~ + 1e-6, lam = ||A^T b||_inf.

    balance (reading P9): the RSOC's leading pair is stored as
    (w', r') = (S w, r / S), S = max(1, ||b|| / sqrt(2)) -- the square root
    of r at x = 0, so that w' = S and r' = r / S are of one size -- an
    automorphism of the rotated cone (2 w' r' = 2 w r), so the row w = 1
    reads w' / S = 1 and r' costs 2 S.  Same problem, same optimal
    value; a solution maps back by w = w' / S, r = S r' (y unchanged:
    `prog.to_literal(x)`).  balance=False gives the literal form, on which
    PDCS with the SPEC's heuristics stalls (P8).
    """
    rng = _rng(seed)
    if dense:
        arow = np.repeat(np.arange(m, dtype=np.int64), nfeat)
        acol = np.tile(np.arange(nfeat, dtype=np.int64), m)
    else:
        pos = bernoulli_positions(rng, m * nfeat, density)
        arow, acol = pos // nfeat, pos % nfeat
        del pos
    aval = rng.uniform(0.0, 1.0, size=arow.shape[0])
    xt = rng.standard_normal(nfeat)
    xt[rng.permutation(nfeat)[: nfeat // 2]] = 0.0
    b = np.bincount(arow, weights=aval * xt[acol], minlength=m) + 1e-6
    lam = float(np.max(np.abs(np.bincount(acol, weights=aval * b[arow], minlength=nfeat))))

    n1 = 2 * nfeat
    iw, ir, iy = n1, n1 + 1, n1 + 2
    n = n1 + 2 + m
    mrows = m + 1
    k = np.bincount(arow, minlength=m).astype(np.int64)        # nnz per A row
    row_ptr = np.zeros(mrows + 1, dtype=np.int64)
    row_ptr[1] = 1
    row_ptr[2:] = 1 + np.cumsum(2 * k + 1)
    nnz = int(row_ptr[-1])
    col = np.empty(nnz, dtype=np.int32)
    val = np.empty(nnz, dtype=np.float64)
    S = max(1.0, (float(b @ b) / 2.0) ** 0.5) if balance else 1.0
    col[0], val[0] = iw, 1.0 / S
    astart = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(k, out=astart[1:])
    within = np.arange(arow.shape[0], dtype=np.int64) - astart[arow]
    base = row_ptr[1:-1][arow]                                  # start of K row arow+1
    col[base + within] = acol
    val[base + within] = -aval
    col[base + k[arow] + within] = nfeat + acol
    val[base + k[arow] + within] = aval
    yslot = row_ptr[2:] - 1
    col[yslot] = iy + np.arange(m)
    val[yslot] = 1.0
    h = np.empty(mrows)
    h[0] = 1.0
    h[1:] = -b
    c = np.zeros(n)
    c[:n1] = lam
    c[ir] = 2.0 * S
    prog = ConicProgram(
        m=mrows, n=n, n1=n1, row_ptr=row_ptr, col_idx=col, vals=val, c=c, h=h,
        l=np.zeros(n1), u=np.full(n1, INF),
        pk=np.array([RSOC], np.int32), pdim=np.array([m + 2], np.int64),
        rk=np.array([ZERO], np.int32), rdim=np.array([mrows], np.int64),
        name=f"lasso_{m}x{nfeat}_d{density:g}_s{seed}" + ("" if balance else "_literal"))
    prog.lasso_A = (arow, acol, aval, m, nfeat)   # original data for ISTA pins
    prog.lasso_b = b
    prog.lasso_lam = lam
    prog.lasso_S = S

    def to_literal(x, S=S, iw=iw, ir=ir):
        """A point of this instance as a point of the literal form (balance=False)."""
        x = np.array(x, dtype=np.float64, copy=True)
        x[iw] /= S
        x[ir] *= S
        return x
    prog.to_literal = to_literal

    def literal(prog=prog, S=S, iw=iw, ir=ir):
        """The literal form (balance=False) of this instance, sharing A and b."""
        if S == 1.0:
            return prog
        v = prog.vals.copy()
        v[0] = 1.0                                    # row w = 1, col iw
        cc = prog.c.copy()
        cc[ir] = 2.0
        return ConicProgram(m=prog.m, n=prog.n, n1=prog.n1, row_ptr=prog.row_ptr, col_idx=prog.col_idx, vals=v,
                            c=cc, h=prog.h, l=prog.l, u=prog.u, pk=prog.pk, pdim=prog.pdim, rk=prog.rk,
                            rdim=prog.rdim, name=prog.name + "_literal")
    prog.literal = literal
    return prog


# --------------------------------------------------------------------------
# Fisher market (Eq. pro:fisher_cp)
# --------------------------------------------------------------------------
def gen_fisher(mbuy: int, ngood: int, density: float = 0.2, seed: int = 0) -> ConicProgram:
    """Fisher market equilibrium as the exp-cone program of PAPER.md:1618.

    Variables (X [mbuy*ngood] buyer-major as printed, (p_i, t_i) pairs),
    X >= 0, p, t free (n1 = n, n2 = 0).  Rows: ngood supply equalities
    sum_i X_ij = b_j; mbuy t-definitions U_i X_i - t_i = 0; mbuy row blocks
    (p_i, 0, t_i) - (0, -1, 0) in K_exp.  U_ij ~ U[0,1] at
    density 0.2, repaired so every row/column has a nonzero;
    w_i ~ U[0,1]; b_j = 0.25.
    """
    rng = _rng(seed)
    pos = bernoulli_positions(rng, mbuy * ngood, density)
    urow, ucol = pos // ngood, pos % ngood
    uval = rng.uniform(0.0, 1.0, size=pos.shape[0])
    w = rng.uniform(0.0, 1.0, size=mbuy)
    # repair empty rows / columns (one uniformly chosen entry each)
    rowcnt = np.bincount(urow, minlength=mbuy)
    add_r = np.nonzero(rowcnt == 0)[0]
    colcnt = np.bincount(ucol, minlength=ngood)
    add_c = np.nonzero(colcnt == 0)[0]
    if add_r.size or add_c.size:
        er = np.concatenate([add_r, rng.integers(0, mbuy, add_c.size)])
        ec = np.concatenate([rng.integers(0, ngood, add_r.size), add_c])
        ev = rng.uniform(0.0, 1.0, size=er.size)
        key = np.concatenate([urow * ngood + ucol, er * ngood + ec])
        allv = np.concatenate([uval, ev])
        key, first = np.unique(key, return_index=True)
        urow, ucol, uval = key // ngood, key % ngood, allv[first]
    nX = mbuy * ngood
    n = nX + 2 * mbuy
    mrows = ngood + mbuy + 3 * mbuy
    # supply rows j: all X[i, j] (cols i*ngood + j), value 1
    sup_rows = np.repeat(np.arange(ngood, dtype=np.int64), mbuy)
    sup_cols = (np.arange(mbuy, dtype=np.int64)[None, :] * ngood
                + np.arange(ngood, dtype=np.int64)[:, None]).ravel()
    sup_vals = np.ones(nX)
    # t rows
    t_rows = np.concatenate([ngood + urow, ngood + np.arange(mbuy)])
    t_cols = np.concatenate([urow * ngood + ucol, nX + 2 * np.arange(mbuy) + 1])
    t_vals = np.concatenate([uval, -np.ones(mbuy)])
    # exp rows: (p_i, -, t_i)
    base = ngood + mbuy + 3 * np.arange(mbuy, dtype=np.int64)
    e_rows = np.concatenate([base, base + 2])
    e_cols = np.concatenate([nX + 2 * np.arange(mbuy), nX + 2 * np.arange(mbuy) + 1])
    e_vals = np.ones(2 * mbuy)
    row_ptr, col, val = csr_from_coo(
        mrows, n, np.concatenate([sup_rows, t_rows, e_rows]),
        np.concatenate([sup_cols, t_cols, e_cols]),
        np.concatenate([sup_vals, t_vals, e_vals]))
    h = np.zeros(mrows)
    h[:ngood] = 0.25
    h[base + 1] = -1.0
    c = np.zeros(n)
    c[nX + 2 * np.arange(mbuy)] = -w
    l = np.full(n, -INF)
    l[:nX] = 0.0
    rk = np.array([ZERO] + [EXP] * mbuy, np.int32)
    rdim = np.array([ngood + mbuy] + [3] * mbuy, np.int64)
    prog = ConicProgram(
        m=mrows, n=n, n1=n, row_ptr=row_ptr, col_idx=col, vals=val, c=c, h=h,
        l=l, u=np.full(n, INF), pk=np.zeros(0, np.int32), pdim=np.zeros(0, np.int64),
        rk=rk, rdim=rdim, name=f"fisher_{mbuy}x{ngood}_s{seed}")
    prog.fisher = (urow, ucol, uval, w, mbuy, ngood)
    return prog


# --------------------------------------------------------------------------
# Multi-period portfolio optimisation (Eq. pro:MPO_SOCP)
# --------------------------------------------------------------------------
def gen_mpo(T: int, nasset: int, seed: int = 0, gamma2: float = 0.05,
            gamma3: float = 0.05, nfactor: int = 5) -> ConicProgram:
    """Constraint-form MPO SOCP of PAPER.md:1694-1705 with synthetic data.

    Per period tau (w = w_{tau+1} in R^{n+1}, u = u_tau in R^n):
      budget  1^T (w - w_tau) = 0                       (Zero; w_0 = w_{1/n})
      market  (w^m)^T Sigma w_[n] = 0                   (Zero)
      |.|     u_i - (w_i - wb_i) >= 0, u_i + (w_i - wb_i) >= 0   (NonNeg)
      u-sum   gamma3 - sum_i Sigma^{1/2}_ii u_i >= 0     (NonNeg)
      risk    (gamma1, Sigma^{1/2}(w - wb)_[n]) in SOC(n+1)
      trade   gamma2 +- (w - w_tau)_i >= 0  for i in [n+1] (NonNeg)
    w >= 0 as bounds, u free.  Synthetic data per SURVEY A24: Sigma = F F^T +
    diag(U[1e-4,4e-4]), F ~ N(0, 0.01^2) (n x 5), perturbed per period;
    r^ ~ U[-0.01, 0.03]; w_b = all cash; gamma1 = ||Sigma^{1/2}(w_{1/n} - wb)||.
    The market portfolio w^m is chosen with (w^m)^T Sigma w_{1/n} = 0.
    """
    rng = _rng(seed)
    n = nasset
    nw = n + 1
    nvar_per = nw + n
    nv = T * nvar_per
    w0 = np.full(nw, 1.0 / nw)          # w_{1/n} incl. cash
    wb = np.zeros(nw)
    wb[n] = 1.0                          # all-cash benchmark (A24)
    F0 = rng.normal(0.0, 0.01, size=(n, nfactor))
    D0 = rng.uniform(1e-4, 4e-4, size=n)
    rows, cols, vals = [], [], []
    h_parts, rk_list, rdim_list = [], [], []
    row = 0
    c = np.zeros(nv)

    def add(rr, cc, vv):
        rows.append(np.asarray(rr, np.int64))
        cols.append(np.asarray(cc, np.int64))
        vals.append(np.asarray(vv, np.float64))

    for tau in range(T):
        F = F0 * (1.0 + 0.05 * rng.standard_normal(F0.shape))
        Dg = D0 * (1.0 + 0.05 * rng.uniform(-1.0, 1.0, size=n))
        Sigma = F @ F.T + np.diag(Dg)
        evals, evecs = np.linalg.eigh(Sigma)
        S12 = (evecs * np.sqrt(np.maximum(evals, 0.0))) @ evecs.T
        rhat = rng.uniform(-0.01, 0.03, size=nw)
        rhat[n] = 0.0
        gamma1 = float(np.linalg.norm(S12 @ (w0 - wb)[:n]))
        # market portfolio orthogonal (in Sigma) to w_{1/n}
        g = rng.uniform(0.0, 1.0, size=n)
        s0 = Sigma @ w0[:n]
        wm = g - (g @ s0) / (s0 @ s0) * s0
        iw = tau * nvar_per            # w_{tau+1} block
        iu = iw + nw                   # u_tau block
        c[iw:iw + nw] = -rhat          # max r^T w -> min -r^T w
        # --- equality rows (Zero block of 2 rows)
        # budget: 1^T w_{tau+1} - 1^T w_tau = 0
        if tau == 0:
            add(np.full(nw, row), iw + np.arange(nw), np.ones(nw))
            h_parts.append([1.0])
        else:
            ip = iw - nvar_per
            add(np.full(2 * nw, row), np.concatenate([ip + np.arange(nw), iw + np.arange(nw)]),
                np.concatenate([-np.ones(nw), np.ones(nw)]))
            h_parts.append([0.0])
        row += 1
        mrow = Sigma @ wm
        add(np.full(n, row), iw + np.arange(n), mrow)
        h_parts.append([0.0])
        row += 1
        rk_list.append(ZERO)
        rdim_list.append(2)
        # --- NonNeg block: 2n abs rows + 1 usum row + 2(n+1) trade rows
        r0 = row
        ar = r0 + np.arange(n)
        add(np.concatenate([ar, ar]), np.concatenate([iu + np.arange(n), iw + np.arange(n)]),
            np.concatenate([np.ones(n), -np.ones(n)]))
        h_parts.append(-wb[:n])            # u - w + wb >= 0  ->  G x - h, h = -wb
        ar2 = r0 + n + np.arange(n)
        add(np.concatenate([ar2, ar2]), np.concatenate([iu + np.arange(n), iw + np.arange(n)]),
            np.concatenate([np.ones(n), np.ones(n)]))
        h_parts.append(wb[:n])             # u + w - wb >= 0
        ru = r0 + 2 * n
        add(np.full(n, ru), iu + np.arange(n), -np.diag(S12).copy())
        h_parts.append([-gamma3])          # -sum diag u + gamma3 >= 0
        rt = ru + 1 + np.arange(nw)
        if tau == 0:
            add(rt, iw + np.arange(nw), np.ones(nw))
            h_parts.append(w0 - gamma2)    # w - w0 + g2 >= 0
            rt2 = rt + nw
            add(rt2, iw + np.arange(nw), -np.ones(nw))
            h_parts.append(-w0 - gamma2)   # -(w - w0) + g2 >= 0
        else:
            ip = iw - nvar_per
            add(np.concatenate([rt, rt]), np.concatenate([iw + np.arange(nw), ip + np.arange(nw)]),
                np.concatenate([np.ones(nw), -np.ones(nw)]))
            h_parts.append(np.full(nw, -gamma2))
            rt2 = rt + nw
            add(np.concatenate([rt2, rt2]), np.concatenate([iw + np.arange(nw), ip + np.arange(nw)]),
                np.concatenate([-np.ones(nw), np.ones(nw)]))
            h_parts.append(np.full(nw, -gamma2))
        nn = 2 * n + 1 + 2 * nw
        row = r0 + nn
        rk_list.append(NONNEG)
        rdim_list.append(nn)
        # --- SOC block (gamma1, S12 (w - wb)_[n])
        rs = row
        h_parts.append([-gamma1])          # head row: 0*x - (-gamma1)
        rr = rs + 1 + np.repeat(np.arange(n), n)
        cc = iw + np.tile(np.arange(n), n)
        add(rr, cc, S12.ravel())
        h_parts.append(S12 @ wb[:n])
        rk_list.append(SOC)
        rdim_list.append(n + 1)
        row = rs + n + 1
    mrows = row
    row_ptr, col, val = csr_from_coo(mrows, nv, np.concatenate(rows),
                                     np.concatenate(cols), np.concatenate(vals))
    h = np.concatenate([np.atleast_1d(np.asarray(p, np.float64)) for p in h_parts])
    assert h.shape[0] == mrows
    # bounds: w >= 0, u free; all variables are box variables (n2 = 0)
    l = np.full(nv, -INF)
    for tau in range(T):
        l[tau * nvar_per: tau * nvar_per + nw] = 0.0
    prog = ConicProgram(
        m=mrows, n=nv, n1=nv, row_ptr=row_ptr, col_idx=col, vals=val, c=c, h=h,
        l=l, u=np.full(nv, INF), pk=np.zeros(0, np.int32), pdim=np.zeros(0, np.int64),
        rk=np.array(rk_list, np.int32), rdim=np.array(rdim_list, np.int64),
        name=f"mpo_T{T}_n{n}_s{seed}")
    return prog


# --------------------------------------------------------------------------
# Mixed-cone planted instance (SURVEY §8(d) cfg 5)
# --------------------------------------------------------------------------
def _cone_pair(rng, kind: int, d: int):
    """A complementary pair (s in K, y in K^*, <s, y> = 0) for one block."""
    if kind == ZERO:
        return np.zeros(d), rng.standard_normal(d)
    if kind == NONNEG:
        s = rng.uniform(0.0, 1.0, d)
        y = rng.uniform(0.0, 1.0, d)
        pick = rng.uniform(size=d) < 0.5
        s[pick] = 0.0
        y[~pick] = 0.0
        return s, y
    if kind in (SOC, RSOC):
        v = rng.standard_normal(d - 1)
        nv = np.linalg.norm(v)
        a, b = rng.uniform(0.0, 1.0, 2)
        mode = rng.integers(0, 3)
        if mode == 1:
            a = 0.0
        elif mode == 2:
            b = 0.0
        s = a * np.concatenate([[nv], v])
        y = b * np.concatenate([[nv], -v])
        if kind == RSOC:   # R = [[1,1],[1,-1]]/sqrt2 maps SOC <-> RSOC, R = R^T = R^-1
            for z in (s, y):
                t0, t1 = z[0], z[1]
                z[0], z[1] = (t0 + t1) / math.sqrt(2.0), (t0 - t1) / math.sqrt(2.0)
        return s, y
    if kind in (EXP, DUAL_EXP):
        rho = rng.uniform(-2.0, 2.0)
        a, b = rng.uniform(0.1, 1.0, 2)
        mode = rng.integers(0, 4)
        if mode == 1:
            a = 0.0
        elif mode == 2:
            b = 0.0
        pe = a * np.array([rho, 1.0, math.exp(rho)])            # in K_exp
        de = b * np.array([-1.0, rho - 1.0, math.exp(-rho)])    # in K_exp^*
        return (pe, de) if kind == EXP else (de, pe)
    raise ValueError(kind)


def _draw_blocks(rng, total: int, mix, soc_dims=(3, 24)):
    kinds, dims = [], []
    rem = total
    names = [k for k, _ in mix]
    probs = np.array([f for _, f in mix], np.float64)
    probs = probs / probs.sum()
    while rem > 0:
        k = int(rng.choice(names, p=probs))
        if k in (EXP, DUAL_EXP):
            d = 3
        elif k in (SOC, RSOC):
            d = int(rng.integers(soc_dims[0], soc_dims[1] + 1))
        else:
            d = int(rng.integers(1, 8))
        if d > rem:
            k, d = NONNEG, rem
        kinds.append(k)
        dims.append(d)
        rem -= d
    return np.array(kinds, np.int32), np.array(dims, np.int64)


def gen_mixed(m: int, n1: int, n2: int, seed: int = 0, row_len=(3, 12),
              soc_dims=(3, 24), scale_spread: float = 1.0,
              row_mix=None, col_mix=None) -> ConicProgram:
    """Mixed-cone instance with a planted KKT pair (SURVEY §8(d) cfg 5).

    G has rows of U{row_len} distinct uniform columns with values
    N(0,1) * 10^{U[-s,s]} * rowfactor * colfactor (s = scale_spread) so that
    rescaling matters.  Row cones / primal cones mix all six kinds.  The pair
    (x*, y*) with h = G x* - s*, c = G^T y* + lam* satisfies Eq. 1-2's KKT
    conditions exactly, so c^T x* is the optimal value.
    """
    rng = _rng(seed)
    n = n1 + n2
    row_mix = row_mix or [(ZERO, .30), (NONNEG, .30), (SOC, .25), (RSOC, .05),
                          (EXP, .075), (DUAL_EXP, .025)]
    col_mix = col_mix or [(ZERO, .01), (NONNEG, .20), (SOC, .40), (RSOC, .15),
                          (EXP, .20), (DUAL_EXP, .04)]
    rk, rdim = _draw_blocks(rng, m, row_mix, soc_dims)
    pk, pdim = _draw_blocks(rng, n2, col_mix, soc_dims) if n2 > 0 else (
        np.zeros(0, np.int32), np.zeros(0, np.int64))
    lens = rng.integers(row_len[0], row_len[1] + 1, size=m)
    lens = np.minimum(lens, n)
    rows = np.repeat(np.arange(m, dtype=np.int64), lens)
    cols = np.concatenate([rng.choice(n, size=L, replace=False) for L in lens]).astype(np.int64)
    rf = 10.0 ** rng.uniform(-scale_spread, scale_spread, size=m)
    cf = 10.0 ** rng.uniform(-scale_spread, scale_spread, size=n)
    vals = rng.standard_normal(rows.shape[0]) * rf[rows] * cf[cols]
    row_ptr, col, val = csr_from_coo(m, n, rows, cols, vals)
    # box part
    btype = rng.integers(0, 4, size=n1)   # 0 free, 1 [l,inf), 2 (-inf,u], 3 [l,u]
    lo = rng.uniform(-1.0, 0.0, n1)
    hi = rng.uniform(0.0, 1.0, n1) + lo + 0.5
    l = np.where((btype == 1) | (btype == 3), lo, -INF)
    u = np.where((btype == 2) | (btype == 3), hi, INF)
    x1 = np.empty(n1)
    lam1 = np.zeros(n1)
    status = rng.integers(0, 3, size=n1)  # 0 interior, 1 at lower, 2 at upper
    for i in range(n1):
        if status[i] == 1 and np.isfinite(l[i]):
            x1[i] = l[i]
            lam1[i] = rng.uniform(0.0, 1.0)
        elif status[i] == 2 and np.isfinite(u[i]):
            x1[i] = u[i]
            lam1[i] = -rng.uniform(0.0, 1.0)
        else:
            fl, fu = np.isfinite(l[i]), np.isfinite(u[i])
            if fl and fu:
                x1[i] = rng.uniform(l[i], u[i])
            elif fl:
                x1[i] = l[i] + rng.uniform(0.0, 1.0)
            elif fu:
                x1[i] = u[i] - rng.uniform(0.0, 1.0)
            else:
                x1[i] = rng.standard_normal()
    x2, lam2 = [], []
    for k, d in zip(pk, pdim):
        xb, lb = _cone_pair(rng, int(k), int(d))
        x2.append(xb)
        lam2.append(lb)
    s_parts, y_parts = [], []
    for k, d in zip(rk, rdim):
        sb, yb = _cone_pair(rng, int(k), int(d))
        s_parts.append(sb)
        y_parts.append(yb)
    x_star = np.concatenate([x1] + x2) if x2 else x1
    y_star = np.concatenate(y_parts)
    s_star = np.concatenate(s_parts)
    lam = np.concatenate([lam1] + lam2) if lam2 else lam1
    Gx = np.bincount(rows_of(row_ptr), weights=val * x_star[col], minlength=m)
    GTy = np.bincount(col, weights=val * y_star[rows_of(row_ptr)], minlength=n)
    h = Gx - s_star
    c = GTy + lam
    prog = ConicProgram(m=m, n=n, n1=n1, row_ptr=row_ptr, col_idx=col, vals=val,
                        c=c, h=h, l=l, u=u, pk=pk, pdim=pdim, rk=rk, rdim=rdim,
                        name=f"mixed_{m}x{n}_s{seed}")
    prog.x_star, prog.y_star = x_star, y_star
    prog.obj_star = float(c @ x_star)
    return prog


def rows_of(row_ptr: np.ndarray) -> np.ndarray:
    m = row_ptr.shape[0] - 1
    return np.repeat(np.arange(m, dtype=np.int64), np.diff(row_ptr))


# --------------------------------------------------------------------------
# Mixed-cone planted instance at scale (SURVEY §8(d) cfg 5), vectorised
# --------------------------------------------------------------------------
def _blocks_of_kind(rng, kind: int, total: int, dims_fn, min_dim: int):
    """Blocks of one kind whose dims sum to exactly `total` (a short last block
    becomes NonNeg)."""
    if total <= 0:
        return np.zeros(0, np.int32), np.zeros(0, np.int64)
    d = dims_fn(max(16, int(2 * total / 3) + 16))
    while d.sum() < total:
        d = np.concatenate([d, dims_fn(max(16, d.shape[0]))])
    cs = np.cumsum(d)
    nb = int(np.searchsorted(cs, total)) + 1
    d = d[:nb].copy()
    d[-1] -= cs[nb - 1] - total
    k = np.full(nb, kind, np.int32)
    if d[-1] < min_dim:
        k[-1] = NONNEG
    return k, d.astype(np.int64)


def _mixed_cones(rng, total: int, shares, giant=()):
    """Cone list over `total` coordinates: kind shares of the coordinates,
    SOC dims log-uniform in [3, 4096] (+ giant SOC blocks), RSOC in [3, 256],
    exp / dual exp 3, Zero / NonNeg runs U{1..64}; blocks in random order."""
    def logu(lo, hi):
        return lambda k: np.floor(np.exp(rng.uniform(math.log(lo), math.log(hi + 1), k))).astype(np.int64)
    dims = {ZERO: lambda k: rng.integers(1, 65, k), NONNEG: lambda k: rng.integers(1, 65, k),
            SOC: logu(3, 4096), RSOC: logu(3, 256), EXP: lambda k: np.full(k, 3), DUAL_EXP: lambda k: np.full(k, 3)}
    mins = {ZERO: 1, NONNEG: 1, SOC: 2, RSOC: 3, EXP: 3, DUAL_EXP: 3}
    kinds, ds = [], []
    used = 0
    for g in giant:
        kinds.append(np.array([SOC], np.int32)); ds.append(np.array([g], np.int64)); used += g
    order = list(shares.items())
    for i, (kind, f) in enumerate(order):
        t = int(round(f * total)) if i < len(order) - 1 else total - used
        if kind == SOC:
            t -= sum(giant)
        t = max(t, 0)
        if kind in (EXP, DUAL_EXP):
            t -= t % 3
        k, d = _blocks_of_kind(rng, kind, t, dims[kind], mins[kind])
        kinds.append(k); ds.append(d); used += int(d.sum())
    k = np.concatenate(kinds); d = np.concatenate(ds)
    if used < total:                      # rounding remainder
        k = np.concatenate([k, [NONNEG]]).astype(np.int32); d = np.concatenate([d, [total - used]])
    p = rng.permutation(k.shape[0])
    return k[p].astype(np.int32), d[p].astype(np.int64)


def _planted_pairs(rng, kinds, dims):
    """Complementary (s in K, y in K*, <s, y> = 0) for every block, vectorised
    per kind (same construction as _cone_pair)."""
    total = int(dims.sum())
    s = np.zeros(total); y = np.zeros(total)
    off = np.concatenate([[0], np.cumsum(dims)[:-1]]).astype(np.int64)
    elem = np.repeat(kinds, dims)
    zr = elem == ZERO
    y[zr] = rng.standard_normal(int(zr.sum()))
    nn = elem == NONNEG
    a = rng.uniform(0.0, 1.0, int(nn.sum())); b = rng.uniform(0.0, 1.0, int(nn.sum()))
    pick = rng.uniform(size=a.shape[0]) < 0.5
    s[nn] = np.where(pick, 0.0, a); y[nn] = np.where(pick, b, 0.0)
    for kind in (SOC, RSOC):
        sel = np.nonzero(kinds == kind)[0]
        if not sel.size:
            continue
        o, d = off[sel], dims[sel]
        idx = np.concatenate([np.arange(oo, oo + dd) for oo, dd in zip(o, d)]) if sel.size < 20000 else \
            np.repeat(o, d) + (np.arange(int(d.sum())) - np.repeat(np.cumsum(d) - d, d))
        v = rng.standard_normal(idx.shape[0])
        head = np.repeat(np.cumsum(d) - d, 1)               # block starts within idx
        v[head] = 0.0
        nv = np.sqrt(np.add.reduceat(v * v, head))
        v[head] = nv
        ab = rng.uniform(0.0, 1.0, (sel.size, 2))
        mode = rng.integers(0, 3, sel.size)
        ab[mode == 1, 0] = 0.0
        ab[mode == 2, 1] = 0.0
        sa = np.repeat(ab[:, 0], d); sb = np.repeat(ab[:, 1], d)
        sv = sa * v
        yv = -sb * v
        yv[head] = sb[head] * nv
        if kind == RSOC:                                    # rotate the leading pair
            for z in (sv, yv):
                t0, t1 = z[head].copy(), z[head + 1].copy()
                z[head] = (t0 + t1) / math.sqrt(2.0)
                z[head + 1] = (t0 - t1) / math.sqrt(2.0)
        s[idx] = sv; y[idx] = yv
    for kind in (EXP, DUAL_EXP):
        sel = np.nonzero(kinds == kind)[0]
        if not sel.size:
            continue
        o = off[sel]
        rho = rng.uniform(-2.0, 2.0, sel.size)
        ab = rng.uniform(0.1, 1.0, (sel.size, 2))
        mode = rng.integers(0, 4, sel.size)
        ab[mode == 1, 0] = 0.0
        ab[mode == 2, 1] = 0.0
        pe = ab[:, :1] * np.stack([rho, np.ones_like(rho), np.exp(rho)], 1)
        de = ab[:, 1:] * np.stack([-np.ones_like(rho), rho - 1.0, np.exp(-rho)], 1)
        if kind == DUAL_EXP:
            pe, de = de, pe
        for j in range(3):
            s[o + j] = pe[:, j]; y[o + j] = de[:, j]
    return s, y


def gen_mixed_large(scale: float = 0.125, seed: int = 0) -> ConicProgram:
    """SURVEY §8(d) cfg 5 at `scale` (1.0: m = 2e7, n = 1e7, nnz ~ 2e9; the
    default 1/8 is one GPU's share of the 8-GPU job).  Rows of U{20..180}
    distinct uniform columns; values N(0,1) 10^U[-2,2] (row) 10^U[-2,2] (col).
    Row cones: 30% Zero, 30% NonNeg, 25% SOC (log-uniform dims in [3, 4096]
    plus 4 blocks of 2.5e5*scale), 5% RSOC ([3, 256]), 7.5% Exp, 2.5% DualExp.
    Columns: 40% box (1/4 each free, [l,inf), (-inf,u], [l,u]), 60% primal
    cones: Zero 1%, NonNeg 20%, SOC 40%, RSOC 15%, Exp 20%, DualExp 4%.
    Planted KKT pair as gen_mixed: h = G x* - s*, c = G^T y* + lam*."""
    rng = _rng(seed)
    m = int(round(2e7 * scale)); n = int(round(1e7 * scale))
    n1 = int(round(0.4 * n)); n2 = n - n1
    lens = rng.integers(20, 181, size=m).astype(np.int64)
    lens = np.minimum(lens, n)
    row_ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    nnz = int(row_ptr[-1])
    rows = np.repeat(np.arange(m, dtype=np.int64), lens)
    key = rows * n + rng.integers(0, n, nnz)
    while True:                                            # distinct columns within each row
        key.sort()
        dup = np.nonzero(key[1:] == key[:-1])[0] + 1
        if dup.size == 0:
            break
        key[dup] = (key[dup] // n) * n + rng.integers(0, n, dup.size)
    col = (key % n).astype(np.int32)
    del key
    rf = 10.0 ** rng.uniform(-2.0, 2.0, m)
    cf = 10.0 ** rng.uniform(-2.0, 2.0, n)
    val = rng.standard_normal(nnz) * rf[rows] * cf[col]
    giant = tuple([max(3, int(2.5e5 * scale))] * 4)
    rk, rdim = _mixed_cones(rng, m, {ZERO: .30, NONNEG: .30, SOC: .25, RSOC: .05, EXP: .075, DUAL_EXP: .025},
                            giant=giant)
    pk, pdim = _mixed_cones(rng, n2, {ZERO: .01, NONNEG: .20, SOC: .40, RSOC: .15, EXP: .20, DUAL_EXP: .04})
    # box part and its planted (x, lam): interior, at lower, at upper
    btype = rng.integers(0, 4, size=n1)
    lo = rng.uniform(-1.0, 0.0, n1)
    hi = rng.uniform(0.0, 1.0, n1) + lo + 0.5
    l = np.where((btype == 1) | (btype == 3), lo, -INF)
    u = np.where((btype == 2) | (btype == 3), hi, INF)
    status = rng.integers(0, 3, size=n1)
    fl, fu = np.isfinite(l), np.isfinite(u)
    atl = (status == 1) & fl
    atu = (status == 2) & fu & ~atl
    inter = ~(atl | atu)
    x1 = np.where(fl & fu, rng.uniform(0.0, 1.0, n1) * (np.where(fu, u, 0) - np.where(fl, l, 0)) + np.where(fl, l, 0),
                  np.where(fl, np.where(fl, l, 0) + rng.uniform(0.0, 1.0, n1),
                           np.where(fu, np.where(fu, u, 0) - rng.uniform(0.0, 1.0, n1), rng.standard_normal(n1))))
    x1 = np.where(atl, l, np.where(atu, u, x1))
    lam1 = np.where(atl, rng.uniform(0.0, 1.0, n1), np.where(atu, -rng.uniform(0.0, 1.0, n1), 0.0))
    lam1[inter] = 0.0
    x2, lam2 = _planted_pairs(rng, pk, pdim)
    s_star, y_star = _planted_pairs(rng, rk, rdim)
    x_star = np.concatenate([x1, x2]); lam = np.concatenate([lam1, lam2])
    Gx = np.bincount(rows, weights=val * x_star[col], minlength=m)
    GTy = np.bincount(col, weights=val * y_star[rows], minlength=n)
    del rows
    prog = ConicProgram(m=m, n=n, n1=n1, row_ptr=row_ptr, col_idx=col, vals=val,
                        c=GTy + lam, h=Gx - s_star, l=l, u=u, pk=pk, pdim=pdim, rk=rk, rdim=rdim,
                        name=f"mixed_cfg5_scale{scale:g}_s{seed}")
    prog.x_star, prog.y_star = x_star, y_star
    prog.obj_star = float(prog.c @ x_star)
    return prog


# --------------------------------------------------------------------------
# configs[4] at its stated size, generated rank-locally (SURVEY §8(d) cfg 5, §8(e))
# --------------------------------------------------------------------------
_CHUNK_ROWS = 1 << 16        # rows per matrix chunk (one RNG stream each)
_BLOCK_GROUP = 4096          # row-cone blocks per planted-pair group (one RNG stream each)


def _stream(seed: int, tag: int, idx: int) -> np.random.Generator:
    """Independent Philox stream per (seed, tag, idx): a chunk's data does not
    depend on which rank draws it or on the number of ranks."""
    return np.random.Generator(np.random.Philox(np.random.SeedSequence([seed, tag, idx])))


@dataclasses.dataclass
class MixedLayout:
    """The cheap global part of cfg 5 (O(m + n) numbers): row lengths, column
    factors, cone lists, the planted primal pair.  Identical on every rank."""
    scale: float
    seed: int
    m: int
    n: int
    n1: int
    row_ptr: np.ndarray
    cf: np.ndarray
    rk: np.ndarray
    rdim: np.ndarray
    pk: np.ndarray
    pdim: np.ndarray
    l: np.ndarray
    u: np.ndarray
    x_star: np.ndarray
    lam: np.ndarray


@dataclasses.dataclass
class ShardedProgram:
    """Rows [rows[0], rows[1]) of a conic program whose other data is global:
    m is the GLOBAL row count; row_ptr (rebased to 0), col_idx, vals, h and
    y_star are this rank's rows only."""
    m: int
    n: int
    n1: int
    rows: tuple
    row_ptr: np.ndarray
    col_idx: np.ndarray
    vals: np.ndarray
    c: np.ndarray
    h: np.ndarray
    l: np.ndarray
    u: np.ndarray
    pk: np.ndarray
    pdim: np.ndarray
    rk: np.ndarray
    rdim: np.ndarray
    name: str = "shard"
    x_star: np.ndarray | None = None
    y_star: np.ndarray | None = None
    obj_star: float | None = None

    @property
    def nnz(self) -> int:             # this rank's nonzeros
        return int(self.row_ptr[-1])

    @property
    def n2(self) -> int:
        return self.n - self.n1


def mixed_full_layout(scale: float = 1.0, seed: int = 0) -> MixedLayout:
    """Global part of SURVEY §8(d) cfg 5 at `scale` (1.0: m = 2e7, n = 1e7,
    nnz ~ 2e9), same recipe as gen_mixed_large (row lengths U{20..180}, column
    factors 10^U[-2,2], row cones 30/30/25/5/7.5/2.5 % with 4 giant SOC blocks,
    columns 40 % box, 60 % cones), drawn from stream (seed, 0, 0)."""
    rng = _stream(seed, 0, 0)
    m = int(round(2e7 * scale)); n = int(round(1e7 * scale))
    n1 = int(round(0.4 * n)); n2 = n - n1
    lens = np.minimum(rng.integers(20, 181, size=m).astype(np.int64), n)
    row_ptr = np.zeros(m + 1, np.int64)
    np.cumsum(lens, out=row_ptr[1:])
    cf = 10.0 ** rng.uniform(-2.0, 2.0, n)
    giant = tuple([max(3, int(2.5e5 * scale))] * 4)
    rk, rdim = _mixed_cones(rng, m, {ZERO: .30, NONNEG: .30, SOC: .25, RSOC: .05, EXP: .075, DUAL_EXP: .025},
                            giant=giant)
    pk, pdim = _mixed_cones(rng, n2, {ZERO: .01, NONNEG: .20, SOC: .40, RSOC: .15, EXP: .20, DUAL_EXP: .04})
    btype = rng.integers(0, 4, size=n1)
    lo = rng.uniform(-1.0, 0.0, n1)
    hi = rng.uniform(0.0, 1.0, n1) + lo + 0.5
    l = np.where((btype == 1) | (btype == 3), lo, -INF)
    u = np.where((btype == 2) | (btype == 3), hi, INF)
    status = rng.integers(0, 3, size=n1)
    fl, fu = np.isfinite(l), np.isfinite(u)
    atl = (status == 1) & fl
    atu = (status == 2) & fu & ~atl
    inter = ~(atl | atu)
    lz, uz = np.where(fl, l, 0.0), np.where(fu, u, 0.0)
    x1 = np.where(fl & fu, rng.uniform(0.0, 1.0, n1) * (uz - lz) + lz,
                  np.where(fl, lz + rng.uniform(0.0, 1.0, n1),
                           np.where(fu, uz - rng.uniform(0.0, 1.0, n1), rng.standard_normal(n1))))
    x1 = np.where(atl, l, np.where(atu, u, x1))
    lam1 = np.where(atl, rng.uniform(0.0, 1.0, n1), np.where(atu, -rng.uniform(0.0, 1.0, n1), 0.0))
    lam1[inter] = 0.0
    x2, lam2 = _planted_pairs(rng, pk, pdim)
    return MixedLayout(scale, seed, m, n, n1, row_ptr, cf, rk, rdim, pk, pdim, l, u,
                       np.concatenate([x1, x2]), np.concatenate([lam1, lam2]))


def _mixed_chunk(L: MixedLayout, c: int):
    """Rows [c R, (c+1) R) of G: distinct uniform columns per row, values
    N(0,1) * rowfactor * colfactor; stream (seed, 1, c)."""
    rng = _stream(L.seed, 1, c)
    a, b = c * _CHUNK_ROWS, min((c + 1) * _CHUNK_ROWS, L.m)
    lens = np.diff(L.row_ptr[a:b + 1])
    nnz = int(lens.sum())
    rows = np.repeat(np.arange(b - a, dtype=np.int64), lens)
    key = rows * L.n + rng.integers(0, L.n, nnz)
    while True:
        key.sort()
        dup = np.nonzero(key[1:] == key[:-1])[0] + 1
        if dup.size == 0:
            break
        key[dup] = (key[dup] // L.n) * L.n + rng.integers(0, L.n, dup.size)
    col = (key % L.n).astype(np.int32)
    rf = 10.0 ** rng.uniform(-2.0, 2.0, b - a)
    val = rng.standard_normal(nnz) * rf[rows] * L.cf[col]
    return col, val


def _mixed_row_pairs(L: MixedLayout, a: int, b: int):
    """Planted (s*, y*) of rows [a, b): whole groups of _BLOCK_GROUP row-cone
    blocks, stream (seed, 2, group), cut to the rows."""
    starts = np.concatenate([[0], np.cumsum(L.rdim)]).astype(np.int64)
    b0 = int(np.searchsorted(starts, a, side="right")) - 1
    b1 = int(np.searchsorted(starts, b, side="left"))
    s = np.empty(b - a); y = np.empty(b - a)
    for g in range(b0 // _BLOCK_GROUP, (max(b1, b0 + 1) - 1) // _BLOCK_GROUP + 1):
        g0, g1 = g * _BLOCK_GROUP, min((g + 1) * _BLOCK_GROUP, len(L.rdim))
        sg, yg = _planted_pairs(_stream(L.seed, 2, g), L.rk[g0:g1], L.rdim[g0:g1])
        lo, hi = max(a, int(starts[g0])), min(b, int(starts[g1]))
        if hi > lo:
            s[lo - a:hi - a] = sg[lo - starts[g0]:hi - starts[g0]]
            y[lo - a:hi - a] = yg[lo - starts[g0]:hi - starts[g0]]
    return s, y


def gen_mixed_shard(L: MixedLayout, rows, allreduce=None, threads=None) -> ShardedProgram:
    """This rank's rows of cfg 5: its chunks of G, its rows of the planted
    (s*, y*), h = G x* - s* on its rows, and c = G^T y* + lam* where the
    G^T y* partials of all ranks are summed by `allreduce` (None: one rank).
    No process ever holds more than its own rows of G.  Chunks are drawn on
    `threads` host threads (their streams are independent); the G^T y*
    partial is summed chunk by chunk in chunk order (deterministic)."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    a, b = int(rows[0]), int(rows[1])
    rp = L.row_ptr
    nnz = int(rp[b] - rp[a])
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float64)
    h = np.empty(b - a)
    s_star, y_star = _mixed_row_pairs(L, a, b)

    def work(c):
        ca, cb = c * _CHUNK_ROWS, min((c + 1) * _CHUNK_ROWS, L.m)
        lo, hi = max(a, ca), min(b, cb)
        if hi <= lo:
            return None
        cc, cv = _mixed_chunk(L, c)
        src = slice(int(rp[lo] - rp[ca]), int(rp[hi] - rp[ca]))
        dst = slice(int(rp[lo] - rp[a]), int(rp[hi] - rp[a]))
        col[dst] = cc[src]; val[dst] = cv[src]
        lr = np.repeat(np.arange(hi - lo, dtype=np.int64), np.diff(rp[lo:hi + 1]))
        h[lo - a:hi - a] = np.bincount(lr, weights=val[dst] * L.x_star[col[dst]], minlength=hi - lo) \
            - s_star[lo - a:hi - a]
        return np.bincount(col[dst], weights=val[dst] * y_star[lo - a + lr], minlength=L.n)

    cpart = np.zeros(L.n)
    chunks = range(a // _CHUNK_ROWS, (max(b, a + 1) - 1) // _CHUNK_ROWS + 1)
    with ThreadPoolExecutor(threads or min(16, os.cpu_count() or 1)) as ex:
        for cp in ex.map(work, chunks):
            if cp is not None:
                cpart += cp
    if allreduce is not None:
        cpart = allreduce(cpart)
    c = cpart + L.lam
    name = f"mixed_full_scale{L.scale:g}_s{L.seed}"
    return ShardedProgram(m=L.m, n=L.n, n1=L.n1, rows=(a, b), row_ptr=rp[a:b + 1] - rp[a], col_idx=col,
                          vals=val, c=c, h=h, l=L.l, u=L.u, pk=L.pk, pdim=L.pdim, rk=L.rk, rdim=L.rdim,
                          name=name, x_star=L.x_star, y_star=y_star, obj_star=float(c @ L.x_star))
