"""Lasso study m8: the SOC of PAPER.md:1641-1659 read as a ROW constraint (G x - h in K_soc^{m+2}
with w, r, y free), literal (y kept) and with y eliminated, against reading A22 (primal RSOC).
Runs the oracle only (test tooling)."""
import sys, os, time, numpy as np
sys.path.insert(0, "/root/repo")
import oracle as O
from instances import gen_lasso
from instances.program import ConicProgram, csr_from_coo, ZERO, SOC
INF = np.inf

def lasso_rowsoc(m, nf, d, seed=0, elim_y=False):
    base = gen_lasso(m, nf, d, seed)
    arow, acol, aval, m_, nf_ = base.lasso_A
    b, lam = base.lasso_b, base.lasso_lam
    s2 = 1/np.sqrt(2)
    if not elim_y:
        n1 = 2*nf; iw, ir, iy = n1, n1+1, n1+2; n = n1+2+m
        R, Cc, V = [0], [iw], [1.0]
        # rows 1..m : y - A x+ + A x- = -b
        R += list(1+arow); Cc += list(acol); V += list(-aval)
        R += list(1+arow); Cc += list(nf+acol); V += list(aval)
        R += list(1+np.arange(m)); Cc += list(iy+np.arange(m)); V += [1.0]*m
        s0 = m+1
        R += [s0, s0, s0+1, s0+1]; Cc += [iw, ir, iw, ir]; V += [s2, s2, s2, -s2]
        R += list(s0+2+np.arange(m)); Cc += list(iy+np.arange(m)); V += [1.0]*m
        mr = 2*m+3
        h = np.zeros(mr); h[0] = 1; h[1:m+1] = -b
        rk = np.array([ZERO, SOC], np.int32); rdim = np.array([m+1, m+2], np.int64)
    else:
        n1 = 2*nf; iw, ir = n1, n1+1; n = n1+2
        R, Cc, V = [0], [iw], [1.0]
        s0 = 1
        R += [s0, s0, s0+1, s0+1]; Cc += [iw, ir, iw, ir]; V += [s2, s2, s2, -s2]
        R += list(s0+2+arow); Cc += list(acol); V += list(aval)
        R += list(s0+2+arow); Cc += list(nf+acol); V += list(-aval)
        mr = m+3
        h = np.zeros(mr); h[0] = 1; h[3:] = b
        rk = np.array([ZERO, SOC], np.int32); rdim = np.array([1, m+2], np.int64)
    rp, ci, vv = csr_from_coo(mr, n, np.array(R), np.array(Cc), np.array(V))
    c = np.zeros(n); c[:n1] = lam; c[ir] = 2.0
    l = np.full(n, -INF); u = np.full(n, INF); l[:n1] = 0
    return ConicProgram(m=mr, n=n, n1=n, row_ptr=rp, col_idx=ci.astype(np.int32), vals=vv, c=c, h=h,
        l=l, u=u, pk=np.zeros(0, np.int32), pdim=np.zeros(0, np.int64), rk=rk, rdim=rdim, name="rowsoc")

def run(prog, iters, chunk=200, tag="", **kw):
    S = O.OracleSolver(prog, **kw)
    t0 = time.time(); done = 0
    while done < iters:
        S.iterate(chunk); done += chunk
        sc = S.scalars()
        if done % (chunk*10) == 0:
            print(tag, done, "best %.2e cur(%.1e %.1e %.1e) rs %d om %.3g" % (sc["best_e"], sc["cur_err_p"], sc["cur_err_d"], sc["cur_err_gap"], sc["restarts"], sc["omega"]), flush=True)
        if sc["best_e"] <= 1e-4: break
    print(tag, "END", done, sc["best_e"], time.time()-t0, flush=True)

if __name__ == "__main__":
    m, nf, d, it, mode = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
    if mode == "rsoc": p = gen_lasso(m, nf, d, 0)
    elif mode == "row": p = lasso_rowsoc(m, nf, d)
    else: p = lasso_rowsoc(m, nf, d, elim_y=True)
    print(mode, p.m, p.n, p.nnz, flush=True)
    run(p, it, tag=mode)
