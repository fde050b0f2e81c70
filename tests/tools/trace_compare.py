"""Compare GPU vs oracle control state at every check (debug aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import oracle as O
import paper_2505_00311_b200 as P
from instances import gen_lasso

prog = gen_lasso(100, 50, 1.0, seed=0, dense=True)
g = P.PdcsSolver(prog)
o = O.OracleSolver(prog)
keys = ["restarts", "k", "omega", "eta", "beta", "e_anchor", "e_prev", "cur_err_p", "cur_err_d", "cur_err_gap", "avg_err_p", "avg_err_d", "avg_err_gap"]
for chk in range(40):
    g.iterate(40); o.iterate(40)
    sg, so = g.scalars(), o.scalars()
    xg, yg = g.get_iterate(P.CURRENT); xo, yo = o.get_iterate(0)
    par = max(np.abs(xg-xo).max()/(1+np.abs(xo).max()), np.abs(yg-yo).max()/(1+np.abs(yo).max()))
    print(f"chk {chk} par {par:.2e}")
    for k in keys:
        a, b = sg[k], so[k]
        flag = "" if abs(a-b) <= 1e-9*(1+abs(b)) else "   <<<"
        print(f"   {k:12s} gpu {a:.15e} orc {b:.15e}{flag}")
    if sg["restarts"] != so["restarts"]:
        break
