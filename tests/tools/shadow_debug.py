import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import oracle as O
import paper_2505_00311_b200 as P
from instances import gen_lasso
prog = gen_lasso(100, 50, 1.0, seed=0, dense=True)
o = O.OracleSolver(prog); g = P.PdcsSolver(prog)
o.iterate(1590)
g.set_state(o.get_state())
for s in range(10):
    o.iterate(1); g.iterate(1)
    so, sg = o.scalars(), g.scalars()
    xg, yg = g.get_iterate(P.CURRENT); xo, yo = o.get_iterate(0)
    par = max(np.abs(xg-xo).max()/(1+np.abs(xo).max()), np.abs(yg-yo).max()/(1+np.abs(yo).max()))
    print(s, f"par {par:.2e} eta g {sg['eta']:.16e} o {so['eta']:.16e} rel {abs(sg['eta']-so['eta'])/so['eta']:.1e}"
          f" num g {sg['last_num']:.6e} o {so['last_num']:.6e} cross g {sg['last_cross']:.6e} o {so['last_cross']:.6e}"
          f" cond(cross) {so['last_cross_abs']/abs(so['last_cross']):.1e}")
