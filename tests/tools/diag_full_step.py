import os
import sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle as O
import paper_2505_00311_b200 as P
from instances import CONFIGS
prog = CONFIGS["mixed"](0)
g = P.PdcsSolver(prog); o = O.OracleSolver(prog)
ro, qo = o.get_scaling()
rng = np.random.default_rng(7)
x = rng.standard_normal(prog.n); y = rng.standard_normal(prog.m)
g.set_iterate(x, y); o.set_iterate(x * qo, y * ro)
g.iterate(1); o.iterate(1)
xg, yg = g.get_iterate(P.PDHG_OUT); xo, yo = o.get_iterate(1)
def owner(kinds, dims, base, idx):
    off = np.concatenate([[0], np.cumsum(dims)]) + base
    b = np.searchsorted(off, idx, side='right') - 1
    return b, int(kinds[b]) if 0 <= b < len(kinds) else -1, int(dims[b]) if 0 <= b < len(kinds) else -1
for name, a, bb, kinds, dims, base in (("x", xg, xo, prog.pk, prog.pdim, prog.n1), ("y", yg, yo, prog.rk, prog.rdim, 0)):
    d = np.abs(a - bb); scale = 1 + np.abs(bb).max()
    top = np.argsort(-d)[:8]
    print(name, 'max rel', d.max() / scale, 'scale', scale)
    for i in top:
        print('  idx', i, 'diff', d[i], 'g', a[i], 'o', bb[i], 'block', owner(kinds, dims, base, i) if i >= base else 'box')
