"""Fisher scaling study (DESIGN.md next-round item 1): the oracle on
gen_fisher(1000, 100) with the allocation rescaled, X' = a X (supply rows
sum_i X'_ij = a b_j, t rows (U_i / a) X'_i - t_i = 0): the same market, the
same t, p and objective; prices scale by 1/a.  Prints (a, status, iterations,
Eq. 9 max, seconds) at tol 1e-4, cap 3e4 iterations.  Test infrastructure:
imports oracle/ only.   python tests/tools/fisher_scaling.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle as O  # noqa: E402
from instances import gen_fisher  # noqa: E402

mb, ng = 1000, 100
for a in (1.0, 10.0, 100.0, 0.1):
    p = gen_fisher(mb, ng, seed=0)
    p.h[:ng] *= a
    for r in range(ng, ng + mb):
        lo, hi = p.row_ptr[r], p.row_ptr[r + 1]
        sel = p.vals[lo:hi] > 0
        p.vals[lo:hi][sel] /= a
    t = time.perf_counter()
    r = O.OracleSolver(p, tol=1e-4, max_iters=30000).solve()
    print(a, r.status, r.iters, max(r.kkt.err_p, r.kkt.err_d, r.kkt.err_gap), round(time.perf_counter() - t, 1),
          flush=True)
