"""Reading P9 study: the oracle on the Lasso proxies of P8,
balanced form (RSOC leading pair (S w, r/S)) next to the literal one.  Prints
one tuple per run: (form, instance, iterations, status, best Eq. 9 of the
returned point, the literal form's Eq. 9 at the back-mapped point, seconds).
Test infrastructure: imports oracle/ only.
  python tests/tools/lasso_balanced.py [--big]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle as O  # noqa: E402
from instances import gen_lasso  # noqa: E402

CASES = [(20000, 2000, 0.01), (10000, 500, 0.1), (1000, 10000, 0.01)]
if "--big" in sys.argv:
    CASES.append((10000, 100000, 1e-4))
for (m, nf, d) in CASES:
    for bal in (True, False):
        p = gen_lasso(m, nf, d, seed=0, balance=bal)
        t = time.perf_counter()
        s = O.OracleSolver(p, tol=1e-4, max_iters=20000)
        r = s.solve()
        x, y = s.get_iterate(3, 1)                 # best point, original space
        e = max(r.kkt.err_p, r.kkt.err_d, r.kkt.err_gap)
        k = O.OracleSolver(p.literal()).kkt_point(p.to_literal(x), y) if bal else None
        el = max(k["err_p"], k["err_d"], k["err_gap"]) if k else e
        print(("balanced" if bal else "literal", (m, nf, d), r.iters, r.status, e, el,
               round(time.perf_counter() - t, 1)), flush=True)
