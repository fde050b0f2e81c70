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
for (m, nf, d) in ([] if "--sweep" in sys.argv else CASES):
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

if "--sweep" in sys.argv:
    # the choice of S: w' = S, r' = r*/S; iterations to 1e-4 against S = f * ||b||^2/2
    import dataclasses
    for (m, nf, d) in CASES[:3]:
        lit = gen_lasso(m, nf, d, seed=0, balance=False)
        S0 = float(lit.lasso_b @ lit.lasso_b) / 2.0
        out = []
        for f in (1e-3, 3e-3, 1e-2, 3e-2, 0.1, 1.0, 1.0 / S0 ** 0.5):
            S = S0 * f
            v = lit.vals.copy(); v[0] = 1.0 / S
            c = lit.c.copy(); c[lit.n1 + 1] = 2.0 * S
            s = O.OracleSolver(dataclasses.replace(lit, vals=v, c=c), tol=1e-4, max_iters=20000)
            r = s.solve()
            x, _ = s.get_iterate(3, 1)
            out.append((round(f, 5), r.status, r.iters, round(x[lit.n1 + 1] * S / S0, 3)))
        print("sweep", (m, nf, d), "S0 = ||b||^2/2 =", round(S0, 1), "(f, status, iters, r*/S0):", out, flush=True)
