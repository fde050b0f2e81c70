"""ncu driver: the tiny Lasso (BASELINE configs[0]) for a few hundred iterations."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00311_b200 as P
from instances import gen_lasso
g = P.PdcsSolver(gen_lasso(100, 50, 1.0, seed=0, dense=True))
g.iterate(int(sys.argv[1]) if len(sys.argv) > 1 else 200)
print("done")
