"""Small driver for ncu: a Lasso instance (rows scaled down, still >> L2) and a few iterations."""
import sys, os, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2505_00311_b200 as P
from instances import gen_lasso, gen_fisher, gen_mpo, gen_mixed_large, mixed_full_layout, gen_mixed_shard

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="lasso")
ap.add_argument("--m", type=int, default=200000)
ap.add_argument("--iters", type=int, default=30)
ap.add_argument("--scale", type=float, default=1.0 / 32)
ap.add_argument("--T", type=int, default=20, help="MPO periods (bench config: 100)")
a = ap.parse_args()
if a.config == "lasso":
    prog = gen_lasso(a.m, 10000, 0.01, seed=0)
elif a.config == "fisher":
    prog = gen_fisher(10000, 1000, 0.2, seed=0)
elif a.config == "mixed":
    prog = gen_mixed_large(a.scale, seed=0)
elif a.config == "mixed_full":
    L = mixed_full_layout(a.scale, 0)
    prog = gen_mixed_shard(L, (0, L.m))
else:
    prog = gen_mpo(a.T, 1000, seed=0)
g = P.PdcsSolver(prog)
g.iterate(a.iters)
print("done", prog.m, prog.n, prog.nnz)
