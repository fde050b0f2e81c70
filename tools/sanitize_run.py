"""Small driver for compute-sanitizer (memcheck / racecheck / synccheck): every
kernel family of the hot path on small instances -- the sliced tiled sweeps with
cp.async double buffering and bank-balanced layouts (tiny tiles, so many staged
segments), the device-balanced tiled build, the L2-panel sweeps, the box-column
order, every projection team, the Eq. 9 check, restarts.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00311_b200 as P
from instances import gen_fisher, gen_lasso, gen_mixed

runs = [
    ("lasso tiled 1 KB", dict(PDCS_TILED="1", PDCS_TILE_KB="1"), lambda: gen_lasso(600, 80, 0.3, seed=1)),
    ("mixed tiled 2 KB", dict(PDCS_TILED="1", PDCS_TILE_KB="2"),
     lambda: gen_mixed(800, 80, 400, seed=2, soc_dims=(3, 600))),
    ("mixed panels 3", dict(PDCS_TILED="0", PDCS_PANELS="3"), lambda: gen_mixed(800, 80, 400, seed=3)),
    ("fisher colperm", dict(PDCS_TILED="0"), lambda: gen_fisher(1100, 20, seed=4)),
]
for name, env, make in runs:
    for k in ("PDCS_TILED", "PDCS_TILE_KB", "PDCS_PANELS"):
        os.environ.pop(k, None)
    os.environ.update(env)
    g = P.PdcsSolver(make())
    r = g.iterate(int(os.environ.get("SAN_ITERS", "45")))
    print(name, "iters", r["iters"], "restarts", r["restarts"], flush=True)
    g.close()
# the standalone projection with every team forced (cluster and grid included)
if os.environ.get("SAN_PROJ", "1") == "0":
    print("done")
    sys.exit(0)
import numpy as np
import torch
from instances import SOC, RSOC, EXP
kinds = np.array([SOC, RSOC, EXP, SOC], np.int32)
dims = np.array([5000, 700, 3, 40], np.int64)
rng = np.random.default_rng(0)
v = torch.from_numpy(rng.standard_normal(int(dims.sum()))).cuda()
D = torch.from_numpy(rng.uniform(0.5, 2.0, int(dims.sum()))).cuda()
D[5001] = D[5000]
for team in ("auto", "thread", "warp", "cta", "cluster", "grid"):
    plan = P.pdcs_proj_create(kinds, dims, team=team)
    out = torch.empty_like(v)
    P.pdcs_proj_run(plan, D, v, out)
    torch.cuda.synchronize()
    P.pdcs_proj_destroy(plan)
    print("proj", team, flush=True)
print("done")
