"""Long solve of a bench config toward Eq. 9 <= tol, logging the trajectory.

The bench's time-to-1e-4 leg is capped at 120 s; this runs the same solve in
slices of `--slice` seconds (pdcs_set_tolerance continues the trajectory, so the
run is the one pdcs_solve would make) up to `--limit` seconds and prints one
JSON line per slice: wall s, accepted iterations, restarts, the best point's
Eq. 9 errors.  Usage:
  python tools/long_solve.py --config lasso --tol 1e-4 --limit 1200 --slice 60
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2505_00311_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="lasso")
ap.add_argument("--tol", type=float, default=1e-4)
ap.add_argument("--limit", type=float, default=1200.0)
ap.add_argument("--slice", type=float, default=60.0)
a = ap.parse_args()

import torch  # noqa: E402

prog, gen_s = bench.build_instance(a.config, 0)
rows = (0, prog.m)
host = bench.pinned(prog, rows)
st = torch.cuda.Stream()
t0 = time.perf_counter()
ctx = bench.make_ctx(P, prog, host, P.pdcs_default_params(tol=a.tol, time_limit_s=a.slice), st.cuda_stream, 0, rows)
print(json.dumps({"config": a.config, "m": prog.m, "n": prog.n, "nnz": prog.nnz, "setup_s": time.perf_counter() - t0}),
      flush=True)
while True:
    r = P.pdcs_solve(ctx)
    k = r.kkt                                  # Eq. 9 of the returned (best) point
    sc = P.pdcs_get_scalars(ctx)
    line = {"wall_s": time.perf_counter() - t0, "status": r.status, "iters": int(sc["total"]),
            "restarts": int(sc["restarts"]), "best_e": sc["best_e"], "err_p": k.err_p, "err_d": k.err_d,
            "err_gap": k.err_gap, "pobj": k.pobj, "dobj": k.dobj, "omega": sc["omega"], "eta": sc["eta"]}
    print(json.dumps(line), flush=True)
    if r.status != 2 or time.perf_counter() - t0 >= a.limit:
        break
    P.pdcs_set_tolerance(ctx, a.tol, a.slice)
P.pdcs_destroy(ctx)
