"""Sweep SpMV row-class bounds (PDCS_SPMV_BINS) on a config; prints per-kernel ms."""
import sys, os, json, time, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00311_b200 as P
from instances import CONFIGS

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="lasso")
ap.add_argument("--iters", type=int, default=40)
ap.add_argument("bins", nargs="*")
a = ap.parse_args()
prog = CONFIGS[a.config](0)
bins = a.bins or ["2,12,96,384,4096"]
for b in bins:
    if ":" in b:
        b, co = b.split(":")
        os.environ["PDCS_CARVEOUT"] = co
    else:
        os.environ.pop("PDCS_CARVEOUT", None)
    os.environ["PDCS_SPMV_BINS"] = b
    g = P.PdcsSolver(prog)
    g.iterate(5)
    g.enable_timing(True)
    t = time.time()
    g.iterate(a.iters)
    el = time.time() - t
    kt = g.kernel_times()
    out = {k: round(v[0] / v[1], 4) for k, v in kt.items() if v[1]}
    tot = sum(v[0] for v in kt.values()) / a.iters
    sc = g.scalars()
    tune = {k: sc[k] for k in sc if k.startswith(("tune", "tiled", "setup"))}
    print(json.dumps({"bins": b, **tune, "ms_per_iter_kernels": round(tot, 4), "wall_ms_per_iter": round(1e3 * el / a.iters, 4), **out}), flush=True)
    g.close()
