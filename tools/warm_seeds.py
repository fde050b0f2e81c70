"""Iterations to Eq. 9 <= 1e-4 with and without the warm-started SOC
multipliers (PDCS_WARM) over a few seeds of a bench family (the count moves
with rounding, P5, so one seed says little).

    python tools/warm_seeds.py --family mpo --seeds 0 1 2 3
"""
import argparse, json, os, subprocess, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

ap = argparse.ArgumentParser()
ap.add_argument("--family", default="mpo")
ap.add_argument("--seeds", type=int, nargs="+", default=[0, 1, 2, 3])
ap.add_argument("--child", nargs=2, default=None)
a = ap.parse_args()
if a.child:
    sys.path.insert(0, ROOT)
    import paper_2505_00311_b200 as P
    from instances import gen_mpo, gen_fisher, gen_mixed_large
    seed = int(a.child[1])
    prog = {"mpo": lambda: gen_mpo(100, 1000, seed=seed), "fisher": lambda: gen_fisher(10000, 1000, 0.2, seed=seed),
            "mixed": lambda: gen_mixed_large(1 / 32, seed=seed)}[a.child[0]]()
    g = P.PdcsSolver(prog, tol=1e-4, time_limit_s=120.0)
    t = time.perf_counter()
    r = g.solve()
    print(json.dumps({"family": a.child[0], "seed": seed, "warm": os.environ.get("PDCS_WARM", "1"),
                      "status": r["status"], "iters": r["iters"], "restarts": r["restarts"],
                      "seconds": time.perf_counter() - t}), flush=True)
    sys.exit(0)
for s in a.seeds:
    for w in ("1", "0"):
        subprocess.run([sys.executable, __file__, "--child", a.family, str(s)], env=dict(os.environ, PDCS_WARM=w))
