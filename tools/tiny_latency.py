"""Per-iteration latency of the graph path on small instances (fixed overheads,
PAPER.md:918): wall time of pdcs_iterate(N) after a warm-up, per accepted step.

    python tools/tiny_latency.py [--iters 2000]
"""
import argparse, json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=2000)
    a = ap.parse_args()
    from instances import gen_lasso, gen_fisher, gen_mpo
    import paper_2505_00311_b200 as P
    cases = {"tiny_lasso_100x50": lambda: gen_lasso(100, 50, 1.0, seed=0, dense=True),
             "lasso_1e4x1e5_d1e-4": lambda: gen_lasso(10_000, 100_000, 1e-4, seed=0),
             "fisher_100x50": lambda: gen_fisher(100, 50, 0.2, seed=0),
             "mpo_T3_n50": lambda: gen_mpo(3, 50, seed=0)}
    for name, mk in cases.items():
        g = P.PdcsSolver(mk())
        g.iterate(200)
        t = time.perf_counter()
        r = g.iterate(a.iters)
        el = time.perf_counter() - t
        print(json.dumps(dict(instance=name, iters=a.iters, us_per_iter=el / a.iters * 1e6,
                              trials=r["trials"], launches=P.pdcs_launch_count(g.ctx))), flush=True)
        g.close()


if __name__ == "__main__":
    main()
