"""PDCS vs vanilla PDHG (App. D).

Both run on the GPU through the C ABI on the same generated instances: PDCS
with its defaults, vanilla PDHG with vanilla_pdhg=1 (tau = sigma = 0.9/||G||_2,
no scaling, restarts, Halpern or primal weights).  Target:
Eq. 9 relative KKT <= tol.  Vanilla's iteration budget is 10x the iterations
PDCS needed, and capped runs are counted at the cap.  The cost
measure is matrix passes over K / K^T (pdcs_result_t.spmv_K + spmv_KT).

    python tools/pdcs_vs_pdhg.py [--tol 1e-4] [--out profiles/r1_pdcs_vs_pdhg.json]
"""
import argparse, json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def instances():
    from instances import gen_lasso, gen_fisher, gen_mpo, gen_mixed
    for s in range(3):
        yield f"lasso_2000x200_d0.05_s{s}", lambda s=s: gen_lasso(2000, 200, 0.05, seed=s)
        yield f"fisher_100x50_s{s}", lambda s=s: gen_fisher(100, 50, 0.2, seed=s)
        yield f"mpo_T5_n50_s{s}", lambda s=s: gen_mpo(5, 50, seed=s)
        yield f"mixed_2000_s{s}", lambda s=s: gen_mixed(2000, 300, 1500, seed=s, soc_dims=(3, 60))


def run(P, prog, tol, max_iters, time_limit, vanilla):
    g = P.PdcsSolver(prog, tol=tol, max_iters=max_iters, time_limit_s=time_limit, vanilla_pdhg=int(vanilla))
    t = time.perf_counter()
    r = P.pdcs_solve(g.ctx)
    el = time.perf_counter() - t
    out = dict(status=r.status, iters=r.iters, trials=r.trials, passes=r.spmv_K + r.spmv_KT,
               kkt=max(r.kkt.err_p, r.kkt.err_d, r.kkt.err_gap), seconds=el, restarts=r.restarts)
    g.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tol", type=float, default=1e-4)
    ap.add_argument("--time-limit", type=float, default=60.0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    from paper_2505_00311_b200 import build
    build.build()
    import paper_2505_00311_b200 as P
    rows = []
    for name, mk in instances():
        prog = mk()
        pd = run(P, prog, a.tol, 2_000_000, a.time_limit, False)
        cap = 10 * max(pd["iters"], 1)
        va = run(P, prog, a.tol, cap, a.time_limit, True)
        solved_v = va["status"] == 0
        va_passes = va["passes"] if solved_v else max(va["passes"], 2 * cap)
        rec = dict(instance=name, m=prog.m, n=prog.n, nnz=prog.nnz, pdcs=pd, vanilla=va,
                   vanilla_capped=not solved_v, ratio=pd["passes"] / va_passes)
        rows.append(rec)
        print(json.dumps(rec), flush=True)
    ratios = [r["ratio"] for r in rows if r["pdcs"]["status"] == 0]
    summ = dict(tol=a.tol, instances=len(rows), pdcs_solved=sum(r["pdcs"]["status"] == 0 for r in rows),
                vanilla_solved=sum(r["vanilla"]["status"] == 0 for r in rows),
                median_pass_ratio_pdcs_over_vanilla=float(np.median(ratios)) if ratios else None)
    print(json.dumps(summ), flush=True)
    if a.out:
        json.dump({"summary": summ, "rows": rows}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
