"""Solve a JSON instance file or a CBF-subset file on the GPU through the C ABI
(SolveReport fields of SPEC.md:599-602).

    python tools/solve_file.py problem.cbf [--tol 1e-6] [--time-limit 60] [--x out.npy]

Prints one JSON report: status, objective in the file's own sense (CBF
constant and OBJSENSE applied), Eq. 9 residuals of the returned point,
iterations, restarts, matrix passes, wall seconds and the parameters used.
"""
import argparse, json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("path")
    ap.add_argument("--tol", type=float, default=1e-6)
    ap.add_argument("--time-limit", type=float, default=0.0)
    ap.add_argument("--max-iters", type=int, default=10**9)
    ap.add_argument("--x", default=None, help="write the primal solution (file variable order) here")
    a = ap.parse_args()
    from instances.io import read_instance, to_cbf_solution
    import paper_2505_00311_b200 as P
    prog = read_instance(a.path)
    t0 = time.perf_counter()
    g = P.PdcsSolver(prog, tol=a.tol, time_limit_s=a.time_limit, max_iters=a.max_iters)
    r = P.pdcs_solve(g.ctx)
    wall = time.perf_counter() - t0
    sign = getattr(prog, "obj_sign", 1.0)
    const = getattr(prog, "obj_const", 0.0)
    rep = dict(instance=a.path, m=prog.m, n=prog.n, nnz=prog.nnz,
               status=P._lib.SOLVE_STATUS.get(r.status, r.status),
               primal_obj=sign * (r.kkt.pobj + const), dual_obj=sign * (r.kkt.dobj + const),
               err_p=r.kkt.err_p, err_d=r.kkt.err_d, err_gap=r.kkt.err_gap, iterations=r.iters,
               trials=r.trials, restarts=r.restarts, spmv_count=r.spmv_K + r.spmv_KT,
               wall_seconds=wall, params=dict(tol=a.tol, time_limit_s=a.time_limit, max_iters=a.max_iters))
    if a.x:
        x, _ = g.get_iterate(P.BEST, P.ORIGINAL)
        np.save(a.x, to_cbf_solution(prog, x) if hasattr(prog, "var_perm") else x)
    g.close()
    print(json.dumps(rep))


if __name__ == "__main__":
    main()
