"""End-to-end solves at the paper's Table 3/4/5 sizes.

Synthetic instances of the paper's three families at the sizes of its tables,
solved on the GPU through the C ABI to relative KKT (Eq. 9) 1e-3 and then,
continuing the same trajectory (pdcs_set_tolerance), to 1e-6:

  Lasso   PAPER.md:1062-1074 (Table 4): A m x n at density 1e-4, U[0,1]
          (recipe PAPER.md:1663-1664), m/n = 1e4/1e5 ... 7.5e5/7.5e6
  Fisher  PAPER.md:969-983 (Table 3): buyers x goods at density 0.2
          (PAPER.md:1618-1623), 1e2 x 5e3 ... 2.8e5 x 1e3
  MPO     PAPER.md:1125-1141 (Table 5): 844 assets, T periods
          3 ... 1440, synthetic covariance (reading A24)

The paper's cuPDCS seconds (H100) are quoted beside each row as context only;
they are not a target (other machine, real CBLIB/Yahoo data where it applies).
Each tolerance stage has its own time limit; one JSON line per instance is
appended to --out as soon as it finishes.

    python tools/paper_sizes.py --suite lasso,fisher,mpo --limit 300 --out X.jsonl
"""
import argparse, json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# (name, family, args, paper cuPDCS seconds at 1e-3, at 1e-6)
SUITE = [
    ("lasso_1e4x1e5", "lasso", (10_000, 100_000), 7.1e-2, 1.1e-1),
    ("lasso_7e4x7e5", "lasso", (70_000, 700_000), 2.9e-1, 8.4e-1),
    ("lasso_4e5x7e6", "lasso", (400_000, 7_000_000), 1.2e2, 2.6e2),
    ("lasso_7e5x7e6", "lasso", (700_000, 7_000_000), 3.2e2, 5.2e2),
    ("lasso_7.5e5x7.5e6", "lasso", (750_000, 7_500_000), 4.7e2, 6.0e2),
    ("fisher_1e2x5e3", "fisher", (100, 5_000), 1.5e1, 3.7e1),
    ("fisher_1e5x1e3", "fisher", (100_000, 1_000), 4.6e2, 1.8e3),
    ("fisher_1.5e5x1e3", "fisher", (150_000, 1_000), 4.3e2, 2.8e3),
    ("fisher_2e5x1e3", "fisher", (200_000, 1_000), 1.1e3, 4.2e3),
    ("fisher_2.5e5x1e3", "fisher", (250_000, 1_000), 1.4e3, 5.7e3),
    ("fisher_2.8e5x1e3", "fisher", (280_000, 1_000), 1.6e3, 6.2e3),
    ("mpo_T3", "mpo", (3, 844), 1.9e0, 7.5e0),
    ("mpo_T48", "mpo", (48, 844), 7.2e0, 1.8e1),
    ("mpo_T96", "mpo", (96, 844), 1.1e1, 5.7e1),
    ("mpo_T360", "mpo", (360, 844), 5.1e1, 4.2e2),
    ("mpo_T1440", "mpo", (1440, 844), 4.9e2, 3.4e3),
    ("mpo_T2160", "mpo", (2160, 844), 5.8e2, 1.0e3),
    ("mpo_T3600", "mpo", (3600, 844), 1.1e3, 9.0e3),
]


def make(family, args, seed):
    from instances import gen_lasso, gen_fisher, gen_mpo
    if family == "lasso":
        return gen_lasso(args[0], args[1], 1e-4, seed=seed)
    if family == "fisher":
        return gen_fisher(args[0], args[1], 0.2, seed=seed)
    return gen_mpo(args[0], args[1], seed=seed)


def host_mem_gb():
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) / 2**20
    except OSError:
        pass
    return None


def est_knnz(family, args):
    if family == "lasso":
        return 2 * args[0] * args[1] * 1e-4 + args[0]
    if family == "fisher":
        return 1.2 * args[0] * args[1]
    return args[0] * (args[1] + 1) ** 2


def run_one(P, name, family, args, paper, limit, seed):
    # generator temporaries + host tiled build (measured: gen_mpo peaks at ~80 B per nonzero)
    need = (105.0 if family == "mpo" else 120.0) * est_knnz(family, args) / 2**30
    if est_knnz(family, args) >= 2**31:
        return dict(instance=name, skipped="local nnz >= 2^31: libpdcs keeps int32 row pointers per rank "
                                           "(shard the rows over ranks)")
    avail = host_mem_gb()
    if avail is not None and need > 0.7 * avail:
        return dict(instance=name, skipped=f"host RAM: ~{need:.0f} GB needed, {avail:.0f} GB available")
    t0 = time.perf_counter()
    prog = make(family, args, seed)
    gen_s = time.perf_counter() - t0
    rec = dict(instance=name, family=family, args=list(args), m=prog.m, n=prog.n, nnz=prog.nnz,
               gen_seconds=gen_s, paper_cupdcs_seconds={"1e-3": paper[0], "1e-6": paper[1]},
               paper_hardware="H100 80 GB (PAPER.md:815), context only")
    t1 = time.perf_counter()
    g = P.PdcsSolver(prog, tol=1e-3, time_limit_s=limit, max_iters=10**9)
    setup = time.perf_counter() - t1
    rec["setup_seconds"] = setup
    stages = []
    solve_total = 0.0
    for tol in (1e-3, 1e-6):
        g.set_tolerance(tol, limit)
        ts = time.perf_counter()
        r = g.solve()
        el = time.perf_counter() - ts
        solve_total += el
        stages.append(dict(tol=tol, status=r["status"], seconds_solve_cum=solve_total,
                           seconds_incl_setup=solve_total + setup, iters=r["iters"],
                           trials=r["trials"], restarts=r["restarts"],
                           kkt_max=max(r["err_p"], r["err_d"], r["err_gap"]),
                           err_p=r["err_p"], err_d=r["err_d"], err_gap=r["err_gap"],
                           pobj=r["pobj"], dobj=r["dobj"],
                           iters_per_s=None))
        if r["status"] != "OPTIMAL":
            break
    for s in stages:
        s["iters_per_s"] = s["iters"] / max(s["seconds_solve_cum"], 1e-9)
    rec["stages"] = stages
    g.close()
    del prog
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--suite", default="lasso,fisher,mpo")
    ap.add_argument("--only", default="", help="comma list of instance names")
    ap.add_argument("--limit", type=float, default=300.0, help="seconds per tolerance stage")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    from paper_2505_00311_b200 import build
    build.build()
    import paper_2505_00311_b200 as P
    fams = set(a.suite.split(","))
    only = set(x for x in a.only.split(",") if x)
    for name, fam, args, *paper in SUITE:
        if fam not in fams or (only and name not in only):
            continue
        try:
            rec = run_one(P, name, fam, args, paper, a.limit, a.seed)
        except Exception as e:  # record and continue (e.g. host RAM for the largest rows)
            rec = dict(instance=name, error=f"{type(e).__name__}: {e}")
        rec["host_mem_available_gb"] = host_mem_gb()
        print(json.dumps(rec), flush=True)
        if a.out:
            with open(a.out, "a") as f:
                f.write(json.dumps(rec) + "\n")


if __name__ == "__main__":
    main()
