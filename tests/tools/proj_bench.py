"""Projection microbenchmarks (Fig. 3, 782-793 Fig. 4).

Fig. 3 setup: a random vector of R^{m(d+1)} projected onto m second-order cones
of dimension d+1, d = ceil(1.2e9 / m), for each parallel strategy (the paper's
thread-, block- and grid-wise, plus this build's warp and 8-CTA cluster teams
and its size-class dispatch "auto").  Fig. 4 setup: a random vector projected
onto N exponential cones (one thread per cone).  Unit scaling, as in the paper
("projecting a randomly generated vector"); the rescaled variant is timed for
the auto dispatch.

Timing: CUDA events on the launch stream, 1 warm-up + R timed runs, mean and
std.  A (strategy, m) whose modelled time exceeds the paper's 15 s limit is
reported as ">15 s" without running.  Effective bandwidth = 16 bytes per
element (one read of v, one write of the result: the algorithmic minimum) over
the time, against MEASURED_PEAKS.json.  CPU baseline: the oracle's per-block
projections (single thread) on a bounded sample of the same cones,
extrapolated per element.

    python tests/tools/proj_bench.py [--fig soc|exp|both] [--reps 3] [--out profiles/r1_proj.json]
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

SOC, EXP = 2, 4
LIMIT_S = 15.0
PREV = None
TEAM_LANES = {"thread": 1, "warp": 32, "cta": 256, "cluster": 2048}


def peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return float(json.load(open(p))["hbm_gbs"]) if os.path.exists(p) else 6650.0


def model_s(team, m, d, sms=148):
    """Crude upper model (8 passes, 4 ns per element-pass per lane, 15 us per
    grid-wide cone) used only to skip runs beyond the paper's 15 s limit."""
    if team == "grid":
        return m * 15e-6 + m * d * 8 * 4e-9 / (2 * sms * 256)
    if team == "auto":
        return 0.0
    lanes = TEAM_LANES[team]
    teams = {"thread": sms * 32 * 64, "warp": sms * 64, "cta": sms * 4, "cluster": sms * 2 // 8}[team]
    waves = math.ceil(m / teams)
    return waves * d * 8 * 4e-9 / lanes


def time_plan(P, torch, plan, D, v, out, reps):
    st = torch.cuda.current_stream()
    P.pdcs_proj_run(plan, D, v, out, st)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        P.pdcs_proj_run(plan, D, v, out, st)
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return float(np.mean(ts)), float(np.std(ts))


def cpu_rate(kind, d, budget=1.5, seed=0):
    """Oracle seconds per element (single thread) on a bounded sample of cones."""
    import oracle as O
    rng = np.random.default_rng(seed)
    done, t0 = 0, time.perf_counter()
    dd = min(d, 2_000_000)
    while True:
        v = rng.standard_normal(dd)
        if kind == SOC:
            O.proj_soc_scaled(v, np.ones(dd))
        else:
            for _ in range(1000):
                O.proj_exp_scaled(rng.standard_normal(3))
            dd = 3000
        done += dd
        el = time.perf_counter() - t0
        if el > budget:
            return el / done, f"{done} elements in {el:.2f}s"


def fig_soc(P, torch, reps, rows, peak_gbs, prev=None):
    ms = [1, 10, 100, 1000, 10**4, 10**5, 10**6, 10**7, 10**8]
    teams = ["auto", "thread", "warp", "cta", "cluster", "grid"]
    for m in ms:
        d = math.ceil(1.2e9 / m)
        n = m * (d + 1)
        kinds = np.full(m, SOC, np.int32)
        dims = np.full(m, d + 1, np.int64)
        g = torch.Generator(device="cuda").manual_seed(m)
        v = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
        out = torch.empty_like(v)
        cpu_s_per_el, cpu_sample = cpu_rate(SOC, d + 1)
        for team in teams + ["auto_rescaled"]:
            tname = "auto" if team == "auto_rescaled" else team
            rec = {"fig": "soc", "m": m, "d": d + 1, "n": n, "team": team,
                   "cpu_oracle_s_extrapolated": cpu_s_per_el * n, "cpu_sample": cpu_sample}
            est = model_s(tname, m, d + 1)
            old = (prev or {}).get((m, team))
            if old is not None and old > 3.0:
                rec.update({"skipped": f"{old:.1f}s in the previous run ({os.path.basename(PREV)})", "previous_s": old})
                rows.append(rec); print(json.dumps(rec), flush=True)
                continue
            if est > LIMIT_S:
                rec.update({"skipped": f"modelled {est:.0f}s > {LIMIT_S:.0f}s limit (PAPER.md:723)"})
                rows.append(rec); print(json.dumps(rec), flush=True)
                continue
            D = None
            if team == "auto_rescaled":
                D = torch.empty_like(v).uniform_(0.5, 2.0, generator=g)
            plan = P.pdcs_proj_create(kinds, dims, team=tname)
            try:
                mean, std = time_plan(P, torch, plan, D, v, out, reps)
                info = P.pdcs_proj_info(plan)
            finally:
                P.pdcs_proj_destroy(plan)
            byts = (24 if D is not None else 16) * n
            rec.update({"seconds": mean, "std": std, "GB/s": byts / mean / 1e9, "frac_hbm": byts / mean / 1e9 / peak_gbs,
                        "over_limit": mean > LIMIT_S, "classes": info["counts"]})
            rows.append(rec); print(json.dumps(rec), flush=True)
            del D
        del v, out
        torch.cuda.empty_cache()


def fig_exp(P, torch, reps, rows, peak_gbs):
    for N in [10**3, 10**4, 10**5, 10**6, 10**7, 10**8, 4 * 10**8]:
        n = 3 * N
        g = torch.Generator(device="cuda").manual_seed(N)
        v = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
        out = torch.empty_like(v)
        cpu_s_per_el, cpu_sample = cpu_rate(EXP, 3)
        plan = P.pdcs_proj_create(np.full(N, EXP, np.int32), np.full(N, 3, np.int64), team="auto")
        try:
            mean, std = time_plan(P, torch, plan, None, v, out, reps)
        finally:
            P.pdcs_proj_destroy(plan)
        rec = {"fig": "exp", "cones": N, "n": n, "seconds": mean, "std": std, "cones_per_s": N / mean,
               "GB/s": 16 * n / mean / 1e9, "frac_hbm": 16 * n / mean / 1e9 / peak_gbs,
               "cpu_oracle_s_extrapolated": cpu_s_per_el * n, "cpu_sample": cpu_sample}
        rows.append(rec); print(json.dumps(rec), flush=True)
        del v, out
        torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--fig", default="both", choices=["soc", "exp", "both"])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=None)
    ap.add_argument("--prev", default=None, help="skip (m, team) runs that took > 3 s in this earlier output")
    a = ap.parse_args()
    import torch
    from paper_2505_00311_b200 import build
    build.build()
    import paper_2505_00311_b200 as P
    rows = []
    pk = peak()
    prev = None
    if a.prev:
        global PREV
        PREV = a.prev
        prev = {(r["m"], r["team"]): r["seconds"] for r in json.load(open(a.prev))["rows"]
                if r["fig"] == "soc" and "seconds" in r}
    if a.fig in ("soc", "both"):
        fig_soc(P, torch, a.reps, rows, pk, prev)
    if a.fig in ("exp", "both"):
        fig_exp(P, torch, a.reps, rows, pk)
    if a.out:
        json.dump({"gpu": torch.cuda.get_device_name(0), "hbm_peak_gbs": pk, "rows": rows}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
