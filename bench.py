#!/usr/bin/env python
"""bench.py — PDCS hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl cuda|reference]

A "step" is one accepted inner iteration of Alg. 1: the PDHG
trial(s) with line search, the reflected-Halpern update, averaging, and the
amortised Eq. 9 check / restart logic every check_interval iterations.  The
workload is BASELINE.json configs[1]: Lasso SOCP, 1e6 samples x 1e4 features,
A 1% dense (K: 1,000,001 x 1,020,002, nnz 2.01e8), seeded synthetic data.

value          iterations/s over all ranks (device-timed with CUDA events on the
               library's stream, inputs resident in HBM)
e2e            iterations/s of the whole job through the C ABI with pinned HOST
               buffers: pdcs_create (H2D upload, transpose) + pdcs_set_cones
               (Ruiz/PC) + pdcs_iterate(K) + pdcs_get_iterate (D2H)
roofline       dominant kernel: algorithmic bytes per launch / mean launch time
cpu_baseline   the CPU oracle (single thread) on a bounded sample of the same job
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PDHG iters/sec & time-to-1e-4 rel KKT; SpMV HBM GB/s vs peak, 1-8 GPUs"
FALLBACK_HBM = 6650.0


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([s.strip() for s in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 5 + i and r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


DATA = {
    "lasso": "synthetic (seeded Philox, PAPER.md:1663 recipe at BASELINE configs[1] size)",
    "tiny_lasso": "synthetic (seeded Philox, PAPER.md:1663 recipe at BASELINE configs[0] size)",
    "fisher": "synthetic (seeded Philox, PAPER.md:1618-1623 recipe at BASELINE configs[2] size)",
    "mpo": "synthetic (seeded Philox, PAPER.md:1694-1705 with synthetic covariances, reading A24, BASELINE configs[3])",
    "mixed": "synthetic (seeded Philox, SURVEY 8(d) cfg 5 planted mixed-cone recipe, one GPU's 1/8 share of BASELINE configs[4])",
    "mixed_full": "synthetic (seeded Philox streams per row chunk, SURVEY 8(d) cfg 5 planted mixed-cone recipe at "
                  "BASELINE configs[4]'s size, generated rank-locally)",
}


def build_instance(config, seed):
    from instances import CONFIGS
    t = time.perf_counter()
    prog = CONFIGS[config](seed)
    return prog, time.perf_counter() - t


def build_shard(args, rank, world, allreduce):
    """configs[4] at its stated size (--config mixed_full, --scale 1.0: m 2e7,
    n 1e7, nnz 2e9), generated rank-locally: every rank draws only its rows
    (instances.gen_mixed_shard); c's G^T y* partials are all-reduced."""
    from instances import mixed_full_layout, gen_mixed_shard
    from paper_2505_00311_b200 import dist as D
    t = time.perf_counter()
    L = mixed_full_layout(args.scale, args.seed)
    rows = D.partition_rows(L.row_ptr, L.rk, L.rdim, world)[rank]
    prog = gen_mixed_shard(L, rows, allreduce=allreduce)
    prog.nnz_total = int(L.row_ptr[-1])
    return prog, rows, time.perf_counter() - t


def local_rows(prog):
    return prog.rows[1] - prog.rows[0] if hasattr(prog, "rows") else prog.m


def spmv_alg_bytes(prog):
    """Algorithmic bytes of the two fused SpMV kernels per launch:
    matrix (8 B value + 4 B column id per nnz) + row pointers (4 B per row) + the
    gathered vector once + the row-indexed epilogue vectors."""
    nnz, m, n = prog.nnz, local_rows(prog), prog.n
    # K sweep: x^ gathered once (8 n); y, h~, carried K x in, K x^, y^ out (40 m); kind byte (m)
    k_dual = 12 * nnz + 4 * (m + 1) + 8 * n + 40 * m + m
    # K^T sweep: y+ gathered once (8 m); x^, x, x0, xsum in, x, K^T y, xsum out (56 n)
    kt_halpern = 12 * nnz + 4 * (n + 1) + 8 * m + 56 * n
    return {"spmv_K_dual": k_dual, "spmv_KT_halpern": kt_halpern}


def elem_alg_bytes(prog):
    """Algorithmic bytes of the two fused elementwise update kernels per launch.
    k_primal_elem over the box / zero / R+ coordinates: kind byte, x, c~, K~^T y
    in; x^ out (33 B), plus 8 B per bound the kernel reads: a box column
    [0, inf) is the kind EK_LO0 and reads none (its bound is in the kind byte),
    every other finite l~ / u~ is one 8-B read.
    k_halpern_y over all rows: y^, y, y0, sum(eta y) in, y+, sum out; the
    carried K x^, K x, K x0 in, K x+ out (80 B)."""
    from instances import ZERO, NONNEG
    pk, pdim = np.asarray(prog.pk), np.asarray(prog.pdim)
    n_elem = prog.n1 + int(pdim[(pk == ZERO) | (pk == NONNEG)].sum())
    l, u = np.asarray(prog.l), np.asarray(prog.u)
    lo0 = (l == 0.0) & ~np.isfinite(u)
    bounds = 8 * int((np.isfinite(l) & ~lo0).sum() + np.isfinite(u).sum())
    return {"primal_elem": 33 * n_elem + bounds, "halpern_y": 80 * local_rows(prog)}


# kernels that run only inside the Eq. 9 check (every check_interval iterations);
# the projection block kernels of the average candidate are not separable by name
CHECK_KERNELS = ("avg_elem", "tiled_check_partial", "check_combine", "spmv_store", "kkt_rows",
                 "kkt_cols", "kkt_reduce", "kkt_decide", "restart_copy")


def round_up(k, q):
    return max(q, ((k + q - 1) // q) * q)


def iter_alg_bytes(prog):
    """SURVEY §8(d) B_iter = [12 nnz + 4(m+1)] + [12 nnz + 4(n+1)] + 8*14*(m+n)."""
    nnz, m, n = prog.nnz, local_rows(prog), prog.n
    return 12 * nnz + 4 * (m + 1) + 12 * nnz + 4 * (n + 1) + 8 * 14 * (m + n)


def pinned(prog, rows):
    """Pinned host copies of this rank's shard (rows [a, b)) and the replicated data."""
    import torch
    from paper_2505_00311_b200 import dist as D
    sh = D.shard(prog, *rows)
    def pin(a, dt):
        return torch.from_numpy(np.ascontiguousarray(a, dt)).pin_memory()
    return dict(row_ptr=pin(sh["row_ptr"], np.int64), col=pin(sh["col"], np.int32),
                val=pin(sh["val"], np.float64), c=pin(prog.c, np.float64), h=pin(sh["h"], np.float64),
                l=pin(prog.l, np.float64), u=pin(prog.u, np.float64))


def literal_form_kkt(P, prog, xb, yb, stream, device):
    """Lasso (reading P9): the solve ran on the balanced SOCP; its best point,
    mapped back by w = w'/S, r = S r', is scored by Eq. 9 OF THE LITERAL FORM
    (PAPER.md:1641-1659 as printed) -- in a second library context, on the GPU."""
    import torch
    lit = prog.literal()
    host = pinned(lit, (0, lit.m))
    ctx = make_ctx(P, lit, host, P.pdcs_default_params(), stream, device, (0, lit.m))
    x = torch.from_numpy(prog.to_literal(xb.numpy()))
    P.pdcs_set_iterate(ctx, x, yb)
    k = P.pdcs_kkt(ctx, P.CURRENT)
    P.pdcs_destroy(ctx)
    return {"S": prog.lasso_S, "err_p": k.err_p, "err_d": k.err_d, "err_gap": k.err_gap,
            "kkt_max": max(k.err_p, k.err_d, k.err_gap), "pobj": k.pobj,
            "note": "best point of the balanced solve mapped to the literal SOCP (w = w'/S, r = S r'), "
                    "Eq. 9 of the literal form"}


def make_ctx(P, prog, host, params, stream, device, rows, uid=None, rank=0, world=1):
    idbuf = None if uid is None else np.frombuffer(uid, dtype=np.uint8).copy()
    ctx = P.pdcs_create(prog.m, prog.n, prog.n1, rows[0], rows[1], host["row_ptr"], host["col"],
                        host["val"], host["c"], host["h"], host["l"], host["u"], params, device, stream,
                        nccl_unique_id=idbuf, rank=rank, world=world)
    P.pdcs_set_cones(ctx, prog.pk, prog.pdim, prog.rk, prog.rdim)
    return ctx


def cpu_baseline(prog, budget_s=20.0):
    """Oracle (single-threaded C++, as it stands) on the same instance: timed
    accepted iterations after one warm-up iteration; setup excluded.  For
    configs[4] at full size (2e9 nnz) the oracle runs the same recipe at 1/64
    scale and its it/s is extrapolated per nonzero (SURVEY §8(d) cfg 5)."""
    import oracle as O
    if getattr(prog, "nnz_total", None):
        from instances import mixed_full_layout, gen_mixed_shard
        L = mixed_full_layout(1.0 / 64, 0)
        small = gen_mixed_shard(L, (0, L.m))
        r = cpu_baseline(small, budget_s)
        f = small.nnz / prog.nnz_total
        r["value"] *= f
        r["sample"] += f"; it/s extrapolated to the full instance per nonzero (x {f:.5f})"
        return r
    t = time.perf_counter()
    S = O.OracleSolver(prog)
    setup = time.perf_counter() - t
    S.iterate(1)
    done, t0 = 0, time.perf_counter()
    while True:
        S.iterate(1)
        done += 1
        el = time.perf_counter() - t0
        if el >= budget_s or done >= 200:
            break
    return {"value": done / el, "unit": "iter/s", "cores": 1, "kind": "oracle",
            "sample": f"{done} accepted iterations of the full {prog.name} instance after 1 warm-up "
                      f"(setup {setup:.1f}s excluded), single thread",
            "host_cpu": _cpu_model(), "nproc": os.cpu_count()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def run_reference(args):
    rank, local, world = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        if rank != 0:
            dist.barrier()
            return
    extrap = 1.0
    if args.config == "mixed_full":         # the oracle on the 1/64-scale recipe, per-nnz extrapolation
        from instances import mixed_full_layout, gen_mixed_shard
        L = mixed_full_layout(args.scale / 64, args.seed)
        prog, gen_s = gen_mixed_shard(L, (0, L.m)), 0.0
        extrap = prog.nnz / float(mixed_full_layout(args.scale, args.seed).row_ptr[-1])
    else:
        prog, gen_s = build_instance(args.config, args.seed)
    import oracle as O
    t = time.perf_counter()
    S = O.OracleSolver(prog)
    setup = time.perf_counter() - t
    S.iterate(min(max(args.warmup, 0), 2))
    # bounded sample: the timed steps stop after REF_BUDGET_S seconds
    budget = float(os.environ.get("REF_BUDGET_S", "90"))
    done, t0 = 0, time.perf_counter()
    while done < args.steps:
        S.iterate(1)
        done += 1
        if time.perf_counter() - t0 > budget:
            break
    el = time.perf_counter() - t0
    v = done / el * extrap
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "iter/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / done,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": _config(prog, args),
            "cpu_baseline": {"value": v, "unit": "iter/s", "kind": "oracle", "cores": 1,
                             "sample": f"{done} of {args.steps} requested accepted iterations of the full "
                                       f"{prog.name} instance (time-capped at {budget:.0f}s) after "
                                       f"{min(max(args.warmup, 0), 2)} warm-up; setup {setup:.1f}s excluded"
                                       + (f"; 1/64-scale recipe, it/s x {extrap:.5f} per nonzero"
                                          if extrap != 1.0 else "")},
            "e2e": {"value": v, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def _config(prog, args):
    return {"workload": args.config, "instance": prog.name, "m": prog.m, "n": prog.n,
            "nnz": getattr(prog, "nnz_total", None) or prog.nnz, "nnz_this_rank": prog.nnz,
            "cones": {"primal": [int(k) for k in np.unique(prog.pk)], "rows": [int(k) for k in np.unique(prog.rk)]},
            "l2": "inputs larger than L2 (matrix %.2f GB > 126 MB)" % (24 * prog.nnz / 1e9),
            "parallelism": f"rows-sharded-x{args.gpus} (NCCL all-reduce, replicated primal)" if args.gpus > 1
            else "single-gpu"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--config", default="lasso")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--scale", type=float, default=1.0, help="mixed_full: fraction of configs[4]'s size")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tol-run", action="store_true")
    ap.add_argument("--tol-time-limit", type=float, default=120.0)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    rank, local, world = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    from paper_2505_00311_b200 import build
    build.build()
    import paper_2505_00311_b200 as P

    from paper_2505_00311_b200 import dist as D
    if args.config == "mixed_full":
        def allreduce(a):
            if world == 1:
                return a
            t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
            torch.distributed.all_reduce(t)
            return t.cpu().numpy()
        prog, rows, gen_s = build_shard(args, rank, world, allreduce)
    else:
        prog, gen_s = build_instance(args.config, args.seed)
        rows = D.partition_rows(prog.row_ptr, prog.rk, prog.rdim, world)[rank]
    uid = None
    if world > 1:
        # rank 0 creates the ncclUniqueId, torch.distributed broadcasts it
        buf = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            buf.copy_(torch.frombuffer(bytearray(P.pdcs_nccl_unique_id()), dtype=torch.uint8))
        torch.distributed.broadcast(buf, 0)
        uid = bytes(buf.cpu().numpy().tobytes())
    host = pinned(prog, rows)
    stream = torch.cuda.Stream()
    sh = stream.cuda_stream
    params = P.pdcs_default_params()
    mk = lambda prm: make_ctx(P, prog, host, prm, sh, local, rows, uid, rank, world)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    # ---------------- device-timed steps (inputs resident in HBM).  The timed
    # window starts on an Eq. 9 check boundary and holds whole check intervals
    # (checks fall every check_interval accepted iterations, restarts only at
    # checks), so the amortised check is inside the per-step time.
    ci = int(params.check_interval)
    steps = round_up(args.steps, ci)
    warmup = round_up(max(args.warmup, 3), ci)
    ctx = mk(params)
    P.pdcs_iterate(ctx, warmup)
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        res = P.pdcs_iterate(ctx, steps)             # CUDA-graph path: one launch per iteration
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = ev0.elapsed_time(ev1)
    launches = P.pdcs_launch_count(ctx)
    # per-kernel CUDA-event timing over a second timed region of the same length
    # (host-driven launches with an event pair around every kernel)
    P.pdcs_enable_timing(ctx, True)
    torch.cuda.synchronize()
    evk0, evk1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    evk0.record(stream)
    P.pdcs_iterate(ctx, steps)
    evk1.record(stream)
    torch.cuda.synchronize()
    ms_timed_pass = evk0.elapsed_time(evk1)
    ktimes = P.pdcs_kernel_times(ctx)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / steps
    value = steps / (ms / 1e3)               # iterations of the (one, row-sharded) problem per second
    P.pdcs_destroy(ctx)

    # ---------------- roofline of the dominant kernel (an SpMV sweep = its
    # partial kernel + the combine/epilogue kernel on the tiled path)
    peak, peak_src = load_peaks()
    algb = spmv_alg_bytes(prog)
    groups = {"spmv_K_dual": ["spmv_K_dual", "tiled_K_partial", "panel_K_partial", "tiled_K_wide_combine"],
              "spmv_KT_halpern": ["spmv_KT_halpern", "tiled_KT_partial", "panel_KT_partial",
                                  "tiled_KT_wide_combine"]}
    sweeps = {}
    for name, parts in groups.items():
        if name in ktimes:
            sweeps[name] = (sum(ktimes[p][0] for p in parts if p in ktimes), ktimes[name][1],
                            [p for p in parts if p in ktimes])
    dom = max(sweeps, key=lambda k: sweeps[k][0]) if sweeps else None
    roof = None
    if dom:
        tot_ms, cnt, parts = sweeps[dom]
        avg_s = tot_ms / cnt / 1e3
        ach = algb[dom] / avg_s / 1e9
        traffic, traffic_src = None, None
        tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tf):
            tj = json.load(open(tf))
            traffic = tj.get(args.config, {}).get(dom)
            traffic_src = f"profiles/ncu_traffic.json (tools/ncu_traffic.py, measured at commit {tj.get('_commit', '?')})"
        roof = {"bound": "hbm", "kernel": dom, "kernels_timed": parts, "achieved": ach, "peak": peak,
                "unit": "GB/s", "frac": ach / peak, "traffic": traffic, "traffic_source": traffic_src,
                "alg_bytes_per_launch": algb[dom],
                "avg_launch_ms": avg_s * 1e3, "launches": cnt, "peak_source": peak_src,
                "other_sweep": {k: {"GB/s": algb[k] / (v[0] / v[1] / 1e3) / 1e9,
                                    "frac": algb[k] / (v[0] / v[1] / 1e3) / 1e9 / peak}
                                for k, v in sweeps.items() if k != dom},
                "fused_update": {k: {"GB/s": b / (ktimes[k][0] / ktimes[k][1] / 1e3) / 1e9,
                                     "frac": b / (ktimes[k][0] / ktimes[k][1] / 1e3) / 1e9 / peak,
                                     "alg_bytes_per_launch": b}
                                 for k, b in elem_alg_bytes(prog).items() if k in ktimes and b > 0}}
    total_kernel_ms = sum(v[0] for v in ktimes.values())
    iter_bytes = iter_alg_bytes(prog)

    # ---------------- e2e through the C ABI with pinned host buffers
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    ctx = mk(params)
    P.pdcs_iterate(ctx, steps)
    xo = torch.empty(prog.n, dtype=torch.float64).pin_memory()
    yo = torch.empty(rows[1] - rows[0], dtype=torch.float64).pin_memory()
    P.pdcs_get_iterate(ctx, P.CURRENT, P.ORIGINAL, xo, yo)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    P.pdcs_destroy(ctx)
    h2d = sum(int(t.numel() * t.element_size()) for t in host.values())
    d2h = (prog.n + rows[1] - rows[0]) * 8
    e2e = {"value": steps / e2e_s, "unit": "iter/s",
           "h2d_bytes_per_step": h2d / steps, "d2h_bytes_per_step": d2h / steps,
           "seconds": e2e_s, "note": "create+set_cones (upload, transpose, Ruiz) + iterate(K) + D2H of (x, y)"}

    # ---------------- time to 1e-4 relative KKT (Eq. 9), fresh context
    tol_run = None
    if not args.no_tol_run:
        p4 = P.pdcs_default_params(tol=1e-4, time_limit_s=args.tol_time_limit)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx = mk(p4)
        torch.cuda.synchronize()
        t_setup = time.perf_counter() - t0
        r = P.pdcs_solve(ctx)
        torch.cuda.synchronize()
        t_all = time.perf_counter() - t0
        xb = yb = None
        if hasattr(prog, "literal") and world == 1:
            xb = torch.empty(prog.n, dtype=torch.float64)
            yb = torch.empty(prog.m, dtype=torch.float64)
            P.pdcs_get_iterate(ctx, P.BEST, P.ORIGINAL, xb, yb)
        P.pdcs_destroy(ctx)
        tol_run = {"tol": 1e-4, "status": r.status, "seconds_incl_setup": t_all,
                   "seconds_solve": r.solve_seconds, "setup_seconds": t_setup, "iters": r.iters,
                   "kkt_max": max(r.kkt.err_p, r.kkt.err_d, r.kkt.err_gap), "restarts": r.restarts}
        if xb is not None:
            tol_run["literal_form"] = literal_form_kkt(P, prog, xb, yb, sh, local)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(prog)

    if rank == 0:
        check_ms = sum(v[0] for k, v in ktimes.items() if k in CHECK_KERNELS)
        line = {"metric": METRIC, "value": value, "unit": "iter/s", "n_gpus": world, "steps": steps,
                "warmup": warmup, "steps_requested": args.steps, "warmup_requested": args.warmup,
                "window": f"{steps // ci} whole check intervals of {ci} accepted iterations, starting on a "
                          f"check boundary (requested --steps/--warmup rounded up)",
                "check_share": check_ms / total_kernel_ms if total_kernel_ms else None,
                "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": DATA.get(args.config, "synthetic (seeded Philox)"),
                "config": _config(prog, args), "clocks": clk.summary(), "e2e": e2e,
                "gpu_launches": launches, "roofline": roof, "cpu_baseline": cpu,
                "time_to_1e-4": tol_run,
                "iter_roofline": {"alg_bytes_per_iter": iter_bytes,
                                  "achieved_GBs": iter_bytes / (ms_per_step / 1e3) / 1e9,
                                  "frac": iter_bytes / (ms_per_step / 1e3) / 1e9 / peak},
                "kernel_ms_per_step": {k: v[0] / steps for k, v in sorted(ktimes.items())},
                "kernel_timing_pass_ms_per_step": ms_timed_pass / steps,
                "kernel_share": {k: v[0] / total_kernel_ms for k, v in sorted(ktimes.items())},
                "final": {"iters": res.iters, "restarts": res.restarts, "trials": res.trials},
                "instance_gen_s": gen_s}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
