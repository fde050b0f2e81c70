"""DRAM traffic of the dominant sweeps at HEAD (bench.py's roofline "traffic").

    python tools/ncu_traffic.py run  --config lasso [--config fisher ...]
        runs ncu (dram__bytes_read/write.sum, gpu__time_duration.sum) over the
        iteration phase of the bench instance (NVTX range "iterate"; setup and
        autotune excluded) and writes profiles/ncu_traffic.json stamped with the
        commit it measured;
    python tools/ncu_traffic.py parse --config lasso --commit HASH
        re-reads gpurun_out/traffic_<config>.csv of an earlier run;
    python tools/ncu_traffic.py drive --config lasso
        the driver ncu profiles (host-driven loop, so every kernel is a launch).

Per sweep = partial + combine kernel of the tiled path, or the one CSR kernel;
traffic per launch = mean over the captured launches of read + write bytes.
The SpMV format is the one the bench's setup autotune keeps (forced here,
because ncu serialises the tiled path's two kernels and distorts the autotune).
"""
import argparse
import csv
import datetime
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# the format the bench's autotune keeps per config
TILED = {"lasso": "1", "fisher": "0", "mpo": "0", "mixed": "0"}
SWEEPS = {"spmv_K_dual": ("k_tiled_sliced<2>", "k_tiled_sliced<2,", "k_tiled_sliced<(int)2,", "k_tiled_sliced<1,",
                          "k_tiled_sliced<(int)1,", "k_tiled_tma<2>", "k_tiled_partial<2>",
                          "k_tiled_combine<EpiDualTrial", "spmv_kernel<EpiDualTrial>"),
          "spmv_KT_halpern": ("k_tiled_sliced<1>", "k_tiled_sliced<1,", "k_tiled_sliced<(int)1,", "k_tiled_tma<1>", "k_tiled_partial<1>",
                              "k_tiled_combine<EpiHalpernX", "spmv_kernel<EpiHalpernX>"),
          "halpern_y": ("k_halpern_y",), "primal_elem": ("k_primal_elem",)}


def drive(config, iters):
    import torch
    import paper_2505_00311_b200 as P
    from instances import CONFIGS
    prog = CONFIGS[config](0)
    g = P.PdcsSolver(prog)
    g.iterate(3)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("iterate")
    g.iterate(iters)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    print("done", prog.name, prog.m, prog.n, prog.nnz)


def run(configs, iters, out, parse_only=False, commit=None):
    res = {}
    head = commit or os.environ.get("PDCS_COMMIT") or subprocess.run(
        ["git", "rev-parse", "--short=12", "HEAD"], cwd=ROOT, capture_output=True, text=True).stdout.strip() \
        or "unknown"
    for cfg in configs:
        csvp = os.path.join(ROOT, "gpurun_out", f"traffic_{cfg}.csv")
        env = dict(os.environ, PDCS_NO_GRAPH="1", PDCS_TILED=TILED[cfg])
        cmd = ["ncu", "--nvtx", "--nvtx-include", "iterate/", "--clock-control", "none", "--csv",
               "--print-units", "base", "--metrics",
               "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
               "-k", "regex:k_tiled|spmv_kernel|k_halpern_y|k_primal_elem", "--log-file", csvp,
               sys.executable, os.path.abspath(__file__), "drive", "--config", cfg, "--iters", str(iters)]
        if not parse_only:
            subprocess.run(cmd, env=env, check=True)
        rows = [r for r in csv.reader(l for l in open(csvp) if not l.startswith("=="))]
        hdr = rows[0]
        ki, mi, vi, idi = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                           hdr.index("ID"))
        per = defaultdict(lambda: defaultdict(float))      # launch id -> metric -> value
        name = {}
        for r in rows[1:]:
            if len(r) <= vi:
                continue
            per[r[idi]][r[mi]] = float(r[vi].replace(",", ""))
            name[r[idi]] = r[ki]
        acc = defaultdict(lambda: [0.0, 0.0, 0])           # sweep part -> bytes, ns, launches
        # K's and K^T's tiled partials are the same kernel (single-element
        # tiles since the carried K x, DESIGN P6): a partial belongs to the
        # sweep of the next combine launch (EpiDualTrial: K, EpiHalpernX: K^T)
        ids = sorted(per, key=int)
        owner = {}
        for k, lid in enumerate(ids):
            if "k_tiled_sliced<" in name[lid] or "k_tiled_partial<" in name[lid] or "k_tiled_tma<" in name[lid]:
                for nxt in ids[k + 1:]:
                    if "k_tiled_combine<" in name[nxt]:
                        owner[lid] = "spmv_K_dual" if "EpiDualTrial" in name[nxt] else "spmv_KT_halpern"
                        break
        for lid, m in per.items():
            for sw, pats in SWEEPS.items():
                if lid in owner and owner[lid] != sw:
                    continue
                for pat in pats:
                    if pat in name[lid]:
                        a = acc[(sw, pat)]
                        a[0] += m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
                        a[1] += m["gpu__time_duration.sum"]
                        a[2] += 1
                        break
        cres = {}
        for sw in SWEEPS:
            parts = {pat: v for (s, pat), v in acc.items() if s == sw and v[2]}
            if parts:
                cres[sw] = sum(v[0] / v[2] for v in parts.values())
                cres[sw + "_parts"] = {pat: {"bytes_per_launch": v[0] / v[2], "ns_per_launch": v[1] / v[2],
                                             "launches": v[2]} for pat, v in parts.items()}
        res[cfg] = cres
    res["_commit"] = head
    res["_when"] = datetime.datetime.now(datetime.timezone.utc).strftime("%Y-%m-%dT%H:%MZ")
    res["_how"] = ("tools/ncu_traffic.py run: ncu --nvtx-include iterate/ (iteration phase only, host-driven "
                   "loop, the bench's SpMV format forced), dram__bytes_read.sum + dram__bytes_write.sum, "
                   "mean per launch, summed over a sweep's partial + combine kernels")
    old = {}
    if os.path.exists(out):
        old = json.load(open(out))
    old.update(res)
    json.dump(old, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["run", "drive", "parse"])
    ap.add_argument("--commit", default=None, help="commit the CSVs were measured at (parse)")
    ap.add_argument("--config", action="append")
    ap.add_argument("--iters", type=int, default=6)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "ncu_traffic.json"))
    a = ap.parse_args()
    cfgs = a.config or ["lasso"]
    if a.mode == "drive":
        drive(cfgs[0], a.iters)
    else:
        run(cfgs, a.iters, a.out, parse_only=a.mode == "parse", commit=a.commit)
