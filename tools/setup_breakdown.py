"""Setup-time breakdown of pdcs_create + pdcs_set_cones on a bench config
(pinned host buffers, as bench.py's e2e leg)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2505_00311_b200 as P
from paper_2505_00311_b200 import dist as D

cfg = sys.argv[1] if len(sys.argv) > 1 else "lasso"
prog, gen_s = bench.build_instance(cfg, 0)
rows = (0, prog.m)
host = bench.pinned(prog, rows)
st = torch.cuda.Stream()
for rep in range(int(os.environ.get('REPS', '2'))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx = bench.make_ctx(P, prog, host, P.pdcs_default_params(), st.cuda_stream, 0, rows)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    sc = P.pdcs_get_scalars(ctx)
    print(json.dumps({"config": cfg, "rep": rep, "wall_s": t1 - t0,
                      **{k: sc[k] for k in sc if k.startswith(("setup", "tiled", "tune"))}}), flush=True)
    ti = []
    for _ in range(2):                         # first: builds the CUDA graph
        t3 = time.perf_counter()
        P.pdcs_iterate(ctx, 40)
        torch.cuda.synchronize()
        ti.append(time.perf_counter() - t3)
    print(json.dumps({"iterate40_first_s": ti[0], "iterate40_second_s": ti[1]}), flush=True)
    t2 = time.perf_counter()
    P.pdcs_destroy(ctx)
    torch.cuda.synchronize()
    print(json.dumps({"destroy_s": time.perf_counter() - t2}), flush=True)
