import json, sys
L = "/tmp/liborc_exp.so"
insts = {"tallA": ["lasso", [20000, 2000, 0.01, 0]], "tallB": ["lasso", [10000, 500, 0.1, 0]], "wide": ["lasso", [1000, 10000, 0.001, 0]]}
vars_ = {"default": (0, {}), "om1": (0, {"omega0": 1.0}), "fpr": (1, {}), "fpr_om1": (1, {"omega0": 1.0}),
         "step": (16, {}), "step_om1": (16, {"omega0": 1.0}), "fpr_step_om1": (17, {"omega0": 1.0}),
         "fpr_step_om1_b1": (17, {"omega0": 1.0, "refl_window": 10**9}), "fpr_om1_b1": (1, {"omega0": 1.0, "refl_window": 10**9})}
sel = sys.argv[1].split(",") if len(sys.argv) > 1 else list(vars_)
out = []
for iname, inst in insts.items():
    for vn in sel:
        v, kw = vars_[vn]
        out.append({"name": vn, "lib": L, "inst": inst, "var": v, "kw": kw, "iters": 20000})
print(json.dumps(out))
