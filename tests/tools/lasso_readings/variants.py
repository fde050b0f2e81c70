import sys, json, multiprocessing as mp
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", ".."))
from probe import run, use_lib
from instances import gen_lasso, gen_fisher, gen_mpo, gen_mixed
def job(args):
    name, lib, inst, kw, iters, var = args
    import os; os.environ['ORC_VARIANT'] = str(var)
    if lib: use_lib(lib)
    kind, a = inst
    prog = {"lasso": gen_lasso, "fisher": gen_fisher, "mpo": gen_mpo, "mixed": gen_mixed}[kind](*a)
    done, h, t = run(prog, iters, **kw)
    return name, inst, done, h[1], int(h[2]), round(t, 1)
if __name__ == "__main__":
    spec = json.loads(sys.argv[1])
    jobs = [(s["name"], s.get("lib"), tuple(s["inst"]), s.get("kw", {}), s.get("iters", 20000), s.get("var", 0)) for s in spec]
    with mp.Pool(8, maxtasksperchild=1) as p:
        for r in p.imap_unordered(job, jobs):
            print(r, flush=True)
