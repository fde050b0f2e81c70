import sys, time, ctypes as C, numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", ".."))
import oracle as O
from instances import gen_lasso
def use_lib(path):
    L = C.CDLL(path); O._declare(L); O._lib = L
    return L
def run(prog, iters, chunk=40, verbose=False, **kw):
    S = O.OracleSolver(prog, **kw)
    t0 = time.time(); hist = []
    done = 0
    while done < iters:
        S.iterate(chunk); done += chunk
        sc = S.scalars()
        e = min(max(sc["cur_err_p"], sc["cur_err_d"], sc["cur_err_gap"]), max(sc["avg_err_p"], sc["avg_err_d"], sc["avg_err_gap"]))
        hist.append((done, sc["best_e"], sc["restarts"], sc["omega"], sc["beta"], sc["eta"]))
        if verbose and done % (chunk*25) == 0:
            print(done, "best %.2e cur(%.1e %.1e %.1e) avg(%.1e %.1e %.1e) rs %d om %.3g beta %.3g eta %.3g" % (
                sc["best_e"], sc["cur_err_p"], sc["cur_err_d"], sc["cur_err_gap"], sc["avg_err_p"], sc["avg_err_d"], sc["avg_err_gap"], sc["restarts"], sc["omega"], sc["beta"], sc["eta"]), flush=True)
        if sc["best_e"] <= float(__import__("os").environ.get("TARGET", "1e-4")): break
    return done, hist[-1], time.time()-t0
if __name__ == "__main__":
    m, nf, d = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
    prog = gen_lasso(m, nf, d, seed=0)
    print(prog.name, prog.m, prog.n, len(prog.vals))
    print(run(prog, int(sys.argv[4]), verbose=True))
