"""Mutation check of the oracle pins: apply each plausible slip to a copy of the
oracle, run the -m "not gpu" pin suites, and report which test kills it.
Usage: python tests/tools/oracle_mutants.py [NAME ...]  (copies the repo under $TMPDIR)."""
import os, shutil, subprocess, sys, tempfile
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
WORK = tempfile.mkdtemp(prefix="oracle_mutants_")
from concurrent.futures import ThreadPoolExecutor
MUTS = {
 "geomean_arith": ("double g = std::sqrt(q[a] * q[a + 1]);", "double g = 0.5 * (q[a] + q[a + 1]);"),
 "pc_infnorm": ("        rm[i] += a;", "        rm[i] = std::max(rm[i], a);"),
 "beta_on_decrease": ("res > *r_start", "res < *r_start"),
 "tie_strict": ("return e_average <= e_current;", "return e_average < e_current;"),
 "avg_grown_eta": ("for (int64_t j = 0; j < n; ++j) xsum[j] += eta_used * x[j];", "for (int64_t j = 0; j < n; ++j) xsum[j] += eta * x[j];"),
 "errd_den": ("double den_d = 1.0 + std::max(nrminf(P.c.data(), n), nrminf(Gty.data(), n));", "double den_d = 1.0 + nrminf(P.c.data(), n);"),
 "errgap_den": ("(1.0 + std::max(std::fabs(pobj), std::fabs(dobj)))", "(1.0 + std::fabs(pobj))"),
 "eta0_max": ("for (int64_t p = K.ptr[i]; p < K.ptr[i + 1]; ++p) s += std::fabs(K.val[p]);", "for (int64_t p = K.ptr[i]; p < K.ptr[i + 1]; ++p) s = std::max(s, std::fabs(K.val[p]));"),
 "omega0_inv": ("omega = std::min(std::max(cn / hn, 1e-4), 1e4);", "omega = std::min(std::max(hn / cn, 1e-4), 1e4);"),
 "power_nosqrt": ("return std::sqrt(lam);", "return lam;"),
 "omega_swap": ("omega = primal_weight(dxn, dyn, omega);", "omega = primal_weight(dyn, dxn, omega);"),
 "dobj_sign": ("if (fu) dual_obj_box -= P.u[j]", "if (fu) dual_obj_box += P.u[j]"),
 "window_sliding": ("if (k % W == W - 1 && res > *r_start) beta *= 0.5;", "if (k >= W - 1 && res > *r_start) beta *= 0.5;"),
}
def one(name):
    src, dst = MUTS[name]
    d = os.path.join(WORK, name)
    shutil.rmtree(d, ignore_errors=True)
    shutil.copytree(ROOT, d, ignore=shutil.ignore_patterns(".git", "gpurun_out", "*.so", "profiles"))
    p = f"{d}/oracle/pdcs_oracle.cpp"
    s = open(p).read()
    assert s.count(src) >= 1, name
    s = s.replace(src, dst)
    open(p, "w").write(s)
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "not gpu", "tests/test_oracle_pins.py", "tests/test_oracle_rule_pins.py"], cwd=d, capture_output=True, text=True)
    tail = [l for l in r.stdout.splitlines() if l.startswith("FAILED")]
    return name, r.returncode, tail[:1]
with ThreadPoolExecutor(4) as ex:
    for res in ex.map(one, sys.argv[1:] or list(MUTS)):
        print(res, flush=True)
