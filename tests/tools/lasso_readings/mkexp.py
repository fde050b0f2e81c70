"""Experimental copy of the oracle with switchable readings (Lasso convergence
study, DESIGN.md §8 / profiles/r2_lasso_readings.txt).  NOT the oracle: it
patches a copy of oracle/pdcs_oracle.cpp into orc_exp.cpp, selected at run
time by ORC_VARIANT bits:
   1 restart rule on the fixed-point residual ||z^ - z||_omega (r2HPDHG style)
   4 'current' restart candidate = P(z^{t,k+1}) instead of z^ (reading A10 alternative)
   8 no average candidate
  16 PDLP step rule eta' = min((1-(k+2)^-0.3) eta_bar, (1+(k+2)^-0.6) eta)
  32 objective / right-hand-side rescaling by 1 + ||c~||_2, 1 + ||h~||_2 (patch32.py)
  64 primal weight never updated (patch64.py)
 128 omega0 = ||c~||_2 / ||h~||_2 (patch128.py)
usage: python mkexp.py [patchNN.py]; g++ -O2 -shared -fPIC -o /tmp/liborc_exp.so orc_exp.cpp
"""
import os
HERE = os.path.dirname(os.path.abspath(__file__))
s = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "..", "oracle", "pdcs_oracle.cpp")).read()
s = s.replace("static int64_t g_rootfail = 0;", "static int64_t g_rootfail = 0;\nstatic int g_var = getenv(\"ORC_VARIANT\") ? atoi(getenv(\"ORC_VARIANT\")) : 0;")
old = "    beta = reflection_beta(k, prm.refl_window, std::sqrt(num), &r_start, beta);"
assert old in s
s = s.replace(old, "    if (k == 0) { fpr0 = std::sqrt(num); }\n    fpr_last = std::sqrt(num);\n" + old)
s = s.replace("  double r_start = 0.0, e_anchor = 0.0, e_prev = -1.0;", "  double r_start = 0.0, e_anchor = 0.0, e_prev = -1.0, fpr0 = -1, fpr_last = -1, fpr_prev = -1;")
old = """    bool restart = restart_rule(e, e_anchor, e_prev, k, total, prm.restart_suff, prm.restart_nec,
                                prm.restart_art);"""
new = """    bool restart = (g_var & 1) ? restart_rule(fpr_last, fpr0, fpr_prev, k, total, prm.restart_suff, prm.restart_nec, prm.restart_art)
                               : restart_rule(e, e_anchor, e_prev, k, total, prm.restart_suff, prm.restart_nec,
                                prm.restart_art);
    fpr_prev = fpr_last;
    if (restart) fpr_prev = -1;"""
assert old in s; s = s.replace(old, new)
old = "    Kkt kc = kkt(xh.data(), yh.data());\n    vector<double> xa(n), ya(m);"
new = """    vector<double> xpz = x, ypz = y;
    if (g_var & 4) { proj_X(xpz.data()); proj_Y(ypz.data()); }
    const vector<double>& xcur = (g_var & 4) ? xpz : xh;
    const vector<double>& ycur = (g_var & 4) ? ypz : yh;
    Kkt kc = kkt(xcur.data(), ycur.data());
    vector<double> xa(n), ya(m);"""
assert old in s; s = s.replace(old, new)
s = s.replace("    bool use_avg = candidate_is_average(ec, ea);", "    bool use_avg = (g_var & 8) ? false : candidate_is_average(ec, ea);")
old = "    const vector<double>& xc = use_avg ? xa : xh;\n    const vector<double>& yc = use_avg ? ya : yh;"
assert old in s
s = s.replace(old, "    const vector<double>& xc = use_avg ? xa : xcur;\n    const vector<double>& yc = use_avg ? ya : ycur;")
old = "        eta = std::min(prm.ls_grow * eta, etabar);"
new = """        if (g_var & 16) eta = std::min((1.0 - std::pow((double)(total + 2), -0.3)) * etabar, (1.0 + std::pow((double)(total + 2), -0.6)) * eta);
        else eta = std::min(prm.ls_grow * eta, etabar);"""
assert old in s; s = s.replace(old, new)
import sys
extra = sys.argv[1] if len(sys.argv) > 1 else None
if extra: exec(open(extra).read())
open(os.path.join(HERE, "orc_exp.cpp"), "w").write(s)
