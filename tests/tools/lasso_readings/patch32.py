s = s.replace("    for (int64_t j = 0; j < n; ++j) xo[j] = xs[j] / q[j];\n    for (int64_t i = 0; i < m; ++i) yo[i] = ys[i] / r[i];",
 "    for (int64_t j = 0; j < n; ++j) xo[j] = xs[j] * sh_ / q[j];\n    for (int64_t i = 0; i < m; ++i) yo[i] = ys[i] * sc_ / r[i];")
s = s.replace("    for (int64_t j = 0; j < n; ++j) ct[j] = P.c[j] / q[j];\n    for (int64_t i = 0; i < m; ++i) ht[i] = P.h[i] / r[i];\n    for (int64_t j = 0; j < P.n1; ++j) { lt[j] = q[j] * P.l[j]; ut[j] = q[j] * P.u[j]; }",
"""    if (g_var & 32) {
      double a = 0, b = 0;
      for (int64_t j = 0; j < n; ++j) { double v = P.c[j] / q[j]; a += v * v; }
      for (int64_t i = 0; i < m; ++i) { double v = P.h[i] / r[i]; b += v * v; }
      sc_ = 1.0 + std::sqrt(a); sh_ = 1.0 + std::sqrt(b);
    }
    for (int64_t j = 0; j < n; ++j) ct[j] = P.c[j] / q[j] / sc_;
    for (int64_t i = 0; i < m; ++i) ht[i] = P.h[i] / r[i] / sh_;
    for (int64_t j = 0; j < P.n1; ++j) { lt[j] = q[j] * P.l[j] / sh_; ut[j] = q[j] * P.u[j] / sh_; }""")
s = s.replace("  double r_start = 0.0, e_anchor = 0.0, e_prev = -1.0,", "  double sc_ = 1.0, sh_ = 1.0;\n  double r_start = 0.0, e_anchor = 0.0, e_prev = -1.0,")
