exec(open(os.path.join(HERE, "patch128.py")).read())
old = "    for (int64_t j = 0; j < n; ++j) x[j] = a * ((1.0 + beta) * xh[j] - beta * x[j]) + b * x0[j];\n    for (int64_t i = 0; i < m; ++i) y[i] = a * ((1.0 + beta) * yh[i] - beta * y[i]) + b * y0[i];"
assert old in s
s = s.replace(old, "    if (g_var & 256) { x = xh; y = yh; } else {\n" + old + "\n    }")
