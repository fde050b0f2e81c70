exec(open(os.path.join(HERE, "patch64.py")).read())
old = "      else if (cn > 0.0 && hn > 0.0) omega = std::min(std::max(cn / hn, 1e-4), 1e4);"
assert old in s
s = s.replace(old, """      else if ((g_var & 128) && cn > 0.0 && hn > 0.0) {
        double c2 = 0, h2 = 0;
        for (int64_t j = 0; j < n; ++j) c2 += ct[j] * ct[j];
        for (int64_t i = 0; i < m; ++i) h2 += ht[i] * ht[i];
        omega = std::sqrt(c2) / std::sqrt(h2);
      }
      else if (cn > 0.0 && hn > 0.0) omega = std::min(std::max(cn / hn, 1e-4), 1e4);""")
