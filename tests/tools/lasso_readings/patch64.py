exec(open(os.path.join(HERE, "patch32.py")).read())
old = "      omega = primal_weight(dxn, dyn, omega);"
assert old in s
s = s.replace(old, "      if (!(g_var & 64)) omega = primal_weight(dxn, dyn, omega);")
