"""Test-side tools (they run the CPU oracle, which only tests/, smoke() and
bench.py's cpu_baseline may execute): mutation check of the oracle pins,
projection sweeps against the oracle, shadow-parity debugging."""
