"""Seeded synthetic conic-program generators (input data only, no method arithmetic).

Shared by the CPU oracle (tests, cpu baseline) and the CUDA path (tests, bench).
"""
from .program import (ConicProgram, ZERO, NONNEG, SOC, RSOC, EXP, DUAL_EXP,
                      KIND_NAMES, csr_from_coo)
from .generators import (gen_lasso, gen_fisher, gen_mpo, gen_mixed, gen_mixed_large, bernoulli_positions,
                         mixed_full_layout, gen_mixed_shard, MixedLayout, ShardedProgram)

# BASELINE.json configs (index -> builder).  configs[0] is the oracle-sized case.
CONFIGS = {
    "tiny_lasso": lambda seed=0: gen_lasso(100, 50, 1.0, seed=seed, dense=True),
    "lasso": lambda seed=0: gen_lasso(1_000_000, 10_000, 0.01, seed=seed),
    "fisher": lambda seed=0: gen_fisher(10_000, 1_000, 0.2, seed=seed),
    "mpo": lambda seed=0: gen_mpo(100, 1000, seed=seed),
    # configs[4] is 2e9 nnz over 2/4/8 GPUs; one GPU's share of the 8-GPU job:
    "mixed": lambda seed=0: gen_mixed_large(0.125, seed=seed),
}

__all__ = ["ConicProgram", "ZERO", "NONNEG", "SOC", "RSOC", "EXP", "DUAL_EXP",
           "KIND_NAMES", "csr_from_coo", "gen_lasso", "gen_fisher", "gen_mpo",
           "gen_mixed", "gen_mixed_large", "bernoulli_positions", "CONFIGS",
           "mixed_full_layout", "gen_mixed_shard", "MixedLayout", "ShardedProgram"]
