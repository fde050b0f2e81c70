"""Rounding sensitivity of Alg. 1 (CPU oracle only).

The adaptive step size eta_{k+1} = min(1.05 eta_k, eta_bar(z_k)) (SPEC.md:354,
440) makes the PDCS iteration map depend on the iterate through eta_bar, and
perturbations of one unit in the last place grow exponentially (here >1e4x per
~600 iterations).  Plain PDHG with a fixed step does not
amplify.  This is why free-running per-iterate parity between two fp64
implementations cannot hold at 2000 iterations, and why the GPU parity tests
shadow the oracle segment by segment.
"""
import copy

import numpy as np

import oracle as O
from instances import gen_lasso


def _divergence(prog, eps, steps, **params):
    p2 = copy.copy(prog)
    p2.h = prog.h * (1.0 + eps)
    a, b = O.OracleSolver(prog, **params), O.OracleSolver(p2, **params)
    out = []
    for _ in range(steps // 40):
        a.iterate(40)
        b.iterate(40)
        xa, ya = a.get_iterate(0)
        xb, yb = b.get_iterate(0)
        out.append(max(np.abs(xa - xb).max() / (1 + np.abs(xa).max()),
                       np.abs(ya - yb).max() / (1 + np.abs(ya).max())))
    return out


def test_pdcs_amplifies_rounding_vanilla_does_not():
    # the literal Lasso form (balance=False): its PDCS trajectory wanders for
    # thousands of iterations (P8), which is where the amplification shows;
    # the balanced form converges in a few hundred and then sits still
    prog = gen_lasso(100, 50, 1.0, seed=0, dense=True, balance=False)
    pdcs = _divergence(prog, 1e-15, 800)
    van = _divergence(prog, 1e-15, 800, vanilla_pdhg=1)
    frozen = _divergence(prog, 1e-15, 800, ls_grow=1.0)    # step never grows
    assert max(pdcs) > 1e-8          # exponential amplification of a 1e-15 perturbation
    assert max(van) < 1e-13          # fixed-step PDHG: no amplification
    assert max(frozen) < 1e-13
    assert pdcs[4] < 1e-9            # ...but over the first 200 iterations it stays < 1e-9
