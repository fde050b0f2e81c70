"""C-ABI boundary checks that run without a GPU (-m "not gpu")."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pdcs.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pdcs_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2505_00311_b200 import build
    return build.build()


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (pdcs_[a-z_0-9]+)", out))
    decl = declared_functions()
    assert len(decl) >= 14
    missing = [f for f in decl if f not in exported]
    assert not missing, missing


def test_library_loads_and_binding_names_match(libpath):
    import paper_2505_00311_b200 as P
    from paper_2505_00311_b200 import _lib
    L = _lib.lib()
    for f in declared_functions():
        assert hasattr(L, f)
        assert f in _lib.EXPORTED, f
        assert hasattr(P, f) or f in ("pdcs_default_params",)
    p = P.pdcs_default_params()
    assert p.tol == 1e-6 and p.ruiz_iters == 10 and p.check_interval == 40 and p.ls_grow == 1.05


def test_sass_is_sm100(libpath):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_create_without_gpu_fails_loudly(libpath):
    """No CPU fallback: without a device pdcs_create returns ERR_CUDA."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2505_00311_b200 as P
    from instances import gen_lasso
    prog = gen_lasso(10, 5, 1.0, dense=True)
    with pytest.raises(P.PdcsError) as ei:
        P.PdcsSolver(prog)
    assert ei.value.code == 7


def test_param_struct_layouts_match():
    """Oracle and product declare the same parameter layout independently."""
    import ctypes as C
    import oracle as O
    from paper_2505_00311_b200 import _lib
    a = [(n, t) for n, t in O.Params._fields_]
    b = [(n, t) for n, t in _lib.pdcs_params._fields_]
    assert [n for n, _ in a] == [n for n, _ in b]
    assert C.sizeof(O.Params) == C.sizeof(_lib.pdcs_params)
