"""include/pdcs.h compiled into a plain C99 client (tests/c/pdcs_c_smoke.c) and
linked against libpdcs.so: host-only calls and the no-device error path on CPU,
a tiny LP solved through the C ABI on the GPU (its optimum is closed-form)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    from paper_2505_00311_b200 import build
    lib = build.build()
    exe = str(tmp_path / "pdcs_c_smoke")
    subprocess.check_call(["gcc", "-std=c99", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "c", "pdcs_c_smoke.c"), "-o", exe,
                           "-L", os.path.dirname(lib), "-lpdcs", "-Wl,-rpath," + os.path.dirname(lib), "-lm"])
    return exe


def test_c_client_host_calls(tmp_path):
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("the no-device path needs a machine without a GPU")
    except ImportError:
        pass
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "host: 0 failures" in r.stdout


@pytest.mark.gpu
def test_c_client_solves_lp(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "gpu: 0 failures" in r.stdout
