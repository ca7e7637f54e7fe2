"""The C++ host façade (include/lbk/larch.hpp): it compiles here (CPU) and
its parity program (tests/cpp/test_parity.cpp, against the reference
library itself) passes on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")


def test_facade_header_compiles():
    src = "#include \"lbk/larch.hpp\"\nnamespace larch = lbk::larch;\nint main(){larch::SolverConfig c; return c.max_iters == 1000 ? 0 : 1;}\n"
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"),
                        "-I", "/usr/local/cuda/include", "-x", "c++", "-"], input=src, text=True,
                       capture_output=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_cpp_parity_program():
    exe = os.path.join(CPP, "test_parity")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", CPP], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
