"""The C++ drop-in host layer (namespace parfrac): its test binary mirrors the reference's
doctest suites (proj/tests/test_dense.cpp) and runs on the B200."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
BIN = ROOT / "paper_2210_03714_b200" / "_lib" / "test_parfrac"


@pytest.mark.gpu
def test_cpp_parity_suite():
    assert BIN.exists(), "build() must produce the C++ test binary"
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


def test_cpp_method_layer_on_host():
    """The exact method layer of the C++ host (f3: Rational on GMP, solve_weights / build_plain /
    build_hybrid, theta) needs no GPU: the same binary with --host-only."""
    if not BIN.exists():  # g++ only (the CUDA engine library is already in the tree)
        from paper_2210_03714_b200 import build

        build.build_host()
        build.build_cpp_tests()
    r = subprocess.run([str(BIN), "--host-only"], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout and "PASS method construction (f3) and theta" in r.stdout
