"""Runs the C++ drop-in test (tests/cpp/test_dropin.cpp): the reference's own
types and call sites with the namespace switched to enprop_b200 give the
reference's results bit for bit (SpMV, dot, axpby, graph, assembly, Dirichlet,
coupled and uncoupled CG, SolverError)."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "build", "test_dropin")


@pytest.mark.gpu
def test_cpp_dropin_matches_reference_bitwise():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/build/test_dropin not built (needs the reference headers at build time)")
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "ALL PASS" in p.stdout
