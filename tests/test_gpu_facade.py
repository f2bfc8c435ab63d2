"""g++-compiled GPU test of the C++ facade (tests/native/test_facade.cpp): itercur::iterative_cur
through include/itercur/driver_b200.hpp against the CPU oracle."""
import os
import subprocess

import pytest

from test_facade_build import ROOT, compile_facade_test

pytestmark = pytest.mark.gpu


def test_cpp_facade_matches_oracle(engine, tmp_path):
    exe = str(tmp_path / "test_facade")
    compile_facade_test(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "facade ok" in r.stdout
