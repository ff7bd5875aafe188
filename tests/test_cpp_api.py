"""Runs the C++ API test driver (tests/cpp/test_cpp_api.cpp, built by
build()): host checks on CPU, compile/run/inverse_lifting on the GPU."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parents[1] / "build" / "test_cpp_api"


def _run(mode):
    if not BIN.exists():
        pytest.skip("C++ API test driver not built")
    r = subprocess.run([str(BIN), mode], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


def test_cpp_api_host():
    _run("host")


@pytest.mark.gpu
def test_cpp_api_gpu():
    _run("gpu")
