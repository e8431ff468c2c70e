"""The C++ host API (include/asnn_b200.hpp) through the reference's test
scenarios and seeded networks vs the oracle (tests/cpp/test_facade.cpp)."""
from __future__ import annotations

import json
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
BIN = ROOT / "build" / "tests" / "test_facade"


def test_cpp_facade():
    if not BIN.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "tests" / "cpp")], check=True)
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["failures"] == 0 and res["checks"] > 100


def test_cpp_facade_links_engine():
    out = subprocess.run(["ldd", str(BIN)], capture_output=True, text=True).stdout
    assert "libasnn_b200.so" in out
