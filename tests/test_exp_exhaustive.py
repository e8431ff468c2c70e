"""The device exp restatement (paper_2005_04347_b200/csrc/exp_glibc.h, the
operation sequence of glibc's FMA build of exp) equals the host libm's exp
-- the one the reference's sigmoid32 calls (network.hpp:45) -- for every one
of the 2^32 float inputs sigmoid32 can receive, and so does the resulting
sigmoid32.  CPU only: it runs the same header compiled for the host
(oracle/exp_check.c); tests/test_gpu_sigmoid.py compares the device itself."""
from __future__ import annotations

import json
import subprocess

import pytest

from conftest import ROOT

CHECK = ROOT / "oracle" / "_ref" / "exp_check"


def test_exp_restatement_matches_host_libm_for_all_floats():
    if not CHECK.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")], check=True)
    r = subprocess.run([str(CHECK)], capture_output=True, text=True, timeout=600)
    res = json.loads(r.stdout)
    assert res["inputs"] == 2 ** 32
    assert res["exp_mismatches"] == 0, res
    assert res["sigmoid32_mismatches"] == 0, res


def test_table_generator_matches_host_libm():
    lib = "/lib/x86_64-linux-gnu/libm.so.6"
    import os
    if not os.path.exists(lib):
        pytest.skip("no host libm at the Debian path")
    r = subprocess.run(["python", str(ROOT / "tools" / "gen_exp_table.py"), "--check", lib],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
