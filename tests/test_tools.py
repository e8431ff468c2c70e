"""Host-side tools that restate reference formatting: tools/bench_csv.py's
format_double must print exactly what the reference's format_double
(io.cpp:19-23, std::to_chars shortest form) prints into its CSV files."""
from __future__ import annotations

import pathlib
import sys

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1] / "tools"))
from bench_csv import format_double  # noqa: E402


def test_format_double_matches_reference(ref):
    rng = np.random.default_rng(3)
    vals = [0.0, -0.0, 1.0, 0.5, 1e-4, 1e-5, 0.0001234, 123.5, 1e16, 1e15, 1234567.0, 1e22, 2.5e-7, 100.0,
            1e5, 12345678901234567890.0, 549.3602000000001, 85.6686, 0.1, 1 / 3, 2.0 ** 60, 2.0 ** -30]
    vals += list(rng.uniform(0, 1e4, 3000)) + list(rng.uniform(0, 20, 2000)) + \
        list(10.0 ** rng.uniform(-12, 20, 3000)) + list(np.round(rng.uniform(0, 1e6, 2000), 3))
    bad = [(v, format_double(v), ref.format_double(v)) for v in vals
           if format_double(v) != ref.format_double(v)]
    assert not bad, bad[:10]
