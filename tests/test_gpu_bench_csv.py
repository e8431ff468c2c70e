"""the reference's bench protocol with device rows
(tools/bench_csv.py) -- file set, headers, row order and number format of
the reference's write_csv / write_meta (proj/src/bench.cpp:103-146), and the
speedup files computed from the timing rows they claim (sequential over
parallel, over device per call, over device resident, over the resident
server)."""
from __future__ import annotations

import csv
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

BACKENDS = ["sequential", "parallel", "device", "device_resident", "device_server"]


def test_bench_csv_schema_and_speedups(tmp_path):
    from oracle.bind import available_ref_dev
    if not available_ref_dev():
        pytest.skip("oracle/_ref/libasnn_ref_dev.so not built")
    prefix = tmp_path / "bench"
    r = subprocess.run([sys.executable, "tools/bench_csv.py", "--connections", "1000,200",
                        "--depths", "3,12", "--reps-seq", "3", "--reps-par", "4", "--csv", str(prefix)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    rows = list(csv.reader(open(f"{prefix}.timings.csv")))
    assert rows[0] == ["network_id", "connections", "layers", "backend", "repetitions", "mean_time_us",
                       "stddev_us"]
    body = rows[1:]
    ids = sorted({b[0] for b in body})
    # the corpus networks all fit one SM's shared memory: every one has a server row
    assert len(body) == 5 * len(ids) == 20
    # bench.cpp:105-110: by network_id (string order), then backend in enum order
    assert [b[0] for b in body] == [i for i in ids for _ in BACKENDS]
    assert [b[3] for b in body] == BACKENDS * len(ids)
    assert [int(b[4]) for b in body] == [3, 4, 4, 4, 4] * len(ids)
    t = {(b[0], b[3]): float(b[5]) for b in body}
    for name, den in (("speedup", "parallel"), ("device_speedup", "device"),
                      ("device_resident_speedup", "device_resident"),
                      ("device_server_speedup", "device_server")):
        s = list(csv.reader(open(f"{prefix}.{name}.csv")))
        assert s[0] == ["network_id", "connections", "layers", "speedup"]
        assert [x[0] for x in s[1:]] == ids
        for x in s[1:]:
            assert float(x[3]) == pytest.approx(t[(x[0], "sequential")] / t[(x[0], den)], rel=1e-9)
    meta = dict(line.rstrip("\n").split("=", 1) for line in open(f"{prefix}.meta"))
    for k in ("hardware_threads", "workers", "warmup_runs", "reps_sequential", "reps_parallel", "seed",
              "connections", "depths", "failures", "device_path"):
        assert k in meta, k
    assert meta["failures"] == "0" and meta["protocol_override"] == "reps"
