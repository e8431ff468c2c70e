"""The reference's `asnn bench` protocol (asnn_main.cpp:312-386, bench.cpp)
with device rows: the same seeded corpus (make_corpus_spec over
--connections x --depths, 8 inputs, 2 outputs, SplitMix64 network seeds), the
reference's sequential (5 reps) and parallel (10 reps) timings of
eval_sequential / eval_parallel (oracle/_ref, timed inside C++), and the
DeviceCompute backend through the maintainer's binding
(integration/asnn_device_backend.cpp, the drop-in of INTEGRATION.md), also
timed inside C++.  Writes the reference's CSV schema (
headers, row order and number format of bench.cpp:103-137):

  <prefix>.timings.csv  network_id,connections,layers,backend,repetitions,mean_time_us,stddev_us
                        backend: sequential, parallel (as the reference), then
                          device          = eval_parallel(DeviceCompute) per call: the
                                            reference's LayeredLayout converted, uploaded,
                                            activated, state back, freed -- every call;
                          device_resident = asnn_dev_activate on a layout uploaded once
                                            (state back);
                          device_server   = the resident server (asnn_dev_server_activate,
                                            persistent kernel, declared outputs back) where
                                            the network fits one SM's shared memory
  <prefix>.speedup.csv                  network_id,connections,layers,speedup  sequential / parallel
  <prefix>.device_speedup.csv           same columns, sequential / device (per call)
  <prefix>.device_resident_speedup.csv  same columns, sequential / device_resident
  <prefix>.device_server_speedup.csv    same columns, sequential / device_server
  <prefix>.meta         key=value lines

Usage: python tools/bench_csv.py --connections 1000,10000,100000 --depths 10,100 --csv out/bench
"""
from __future__ import annotations

import argparse
import math
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2005_04347_b200 as A  # noqa: E402
from oracle.bind import RefDev  # noqa: E402


def format_double(v: float) -> str:
    """std::to_chars(double) (io.cpp:19-23): shortest round-trip digits, the
    shorter of fixed and scientific notation (fixed on a tie)."""
    if v == 0:
        return "0" if math.copysign(1, v) > 0 else "-0"
    r = repr(float(v))
    mant, _, ex = r.partition("e")
    neg = mant.startswith("-")
    mant = mant.lstrip("-")
    digits = mant.replace(".", "").lstrip("0")
    point = (mant.index(".") if "." in mant else len(mant)) + (int(ex) if ex else 0)
    lead = len(mant.split(".")[0].lstrip("0")) if mant.split(".")[0].lstrip("0") else 0
    if lead == 0:  # 0.000ddd
        zeros = len(mant.split(".")[1]) - len(mant.split(".")[1].lstrip("0"))
        point = -zeros + (int(ex) if ex else 0)
    digits = digits.rstrip("0") or "0"
    e10 = point - 1
    sci = digits[0] + ("." + digits[1:] if len(digits) > 1 else "") + "e" + ("-" if e10 < 0 else "+") + \
        f"{abs(e10):02d}"
    if point <= 0:
        fixed = "0." + "0" * (-point) + digits
    elif point >= len(digits):
        fixed = str(int(abs(v)))  # an integer: to_chars prints its exact value
    else:
        fixed = digits[:point] + "." + digits[point:]
    out = fixed if len(fixed) <= len(sci) else sci
    return ("-" if neg else "") + out


def stats(samples):
    m = sum(samples) / len(samples)
    sd = math.sqrt(sum((s - m) ** 2 for s in samples) / (len(samples) - 1)) if len(samples) > 1 else 0.0
    return m, sd


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--connections", required=True)
    ap.add_argument("--depths", required=True)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--reps-seq", type=int, default=5)
    ap.add_argument("--reps-par", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--workers", type=int, default=0)
    ap.add_argument("--input-value", type=float, default=0.5)
    ap.add_argument("--csv", required=True)
    a = ap.parse_args()
    conns = [int(x) for x in a.connections.split(",")]
    depths = [int(x) for x in a.depths.split(",")]
    ref = RefDev()
    master = A.SplitMix64(a.seed)
    records, speed, dspeed, rspeed, sspeed, failures = [], [], [], [], [], []
    for d in depths:
        for c in conns:
            nid = f"c{c}_d{d}"
            spec = A.corpus_spec(c, d, 8, 2, master.next())
            try:
                rn = ref.generate(spec)
                if rn.preprocess():
                    raise RuntimeError("preprocessing failed")
                lay = rn.layout()
                n_in = len(lay["input_order"])
                x = np.full((1, n_in), np.float32(a.input_value), np.float32)
                layers = int(lay["total_layers"])
                arrs = rn.arrays()
                n_conn = len(arrs["source"])

                def ref_reps(mode, reps):
                    for _ in range(a.warmup):
                        rn.eval_batch(x, mode, a.workers)
                    return [rn.eval_batch(x, mode, a.workers)[0] * 1e6 for _ in range(reps)]

                seq = stats(ref_reps(0, a.reps_seq))
                par = stats(ref_reps(1, a.reps_par))
                # device rows through the reference-side binding, timed inside C++
                dev = ref.timed(rn, x[0], resident=False, warmup=a.warmup, reps=a.reps_par)
                res = ref.timed(rn, x[0], resident=True, warmup=a.warmup, reps=a.reps_par)
                srv = ref.server_timed(rn, x[0], warmup=a.warmup, reps=a.reps_par)
                records += [(nid, n_conn, layers, "sequential", a.reps_seq, *seq),
                            (nid, n_conn, layers, "parallel", a.reps_par, *par),
                            (nid, n_conn, layers, "device", a.reps_par, *dev),
                            (nid, n_conn, layers, "device_resident", a.reps_par, *res)]
                if srv is not None:
                    records.append((nid, n_conn, layers, "device_server", a.reps_par, *srv))
                    sspeed.append((nid, n_conn, layers, seq[0] / srv[0]))
                speed.append((nid, n_conn, layers, seq[0] / par[0]))
                dspeed.append((nid, n_conn, layers, seq[0] / dev[0]))
                rspeed.append((nid, n_conn, layers, seq[0] / res[0]))
                print(f"{nid}: seq_us={format_double(seq[0])} par_us={format_double(par[0])} "
                      f"device_us={format_double(dev[0])} resident_us={format_double(res[0])} "
                      f"speedup={format_double(seq[0] / par[0])} device_speedup={format_double(seq[0] / dev[0])} "
                      f"device_resident_speedup={format_double(seq[0] / res[0])}"
                      + (f" server_us={format_double(srv[0])}" if srv else ""))
            except Exception as e:  # bench.cpp:105-107: recorded and skipped
                failures.append((nid, str(e)))
                print(f"failed {nid}: {e}", file=sys.stderr)
    order = {"sequential": 0, "parallel": 1, "device": 2, "device_resident": 3, "device_server": 4}
    records.sort(key=lambda r: (r[0], order[r[3]]))
    with open(a.csv + ".timings.csv", "w") as f:
        f.write("network_id,connections,layers,backend,repetitions,mean_time_us,stddev_us\n")
        for r in records:
            f.write(f"{r[0]},{r[1]},{r[2]},{r[3]},{r[4]},{format_double(r[5])},{format_double(r[6])}\n")
    for path, rows in ((a.csv + ".speedup.csv", speed), (a.csv + ".device_speedup.csv", dspeed),
                       (a.csv + ".device_resident_speedup.csv", rspeed),
                       (a.csv + ".device_server_speedup.csv", sspeed)):
        with open(path, "w") as f:
            f.write("network_id,connections,layers,speedup\n")
            for r in sorted(rows):
                f.write(f"{r[0]},{r[1]},{r[2]},{format_double(r[3])}\n")
    with open(a.csv + ".meta", "w") as f:
        threads = ref.L.ref_max_threads()
        for k, v in [("hardware_threads", threads), ("workers", a.workers or threads),
                     ("warmup_runs", a.warmup), ("reps_sequential", a.reps_seq), ("reps_parallel", a.reps_par),
                     ("protocol_override", "none" if (a.reps_seq, a.reps_par) == (5, 10) else "reps"),
                     ("seed", a.seed), ("connections", a.connections), ("depths", a.depths),
                     ("corpus_inputs", 8), ("corpus_outputs", 2), ("input_value", a.input_value),
                     ("include_preprocessing", 0), ("device_backend", "B200 sm_100a (libasnn_b200.so)"),
                     ("device_path", "integration/asnn_device_backend.cpp eval_device (per call), "
                                     "asnn_dev_activate (resident), asnn_dev_server_activate (server, "
                                     "declared outputs); timed in C++"),
                     ("failures", len(failures))] + [(f"failure_{n}", r) for n, r in failures]:
            f.write(f"{k}={v}\n")


if __name__ == "__main__":
    main()
