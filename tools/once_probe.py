"""Cost split of the one-call path (once.cu) on the reference bench corpus:
asnn_eval_buf_run alone (DMA + kernel + synchronise + state copy, the staged
layout reused) per kernel variant, next to the whole per-call drop-in timed in
C++ through the reference binding (staging fill included).

  python tools/once_probe.py [--reps 200]
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_04347_b200 as A  # noqa: E402
from oracle.bind import RefDev  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=200)
    a = ap.parse_args()
    ref = RefDev()
    master = A.SplitMix64(42)
    for d in (10, 100):
        for c in (1000, 10000, 100000, 1000000):
            spec = A.corpus_spec(c, d, 8, 2, master.next())
            rn = ref.generate(spec)
            rn.preprocess()
            lay = rn.layout()
            L = A.LayeredLayout(lay["total_layers"], lay["layer_offsets"], lay["node_ids"], lay["row_ptr"],
                                lay["in_nodes"], lay["in_weights"], lay["input_order"],
                                lay["dropped_connections"], lay["id_bound"])
            x = np.full(len(L.input_order), 0.5, np.float32)
            row = [f"c{c}_d{d}"]
            for m in ("auto", "1", "5", "6", "2", "4"):
                if m == "auto":
                    os.environ.pop("ASNN_ONCE_MODE", None)
                else:
                    os.environ["ASNN_ONCE_MODE"] = m
                buf = A.EvalBuffer()
                buf.stage_layout(L, x)
                for _ in range(10):
                    buf.run()
                t0 = time.perf_counter()
                for _ in range(a.reps):
                    buf.run()
                us = (time.perf_counter() - t0) / a.reps * 1e6
                row.append(f"run[{m}->{buf.mode}]={us:.1f}us")
                buf.free()
            os.environ.pop("ASNN_ONCE_MODE", None)
            import ctypes as C
            acc = (C.c_double * 4)()
            ref.L.ref_dev_phase_clock(1, acc)
            dev = ref.timed(rn, x, resident=False, warmup=5, reps=50)
            ref.L.ref_dev_phase_clock(0, acc)
            ph = [v / 55 for v in acc]
            row.append(f"per_call={dev[0]:.1f}us[state={ph[0]:.1f} sizes={ph[1]:.1f} fill={ph[2]:.1f} "
                       f"run={ph[3]:.1f}]")
            seq = min(rn.eval_batch(x[None, :], 0)[0] for _ in range(20)) * 1e6
            row.append(f"seq={seq:.1f}us")
            print(" ".join(row), flush=True)


if __name__ == "__main__":
    main()
