"""Randomised parity of the one-call path (csrc/once.cu) against the oracle:
random reference-generator networks (10 .. 300k connections, depth 3 .. 120,
random inputs), every kernel variant, bitwise; plus injected out-of-range ids
(predecessor / node), which must come back as ValueError without touching
memory out of bounds.

  python tools/once_fuzz.py [--nets 300] [--seed 7]
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_04347_b200 as A  # noqa: E402
from oracle.bind import Oracle  # noqa: E402

MODES = ["auto", "1", "2", "3", "4", "5", "6"]


def to_layout(d):
    return A.LayeredLayout(d["total_layers"], d["layer_offsets"], d["node_ids"], d["row_ptr"], d["in_nodes"],
                           d["in_weights"], d["input_order"], d["dropped_connections"], d["id_bound"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nets", type=int, default=300)
    ap.add_argument("--seed", type=int, default=7)
    a = ap.parse_args()
    o = Oracle()
    rng = np.random.default_rng(a.seed)
    sm = A.SplitMix64(a.seed)
    t0 = time.time()
    checked = values = mismatches = errors_ok = 0
    per_mode = {m: 0 for m in MODES}
    for n in range(a.nets):
        conns = int(np.exp(rng.uniform(np.log(10), np.log(300000))))
        depth = int(rng.integers(3, 121))
        spec = A.corpus_spec(conns, depth, int(rng.integers(1, 17)), int(rng.integers(1, 5)), sm.next())
        try:
            net = A.generate(spec)
        except Exception:
            continue
        d = o.layout(net)
        lay = to_layout(d)
        x = rng.uniform(-3, 3, len(lay.input_order)).astype(np.float32)
        ref = o.eval_batch(d, x[None, :])[0].view(np.uint32)
        for m in MODES:
            if m == "auto":
                os.environ.pop("ASNN_ONCE_MODE", None)
            else:
                os.environ["ASNN_ONCE_MODE"] = m
            got = A.eval_once(lay, x).view(np.uint32)
            bad = int((got != ref).sum())
            mismatches += bad
            values += got.size
            checked += 1
            per_mode[m] += 1
            if bad:
                print(f"MISMATCH net {n} mode {m}: {bad} values", flush=True)
        os.environ.pop("ASNN_ONCE_MODE", None)
        # injected out-of-range ids
        if len(lay.in_nodes):
            badl = to_layout(d)
            badl.in_nodes = badl.in_nodes.copy()
            badl.in_nodes[int(rng.integers(len(badl.in_nodes)))] = lay.id_bound + int(rng.integers(1, 1000))
            try:
                A.eval_once(badl, x)
                print(f"NO ERROR for bad predecessor, net {n}", flush=True)
            except ValueError:
                errors_ok += 1
        badl = to_layout(d)
        badl.node_ids = badl.node_ids.copy()
        badl.node_ids[int(rng.integers(len(badl.node_ids)))] = lay.id_bound + 5
        try:
            A.eval_once(badl, x)
            print(f"NO ERROR for bad node id, net {n}", flush=True)
        except ValueError:
            errors_ok += 1
    print(f"networks {a.nets}, evaluations {checked} (per variant {per_mode}), values {values}, "
          f"mismatches {mismatches}, injected errors reported {errors_ok}, {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
