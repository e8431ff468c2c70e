"""SPEC invariant "every op slot is written exactly once" on the device path
(proj/tests/test_eval.cpp:199-213): the write-count build of the
engine (build/debug/libasnn_b200_wc.so, every producer of an activation adds
1 to a counter of its (position, column)) sweeps networks under every
strategy -- per-level k_rows / k_level / k_warp_rows, heavy rows split into
segments across levels (partial sums parked in accbuf, only the last segment
writes the slot), k_heavy, K-cta (plain and pipelined), populations, layouts
with position-less predecessors -- and every (position, column < n_vec)
count must be exactly 1.  Runs in a child process that loads the debug
library through ASNN_B200_LIB."""
from __future__ import annotations

import json
import os
import pathlib
import subprocess
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
WC_LIB = ROOT / "build" / "debug" / "libasnn_b200_wc.so"


@pytest.mark.gpu
def test_every_op_slot_written_exactly_once():
    assert WC_LIB.exists(), "build() makes the write-count library"
    env = dict(os.environ, ASNN_B200_LIB=str(WC_LIB))
    r = subprocess.run([sys.executable, __file__], env=env, capture_output=True, text=True,
                       timeout=900, cwd=str(ROOT))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["cases"] >= 40 and res["bad"] == [], res


def _counts(dl, n_vec):
    import ctypes as C
    from paper_2005_04347_b200 import _lib
    n = dl.info()["node_count"]
    c = np.zeros(n * n_vec, np.uint32)
    dl.dev.check(dl.dev.lib.asnn_dev_debug_write_counts(dl.h, n_vec, _lib.ptr(c, C.c_uint32)))
    return c.reshape(n, n_vec)


def _child():
    sys.path.insert(0, str(ROOT))
    import paper_2005_04347_b200 as A
    from oracle.bind import Oracle
    dev = A.Device.get(0)
    cases, bad = 0, []

    def check(tag, dl, n_vec):
        nonlocal cases
        c = _counts(dl, n_vec)
        cases += 1
        if not np.all(c == 1):
            bad.append({"case": tag, "n_vec": n_vec, "min": int(c.min()), "max": int(c.max()),
                        "wrong": int((c != 1).sum()), "kind": dl.plan(n_vec)["strategy"]})

    rng = A.SplitMix64(2024)
    nets = {"gen": A.generate(A.random_spec(rng, 3000, 30000)),
            "deep": A.generate(A.GenSpec(8, 4, 3000, 30000, 300, seed=5)),
            "mlp": A.generate_mlp(12, 300, 0.1, 3),
            "powerlaw": A.generate_powerlaw(200_000, 40, 512, 512, 10_000_000, 2.1, 7)}
    for name, net in nets.items():
        dl = A.DeviceLayout.from_network(net)
        for mode in (0, 1, 2, 3, 4):
            dev.set_sweep_mode(mode)
            for B in ((1, 4, 64, 130, 256) if name != "powerlaw" else (1, 16, 64)):
                check(f"{name}/mode{mode}", dl, B)
        dev.set_sweep_mode(3)
        dev.set_heavy_threshold(16)          # k_heavy for every row above in-degree 16
        check(f"{name}/heavy16", dl, 64)
        dev.set_heavy_threshold(512)
        dev.set_sweep_mode(0)
        dl.free()
    pop = [A.generate(A.GenSpec(6, 3, 150, 900, 7, seed=rng.next())) for _ in range(40)]
    dl = A.DeviceLayout.from_population(pop)
    for mode in (0, 1, 2):
        dev.set_sweep_mode(mode)
        for B in (1, 32, 128):
            check(f"population/mode{mode}", dl, B)
    dev.set_sweep_mode(0)
    # predecessors without a position (the zero row is read, never written)
    o = Oracle()
    net = A.generate(A.random_spec(rng, 500, 4000))
    d = o.layout(net)
    d["in_nodes"] = d["in_nodes"].copy()
    d["in_nodes"][np.random.default_rng(1).random(len(d["in_nodes"])) < 0.05] = int(net.nodes.max()) + 5
    d["id_bound"] = int(net.nodes.max()) + 6
    dl = A.DeviceLayout.from_layout(A.LayeredLayout(d["total_layers"], d["layer_offsets"], d["node_ids"],
                                                    d["row_ptr"], d["in_nodes"], d["in_weights"],
                                                    d["input_order"], 0, d["id_bound"], net.outputs))
    for mode in (0, 1, 2, 3, 4):
        dev.set_sweep_mode(mode)
        for B in (1, 64, 256):
            check(f"zero-row/mode{mode}", dl, B)
    dev.set_sweep_mode(0)
    print(json.dumps({"cases": cases, "bad": bad}))


if __name__ == "__main__":
    _child()
