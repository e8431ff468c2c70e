"""Parity of the opt-in K-rows-window level kernel (win_rows.cuh, ASNN_LEVEL_WIN=1):
levels of whole rows whose sources lie in one narrow window of positions
(pruned MLPs, config 2's shape) are gathered from a shared-memory copy of the
window.  The switch is read once per process, so the sweeps run in a child
process; every state value must be bitwise equal to the oracle's
(eval.cpp:20-21 summation order), and the write-count build must see every op
slot written once."""
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


def _run(extra_env: dict) -> dict:
    env = dict(os.environ, ASNN_LEVEL_WIN="1", **extra_env)
    r = subprocess.run([sys.executable, __file__], env=env, capture_output=True, text=True,
                       timeout=900, cwd=str(ROOT))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
def test_level_window_bitwise_against_oracle():
    res = _run({})
    assert res["cases"] >= 8 and res["bad"] == [], res


@pytest.mark.gpu
def test_level_window_writes_every_slot_once():
    assert WC_LIB.exists(), "build() makes the write-count library"
    res = _run({"ASNN_B200_LIB": str(WC_LIB), "ASNN_WIN_CHILD_WC": "1"})
    assert res["cases"] >= 8 and res["bad"] == [], res


def _child():
    sys.path.insert(0, str(ROOT))
    import ctypes as C
    import paper_2005_04347_b200 as A
    from paper_2005_04347_b200 import _lib
    from oracle.bind import Oracle
    wc = os.environ.get("ASNN_WIN_CHILD_WC") == "1"
    dev = A.Device.get(0)
    dev.set_sweep_mode(3)                # per-level launches of whole rows
    o = Oracle()
    cases, bad = 0, []
    rng = np.random.default_rng(7)
    nets = {"mlp-300": A.generate_mlp(12, 300, 0.1, 3),
            "mlp-500": A.generate_mlp(6, 500, 0.1, 11),
            "mlp-dense": A.generate_mlp(4, 200, 0.5, 5)}
    for name, net in nets.items():
        d = o.layout(net)
        lay = A.LayeredLayout(d["total_layers"], d["layer_offsets"], d["node_ids"], d["row_ptr"],
                              d["in_nodes"], d["in_weights"], d["input_order"], d["dropped_connections"],
                              d["id_bound"], np.asarray(net.outputs, np.uint32))
        dl = A.DeviceLayout.from_layout(lay)
        for B in (128, 160, 256, 1024):
            cases += 1
            if wc:
                n = dl.info()["node_count"]
                c = np.zeros(n * B, np.uint32)
                dev.check(dev.lib.asnn_dev_debug_write_counts(dl.h, B, _lib.ptr(c, C.c_uint32)))
                if not np.all(c == 1):
                    bad.append({"case": f"{name}/B{B}", "min": int(c.min()), "max": int(c.max())})
                continue
            X = rng.uniform(-2, 2, (B, len(net.inputs))).astype(np.float32)
            _, st = dl.activate(X, outputs=True, state=True)
            ref = o.eval_batch(d, X)
            ne = int((st.view(np.uint32) != ref.view(np.uint32)).sum())
            if ne:
                bad.append({"case": f"{name}/B{B}", "differ": ne})
        dl.free()
    # the windowed kernel is the one that ran (kernel names seen by CUPTI)
    import torch
    from torch.profiler import ProfilerActivity, profile
    net = nets["mlp-500"]
    d = o.layout(net)
    dl = A.DeviceLayout.from_network(net)
    X = rng.uniform(-2, 2, (256, len(net.inputs))).astype(np.float32)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        dl.activate(X, outputs=True, state=False)
        torch.cuda.synchronize()
    names = {e.name for e in prof.events()}
    if not any("k_rows_win" in n for n in names):
        bad.append({"case": "kernel-not-launched", "names": sorted(names)[:20]})
    dl.free()
    dev.set_sweep_mode(0)
    print(json.dumps({"cases": cases, "bad": bad}))


if __name__ == "__main__":
    _child()
