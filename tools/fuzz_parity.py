"""Randomised parity sweep (GPU): random networks of the reference's
generator (netgen.cpp:71-157 via api.generate / random_spec), power-law
bands and MLPs, random batch widths (1 .. 300, odd ones included), every
sweep strategy (auto, per-level + segments, K-cta, per-level whole rows) and
several heavy-row thresholds -- each activation compared bit for bit with
the oracle's eval_sequential restatement.  Runs until the time budget is
spent and prints one summary line (profiles/r1_fuzz.txt).

    python tools/fuzz_parity.py [seconds] [seed]"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2005_04347_b200 as A  # noqa: E402
from oracle.bind import Oracle  # noqa: E402


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rng = np.random.default_rng(seed)
    sm = A.SplitMix64(seed)
    oracle = Oracle()
    dev = A.Device.get(0)
    stats = {"networks": 0, "activations": 0, "mismatches": 0, "edges_max": 0, "batches": set(),
             "strategies": set()}
    failures = []
    t_end = time.perf_counter() + budget
    while time.perf_counter() < t_end:
        kind = rng.integers(0, 4)
        if kind <= 1:
            net = A.generate(A.random_spec(sm, 50, int(rng.choice([2000, 20000, 120000]))))
        elif kind == 2:
            n = int(rng.integers(2000, 40000))
            net = A.generate_powerlaw(n, int(rng.integers(3, 30)), int(rng.integers(2, 64)),
                                      int(rng.integers(1, 32)), n * int(rng.integers(5, 40)), 2.1,
                                      int(rng.integers(1, 1 << 30)))
        else:
            net = A.generate_mlp(int(rng.integers(3, 40)), int(rng.integers(8, 300)), float(rng.uniform(0.05, 0.5)),
                                 int(rng.integers(1, 1 << 30)))
        d = oracle.layout(net)
        dl = A.DeviceLayout.from_network(net)
        stats["networks"] += 1
        stats["edges_max"] = max(stats["edges_max"], len(net.source))
        for _ in range(3):
            B = int(rng.choice([1, 2, 3, 4, 7, 8, 16, 17, 32, 33, 64, 100, 128, 129, 256, 300]))
            X = rng.uniform(-3, 3, (B, len(net.inputs))).astype(np.float32)
            want = oracle.eval_batch(d, X)
            for mode in (0, 1, 2, 3):
                thr = int(rng.choice([16, 64, 512, 4096]))
                dev.set_sweep_mode(mode)
                dev.set_heavy_threshold(thr)
                try:
                    out, st = dl.activate(X, outputs=True, state=True)
                finally:
                    dev.set_sweep_mode(0)
                    dev.set_heavy_threshold(512)
                stats["activations"] += 1
                stats["batches"].add(B)
                stats["strategies"].add(dl.plan(B)["strategy"] if mode == 0 else f"mode{mode}")
                ok = np.array_equal(st.view(np.uint32), want.view(np.uint32)) and np.array_equal(
                    out.view(np.uint32), st[:, net.outputs].view(np.uint32))
                if not ok:
                    stats["mismatches"] += 1
                    failures.append({"edges": len(net.source), "B": B, "mode": mode, "thr": thr})
        dl.free()
    stats["batches"] = sorted(stats["batches"])
    stats["strategies"] = sorted(stats["strategies"])
    stats["failures"] = failures[:10]
    stats["seconds"] = budget
    stats["seed"] = seed
    print(json.dumps(stats))
    sys.exit(1 if failures else 0)


if __name__ == "__main__":
    main()
