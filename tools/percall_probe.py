"""Per-call drop-in cost broken into its C-ABI stages (tool, not product):
eval_parallel(DeviceCompute) = upload the host layout + activate one vector
(id-indexed state back) + free, on the reference bench corpus shapes."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2005_04347_b200 as A  # noqa: E402
from oracle.bind import Oracle  # noqa: E402


def t_us(fn, n=50):
    for _ in range(5):
        fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t0) / n * 1e6


def main():
    o = Oracle()
    master = A.SplitMix64(42)
    for conn in (1000, 10000, 100000, 1000000):
        spec = A.corpus_spec(conn, 10, 8, 2, master.next())
        net = A.generate(spec)
        d = o.layout(net)
        lay = A.LayeredLayout(d["total_layers"], d["layer_offsets"], d["node_ids"], d["row_ptr"], d["in_nodes"],
                              d["in_weights"], d["input_order"], d["dropped_connections"], d["id_bound"])
        x = np.full(len(d["input_order"]), 0.5, np.float32)
        cfg = A.ParallelConfig(backend=A.Backend.DeviceCompute)
        r = {}
        r["eval_parallel per call"] = t_us(lambda: A.eval_parallel(lay, x, cfg))
        r["upload"] = t_us(lambda: A.DeviceLayout.from_layout(lay).free())
        dl = A.DeviceLayout.from_layout(lay)
        r["activate state (resident)"] = t_us(lambda: dl.activate(x[None, :], outputs=False, state=True))
        r["activate outputs (resident)"] = t_us(lambda: dl.activate(x[None, :], outputs=True, state=False))
        dev = A.Device.get(0)
        A.DeviceLayout.from_layout(lay).free()
        print(conn, {k: round(v, 1) for k, v in r.items()}, "upload timings", dev.timings(), flush=True)
        dl.free()


if __name__ == "__main__":
    main()
