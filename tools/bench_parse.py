"""Loading throughput: the reference's parse_network
(oracle/_ref, one host thread) against the device loader on the same `asnn 1`
text of a config's network, and the device's text -> resident layout
(parse + validate + compute_required + segment + flatten, no host round trip).  Usage: python tools/bench_parse.py [c2|c3|c4] [scale]"""
import json
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2005_04347_b200 as A  # noqa: E402
from oracle.bind import Ref  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    net = bench.make_network(cfg, scale)[0]
    ref = Ref()
    rn = ref.network(net)
    t0 = time.perf_counter()
    text = ref.serialize(rn)
    t_ser = time.perf_counter() - t0
    A.parse_network(text)  # warm-up (context, allocations)
    t0 = time.perf_counter()
    got = A.parse_network(text)
    t_dev = time.perf_counter() - t0
    A.DeviceLayout.from_text(text).free()  # warm-up
    t0 = time.perf_counter()
    dl = A.DeviceLayout.from_text(text)
    t_load = time.perf_counter() - t0
    dl.free()
    t0 = time.perf_counter()
    rn2, err = ref.parse(text)
    t_ref = time.perf_counter() - t0
    assert err is None and len(got.source) == len(net.source)
    print(json.dumps({"config": cfg, "scale": scale, "bytes": len(text), "edges": int(len(net.source)),
                      "reference_parse_s": round(t_ref, 4), "device_parse_s": round(t_dev, 4),
                      "device_GBps": round(len(text) / t_dev / 1e9, 3),
                      "reference_MBps": round(len(text) / t_ref / 1e6, 1),
                      "speedup": round(t_ref / t_dev, 1), "serialize_s": round(t_ser, 2),
                      "device_load_to_layout_s": round(t_load, 4)}))


if __name__ == "__main__":
    main()
