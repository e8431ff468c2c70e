"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_*) of
`bench.py --ncu-sweeps 2`: the last sweep's per-kernel shares, DRAM traffic and
L2 hit rate.  Usage: python profiles/summarize_launches.py <csv> [alg_bytes]"""
import collections
import csv
import json
import sys


def load(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    out = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = int(d["ID"])
        e = out.setdefault(key, {"name": d["Kernel Name"].split("(")[0]})
        try:
            v = float(d["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        unit = d["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3,
                 "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3, "%": 1}.get(unit, 1)
        e[d["Metric Name"]] = v * scale
    return list(out.values())


def main():
    keep = ("k_level", "k_rows", "k_heavy", "k_sense", "k_gather_out", "k_state", "k_cta")
    launches = [l for l in load(sys.argv[1])
                if l["name"].replace("void ", "").split("::")[-1].split("<")[0] in keep]
    # the last sweep starts at the last k_sense launch
    starts = [i for i, l in enumerate(launches) if l["name"].endswith("k_sense")]
    sweep = launches[starts[-1]:] if starts else launches
    by = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for l in sweep:
        n = l["name"].replace("void ", "")
        by[n][0] += 1
        by[n][1] += l.get("gpu__time_duration.sum", 0.0)
        by[n][2] += l.get("dram__bytes_read.sum", 0.0) + l.get("dram__bytes_write.sum", 0.0)
    tot_t = sum(v[1] for v in by.values())
    tot_b = sum(v[2] for v in by.values())
    res = {"launches": len(sweep), "serialized_us": tot_t, "dram_bytes": tot_b, "kernels": {}}
    for n, (c, t, b) in sorted(by.items(), key=lambda kv: -kv[1][1]):
        res["kernels"][n] = {"launches": c, "us": round(t, 1), "share": round(t / tot_t, 4),
                             "dram_bytes": b, "dram_gbs": round(b / (t * 1e3), 1) if t else 0}
    if len(sys.argv) > 2:
        alg = float(sys.argv[2])
        res["alg_bytes"] = alg
        res["traffic_over_alg"] = round(tot_b / alg, 4)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
