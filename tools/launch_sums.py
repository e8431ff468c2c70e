"""Per-kernel sums of an ncu launch list of `bench.py --ncu-sweeps N` (last sweep):
launches, serialized ms, DRAM GB and GB/s.  Usage: python tools/launch_sums.py <csv>..."""
import collections
import csv
import sys


def sums(path):
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    h = rows[0]
    ik, im, iv, iid = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    d = collections.defaultdict(dict)
    for r in rows[1:]:
        if len(r) != len(h):
            continue
        d[int(r[iid])][r[im]] = float(r[iv].replace(",", ""))
        d[int(r[iid])]["name"] = r[ik].split("(")[0].replace("void ", "")
    ids = sorted(d)
    first = [i for i in ids if "k_sense" in d[i]["name"] or "k_cta" in d[i]["name"]][-1]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i in ids:
        if i < first:
            continue
        a = agg[d[i]["name"]]
        a[0] += 1
        a[1] += d[i]["gpu__time_duration.sum"]
        a[2] += d[i].get("dram__bytes_read.sum", 0) + d[i].get("dram__bytes_write.sum", 0)
    return agg


for p in sys.argv[1:]:
    print(p)
    for k, (n, ns, b) in sorted(sums(p).items(), key=lambda kv: -kv[1][1]):
        print(f"  {k:40s} {n:4d} {ns / 1e6:9.3f} ms {b / 1e9:8.2f} GB {b / ns if ns else 0:8.1f} GB/s")
