"""SM cycles per op of dependent chains on this GPU (asnn_dev_latency_probe)."""
import ctypes as C
import json
import sys

sys.path.insert(0, ".")
import paper_2005_04347_b200 as A  # noqa: E402

dev = A.Device.get(0)
names = ["sigmoid32", "DFMA", "FADD", "LDS chain", "double div", "exp_glibc", "empty loop iter"]
res = {}
for w, nm in enumerate(names):
    c = C.c_double()
    dev.check(dev.lib.asnn_dev_latency_probe(dev.h, w, 4096, C.byref(c)))
    res[nm] = round(c.value, 1)
print(json.dumps(res))
