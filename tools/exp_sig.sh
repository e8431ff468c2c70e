#!/bin/bash
# Fast sigmoid32: exhaustive self-check, GPU tests, and sweep times.
mkdir -p gpurun_out
timeout 300 python -c "
import ctypes as C, sys; sys.path.insert(0,'.')
import paper_2005_04347_b200 as A
dev=A.Device.get(0); b=C.c_uint64(); s=C.c_uint64()
dev.check(dev.lib.asnn_dev_sigmoid_selfcheck(dev.h, C.byref(b), C.byref(s)))
print('selfcheck mismatches', b.value, 'exact-path', s.value)
"
timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
run() { timeout 300 python bench.py "$@" --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), "value %.4g" % d["value"], "e2e %.4g" % d["e2e"]["value"])'; }
for C in c1 c3 c5 c2 c4; do echo "$C $(run --config $C)"; done
timeout 120 python tools/latency_probe.py
