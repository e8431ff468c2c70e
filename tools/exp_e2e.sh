#!/bin/bash
# Host-buffer paths: parity tests, then e2e numbers for C1/C5/C4.
mkdir -p gpurun_out
python -m pytest tests/test_gpu_hostio.py tests/test_gpu_activate.py tests/test_gpu_segments.py tests/test_gpu_preprocess.py -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -4 gpurun_out/pytest_gpu.txt
run() { python bench.py "$@" --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), "value %.4g" % d["value"], "e2e %.4g" % d["e2e"]["value"], d["gpu_launches"])'; }
for C in c1 c5 c3 c2 c4; do echo "$C $(run --config $C)"; done
