#!/bin/bash
# K-cta pipelined consumers: full GPU tests, then C1/C3/C5 with and without.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
run() { timeout 300 python bench.py "$@" --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), "value %.4g" % d["value"], "e2e %.4g" % d["e2e"]["value"])'; }
for C in c1 c3 c5; do echo "$C pipe $(run --config $C)"; echo "$C nopipe $(ASNN_CTA_PIPE=0 run --config $C)"; done
