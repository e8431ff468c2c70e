#!/bin/bash
# C4 tuning run: parity tests for the activation paths, then sweep-time variants.
mkdir -p gpurun_out
python -m pytest tests/test_gpu_segments.py tests/test_gpu_activate.py -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
run() { python bench.py "$@" --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), "%.4g" % d["value"], round(d["roofline"]["frac"],3))'; }
echo "c4 default $(run --config c4)"
for MB in 32 64 96; do echo "c4 l2persist=$MB $(ASNN_L2_PERSIST_MB=$MB run --config c4)"; done
for V in 6 7; do echo "c4 variant=$V $(ASNN_LEVEL_VARIANT=$V run --config c4)"; done
echo "c2 default $(run --config c2)"
${EXTRA:-true}
