#!/bin/bash
# Row-item kernel variants (ASNN_LEVEL_VARIANT) on C4 and C2, per-level launches (mode 3).
mkdir -p gpurun_out
run() { python bench.py "$@" --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), "%.4g" % d["value"], round(d["roofline"]["frac"],3), d["roofline"]["kernel"][:9])'; }
for V in 1 5 6 7 8; do
  echo "c4 variant=$V $(ASNN_SWEEP_MODE=3 ASNN_LEVEL_VARIANT=$V ASNN_HEAVY_THRESHOLD=512 run --config c4)"
  echo "c2 variant=$V $(ASNN_SWEEP_MODE=3 ASNN_LEVEL_VARIANT=$V run --config c2)"
done
