#!/bin/bash
# Heavy-row segments: GPU parity tests, then C4/C2 sweeps.
mkdir -p gpurun_out
python -m pytest tests/test_gpu_segments.py tests/test_gpu_activate.py -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -5 gpurun_out/pytest_gpu.txt
run() { python bench.py "$@" --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), "%.4g" % d["value"], round(d["roofline"]["frac"],3), d["roofline"]["kernel"][:12])'; }
for T in 128 256 512; do for M in 32 64 128; do
  echo "c4 thr=$T min=$M $(ASNN_HEAVY_THRESHOLD=$T ASNN_SEG_MIN=$M run --config c4)"
done; done
echo "c4 thr=256 long=1024 $(ASNN_HEAVY_THRESHOLD=256 ASNN_SEG_LONG=1024 run --config c4)"
echo "c4 mode3 $(ASNN_SWEEP_MODE=3 run --config c4)"
echo "c2 $(run --config c2)"
