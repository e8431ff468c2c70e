#!/bin/bash
# Round-end evidence run (one GPU): GPU tests, every config's bench line with
# its CPU baseline, the default bench invocation and the reference arm.
set -u
mkdir -p gpurun_out
python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; tail -1 gpurun_out/pytest_gpu.txt
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv,noheader > gpurun_out/gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/host.txt
for C in c1 c2 c3 c5; do
  python bench.py --config $C --steps 20 --warmup 5 --cpu-budget 10 2>/dev/null | tail -1 > gpurun_out/bench_$C.json
done
python bench.py 2>/dev/null | tail -1 > gpurun_out/bench_c4.json          # the driver's default invocation
python bench.py --impl reference --steps 5 --warmup 3 2>/dev/null | tail -1 > gpurun_out/bench_c4_reference.json
python tools/latency_probe.py > gpurun_out/latency.json 2>&1
ls -la gpurun_out
