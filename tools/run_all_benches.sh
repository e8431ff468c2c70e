#!/bin/bash
# Evidence run (one GPU): GPU tests, every config's bench line with its CPU
# baseline, the default bench invocation, the reference arm, the ncu launch
# lists of C4/C2 (per-kernel shares, DRAM traffic per sweep) and one full ncu
# capture of the dominant kernel (k_rows on a middle C4 level).
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; tail -1 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv,noheader > gpurun_out/gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/host.txt
for C in c1 c2 c3 c5; do
  timeout 600 python bench.py --config $C --steps 20 --warmup 5 --cpu-budget 10 2>/dev/null | tail -1 > gpurun_out/bench_$C.json
done
timeout 900 python bench.py 2>/dev/null | tail -1 > gpurun_out/bench_c4.json          # the driver's default invocation
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 2>/dev/null | tail -1 > gpurun_out/bench_c4_reference.json
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for C in c4 c2; do
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${C}_launches.csv python bench.py --config $C --ncu-sweeps 2 > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rows -s 50 -c 1 -o gpurun_out/c4_k_rows python bench.py --config c4 --ncu-sweeps 1 > /dev/null 2>&1
timeout 120 python tools/latency_probe.py > gpurun_out/latency.json 2>&1
timeout 900 python tools/bench_parse.py c2 > gpurun_out/parse_bench.txt 2>&1
ls -la gpurun_out
