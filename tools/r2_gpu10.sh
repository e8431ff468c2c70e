python tools/percall_probe.py > gpurun_out/r2_percall.txt 2>&1
python tools/call_overhead.py >> gpurun_out/r2_percall.txt 2>&1
python -m pytest tests/test_gpu_bench_csv.py -x -q 2>&1 | tail -3 >> gpurun_out/r2_percall.txt
python bench.py --config c1 --steps 200 --warmup 20 --no-cpu-baseline >> gpurun_out/r2_percall.txt 2>&1
