for v in "ASNN_CTA_PIPE_MAX=256" "ASNN_CTA_PIPE_MAX=128"; do for c in c1 c3 c5; do echo "$v $c" >> gpurun_out/r2_t12.txt; env $v python bench.py --config $c --steps 50 --warmup 10 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['value'])" >> gpurun_out/r2_t12.txt 2>&1; done; done
python tools/percall_probe.py >> gpurun_out/r2_t12.txt 2>&1
python tools/call_overhead.py >> gpurun_out/r2_t12.txt 2>&1
python -m pytest tests/test_gpu_activate.py tests/test_gpu_integration.py -x -q 2>&1 | tail -2 >> gpurun_out/r2_t12.txt
