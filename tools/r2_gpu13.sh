for v in 5 9 10 11 12; do for c in c2 c4; do echo "variant $v $c" >> gpurun_out/r2_t13.txt; ASNN_LEVEL_VARIANT=$v python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'])" >> gpurun_out/r2_t13.txt 2>&1; done; done
ASNN_LEVEL_VARIANT=11 python -m pytest tests/test_gpu_activate.py tests/test_gpu_segments.py -x -q 2>&1 | tail -2 >> gpurun_out/r2_t13.txt
python tools/percall_probe.py >> gpurun_out/r2_t13.txt 2>&1
