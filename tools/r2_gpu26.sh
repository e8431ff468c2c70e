O=gpurun_out/r2_t26.txt
timeout 900 python -m pytest tests/test_gpu_activate.py tests/test_gpu_segments.py tests/test_gpu_integration.py tests/test_gpu_writecount.py tests/test_gpu_fullsize.py tests/test_gpu_concurrency.py tests/test_gpu_group.py -x -q > gpurun_out/r2_t26_pytest.txt 2>&1; echo "pytest rc=$?" > $O
for c in c3 c1 c5; do
  echo "cfg $c" >> $O
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>>$O | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d.get('e2e',{}).get('value'), d['value'])" >> $O 2>&1
done
