O=gpurun_out/r2_t29.txt
timeout 900 python -m pytest tests/test_gpu_activate.py tests/test_gpu_segments.py tests/test_gpu_integration.py tests/test_gpu_writecount.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r2_t29_pytest.txt 2>&1; echo "pytest rc=$?" > $O
for dv in 3 6 12 24; do
  echo "c3 group div $dv" >> $O
  ASNN_CHAIN_GROUP_DIV=$dv timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline 2>>$O | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d.get('e2e',{}).get('value'), d['value'])" >> $O 2>&1
done
echo "c1" >> $O
timeout 300 python bench.py --config c1 --steps 20 --warmup 5 --no-cpu-baseline 2>>$O | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d.get('e2e',{}).get('value'), d['value'])" >> $O 2>&1
