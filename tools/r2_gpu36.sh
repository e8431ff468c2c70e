O=gpurun_out/r2_t36.txt
ASNN_LEVEL_VARIANT=13 timeout 900 python -m pytest tests/test_gpu_activate.py tests/test_gpu_segments.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r2_t36_pytest.txt 2>&1; echo "pytest rc=$?" > $O
for v in 5 13; do
  echo "c2 variant $v" >> $O
  ASNN_LEVEL_VARIANT=$v timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline 2>>$O | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'])" >> $O 2>&1
done
