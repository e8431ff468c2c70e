O=gpurun_out/r2_t40.txt
timeout 900 python -m pytest tests/test_gpu_sigmoid.py tests/test_gpu_activate.py tests/test_gpu_serve.py -x -q > gpurun_out/r2_t40_pytest.txt 2>&1; echo "pytest rc=$?" > $O
for c in c5 c3 c2; do
  echo "cfg $c" >> $O
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>>$O | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'])" >> $O 2>&1
done
