O=gpurun_out/r2_t49.txt
timeout 900 python -m pytest tests/test_gpu_sigmoid.py tests/test_gpu_activate.py tests/test_gpu_serve.py -x -q -s > gpurun_out/r2_t49_pytest.txt 2>&1; echo "pytest rc=$?" > $O
grep resident gpurun_out/r2_t49_pytest.txt >> $O
for c in c3 c5 c1 c2; do
  echo "cfg $c" >> $O
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline 2>>$O | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['us_per_step'])" >> $O 2>&1
done
