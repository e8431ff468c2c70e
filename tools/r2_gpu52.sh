O=gpurun_out/r2_t52.txt
timeout 600 python -m pytest tests/test_gpu_serve.py -x -q -s > gpurun_out/r2_t52_pytest.txt 2>&1; echo "pytest rc=$?" > $O
grep resident gpurun_out/r2_t52_pytest.txt >> $O
timeout 300 python tools/serve_probe.py >> $O 2>&1
timeout 300 python bench.py --config c1 --steps 200 --warmup 20 --no-cpu-baseline 2>>$O | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c1', d['ms_per_step'], d['e2e'])" >> $O 2>&1
for t in 256 384 448 512; do
  echo "c5 tmax=$t" >> $O
  ASNN_CTA_TMAX=$t timeout 300 python bench.py --config c5 --steps 20 --warmup 5 --no-cpu-baseline 2>>$O | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'])" >> $O 2>&1
done
