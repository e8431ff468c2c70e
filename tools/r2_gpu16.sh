# K-chain first run: parity suites that exercise K-cta, then C3/C1 timings chain on/off
O=gpurun_out/r2_t16.txt
timeout 900 python -m pytest tests/test_gpu_activate.py tests/test_gpu_segments.py tests/test_gpu_integration.py tests/test_gpu_writecount.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r2_t16_pytest.txt 2>&1; echo "pytest rc=$?" > $O
for c in c3 c1; do for ch in 1 0; do
  echo "cfg $c chain=$ch" >> $O
  ASNN_CTA_CHAIN=$ch timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>>$O | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d.get('e2e',{}).get('value'), d['value'])" >> $O 2>&1
done; done
