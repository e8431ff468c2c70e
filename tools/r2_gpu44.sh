O=gpurun_out/r2_t44.txt
timeout 1200 python -m pytest tests/test_gpu_activate.py tests/test_gpu_fullsize.py tests/test_gpu_writecount.py tests/test_gpu_segments.py -x -q > gpurun_out/r2_t44_pytest.txt 2>&1; echo "pytest rc=$?" > $O
for w in 1 0; do
  echo "c3 chain_win=$w" >> $O
  ASNN_CHAIN_WIN=$w timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline 2>>$O | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'])" >> $O 2>&1
done
