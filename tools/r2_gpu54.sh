O=gpurun_out/r2_t54.txt
timeout 1200 python -m pytest tests/test_gpu_activate.py tests/test_gpu_fullsize.py tests/test_gpu_segments.py tests/test_gpu_writecount.py -x -q > gpurun_out/r2_t54_pytest.txt 2>&1; echo "pytest rc=$?" > $O
tail -2 gpurun_out/r2_t54_pytest.txt >> $O
for w in 1 0; do
  echo "c2 level_win=$w" >> $O
  ASNN_LEVEL_WIN=$w timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline 2>>$O | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'])" >> $O 2>&1
done
echo "c4" >> $O
timeout 300 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline 2>>$O | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'])" >> $O 2>&1
