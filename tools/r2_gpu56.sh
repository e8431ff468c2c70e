O=gpurun_out/r2_t56.txt
: > $O
for w in 1 0 1; do
  echo "c2 level_win=$w" >> $O
  ASNN_LEVEL_WIN=$w timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline 2>>$O | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'])" >> $O 2>&1
done
timeout 600 python -m pytest tests/test_gpu_activate.py -x -q -k "c2 or wide or mlp" > gpurun_out/r2_t56_pytest.txt 2>&1; echo "pytest rc=$?" >> $O
tail -2 gpurun_out/r2_t56_pytest.txt >> $O
