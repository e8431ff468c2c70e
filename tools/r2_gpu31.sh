O=gpurun_out/r2_t31.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_t31_pytest.txt 2>&1; echo "pytest rc=$?" > $O
for c in c3 c1 c5 c2; do
  echo "cfg $c" >> $O
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>>$O | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d.get('e2e',{}).get('value'), d['value'])" >> $O 2>&1
done
