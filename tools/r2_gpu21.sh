O=gpurun_out/r2_t21.txt
echo > $O
for c in c3 c1 c5; do
  echo "cfg $c" >> $O
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>>$O | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d.get('e2e',{}).get('value'), d['value'])" >> $O 2>&1
done
echo "prof c3" >> $O
ASNN_B200_LIB=$PWD/build/exp/libasnn_b200_prof.so timeout 300 python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline 2>&1 | grep "chain prof\|producer" | tail -7 >> $O
