O=gpurun_out/r2_t47.txt
echo > $O
for cfg in "1 2" "1 1" "0 2"; do set -- $cfg
  echo "c3 chain_win=$1 ctas=$2" >> $O
  ASNN_CHAIN_WIN=$1 ASNN_CHAIN_WIN_CTAS=$2 timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline 2>>$O | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'])" >> $O 2>&1
done
