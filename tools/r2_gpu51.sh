O=gpurun_out/r2_t51.txt
echo > $O
for t in 256 384 448 512; do
  echo "c5 tmax=$t" >> $O
  ASNN_CTA_TMAX=$t timeout 300 python bench.py --config c5 --steps 20 --warmup 5 --no-cpu-baseline 2>>$O | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'])" >> $O 2>&1
done
for c in 64 32; do
  echo "c5 cmax=$c" >> $O
  ASNN_CTA_CMAX=$c timeout 300 python bench.py --config c5 --steps 20 --warmup 5 --no-cpu-baseline 2>>$O | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'])" >> $O 2>&1
done
