O=gpurun_out/r2_t41.txt
echo > $O
for i in 1 2 3; do
  timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline 2>>$O | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2', d['ms_per_step'])" >> $O 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:k_cta -s 1 -c 1 -o gpurun_out/r2_c5_k_cta python bench.py --config c5 --ncu-sweeps 2 > gpurun_out/r2_t41_ncu.txt 2>&1
