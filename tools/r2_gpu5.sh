python -m pytest tests/test_gpu_writecount.py -x -q 2>&1 | tail -5 > gpurun_out/r2_t5.txt
for w in 12 13 14 15; do echo "W=2^$w" >> gpurun_out/r2_t5.txt; ASNN_CTA_WIN_LOG2=$w python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'])" >> gpurun_out/r2_t5.txt 2>&1; done
ncu --set full --import-source on --clock-control none -k regex:k_cta -c 1 -o gpurun_out/r2_c3_win python bench.py --config c3 --ncu-sweeps 1 > /dev/null 2>&1
ASNN_CTA_WIN=0 ncu --set full --import-source on --clock-control none -k regex:k_cta -c 1 -o gpurun_out/r2_c3_nowin python bench.py --config c3 --ncu-sweeps 1 > /dev/null 2>&1
ls -la gpurun_out >> gpurun_out/r2_t5.txt
