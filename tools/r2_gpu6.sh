python -m pytest tests/test_gpu_activate.py tests/test_gpu_writecount.py -x -q 2>&1 | tail -4 > gpurun_out/r2_t6.txt
python -m pytest tests/test_gpu_fullsize.py -x -q -k "c3" 2>&1 | tail -2 >> gpurun_out/r2_t6.txt
for v in "ASNN_CTA_STAGE=1" "ASNN_CTA_STAGE=0" "ASNN_CTA_WIN=0"; do echo "$v" >> gpurun_out/r2_t6.txt; env $v python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'])" >> gpurun_out/r2_t6.txt 2>&1; done
for w in 13 14; do echo "W=2^$w" >> gpurun_out/r2_t6.txt; ASNN_CTA_WIN_LOG2=$w python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'])" >> gpurun_out/r2_t6.txt 2>&1; done
ncu --set full --import-source on --clock-control none -k regex:k_cta -c 1 -o gpurun_out/r2_c3_win2 python bench.py --config c3 --ncu-sweeps 1 > /dev/null 2>&1
