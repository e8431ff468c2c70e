python -m pytest tests/test_gpu_activate.py tests/test_gpu_writecount.py -x -q 2>&1 | tail -15 > gpurun_out/r2_t4.txt
python -m pytest tests/test_gpu_fullsize.py -x -q -k "c3" 2>&1 | tail -5 >> gpurun_out/r2_t4.txt
python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_bench_c3_win.json 2>&1
ASNN_CTA_WIN=0 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_bench_c3_nowin.json 2>&1
