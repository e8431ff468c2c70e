python tools/percall_probe.py > gpurun_out/r2_percall2.txt 2>&1
python -m pytest tests/test_gpu_activate.py tests/test_gpu_segments.py tests/test_gpu_preprocess.py -x -q 2>&1 | tail -2 >> gpurun_out/r2_percall2.txt
ncu --set full --import-source on --clock-control none -k regex:k_cta -s 5 -c 1 -o gpurun_out/r2_c1_kcta python bench.py --config c1 --ncu-sweeps 8 > /dev/null 2>&1
