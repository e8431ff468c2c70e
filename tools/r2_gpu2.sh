set -x
python -m pytest tests/test_gpu_group.py tests/test_gpu_activate.py -x -q 2>&1 | tail -8 > gpurun_out/r2_group.txt
python -m pytest tests/test_gpu_fullsize.py -x -q -k "reference_golden" 2>&1 | tail -8 > gpurun_out/r2_fullsize.txt
python bench.py --config c4 --steps 10 --warmup 3 > gpurun_out/r2_bench_c4.json 2> gpurun_out/r2_bench_c4.err
python bench.py --impl reference --config c4 --steps 5 --warmup 3 > gpurun_out/r2_bench_c4_ref.json 2> gpurun_out/r2_bench_c4_ref.err
ASNN_BENCH_ONE_GPU=1 python bench.py --gpus 2 --config c4 --scale 0.1 --steps 5 --warmup 3 > gpurun_out/r2_bench_onegpu2.json 2> gpurun_out/r2_bench_onegpu2.err
ASNN_BENCH_ONE_GPU=1 python bench.py --gpus 2 --config c5 --scale 0.1 --steps 5 --warmup 3 > gpurun_out/r2_bench_onegpu2_c5.json 2> gpurun_out/r2_bench_onegpu2_c5.err
