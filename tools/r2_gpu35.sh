O=gpurun_out/r2_t35.txt
mkdir -p gpurun_out/r2_bench_csv
timeout 900 python tools/bench_csv.py --connections 1000,10000,100000,1000000 --depths 10,100 --csv gpurun_out/r2_bench_csv/r2_bench > $O 2>&1; echo "rc=$?" >> $O
timeout 600 python -m pytest tests/test_gpu_bench_csv.py -x -q >> $O 2>&1
