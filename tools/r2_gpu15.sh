# round-2 re-entry check: full GPU suite, smoke, default bench line
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_t15.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_t15_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_t15.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/r2_t15.txt 2>&1
timeout 600 python bench.py > gpurun_out/r2_t15_bench.json 2> gpurun_out/r2_t15_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r2_t15_bench_ref.json 2> gpurun_out/r2_t15_bench_ref.err
