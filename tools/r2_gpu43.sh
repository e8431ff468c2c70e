O=gpurun_out/r2_t43.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2_t43_pytest.txt 2>&1; echo "pytest rc=$?" > $O
tail -3 gpurun_out/r2_t43_pytest.txt >> $O
ASNN_BENCH_ONE_GPU=1 timeout 900 python bench.py --gpus 2 --config c3 > gpurun_out/r2_t43_g2_c3.json 2> gpurun_out/r2_t43_g2_c3.err; echo "g2 c3 rc=$?" >> $O
ASNN_BENCH_ONE_GPU=1 timeout 900 python bench.py --gpus 2 --config c5 > gpurun_out/r2_t43_g2_c5.json 2> gpurun_out/r2_t43_g2_c5.err; echo "g2 c5 rc=$?" >> $O
timeout 900 python bench.py --impl reference --config c3 > gpurun_out/r2_t43_ref_c3.json 2> gpurun_out/r2_t43_ref_c3.err; echo "ref c3 rc=$?" >> $O
