O=gpurun_out/r2_t50.txt
timeout 1200 python -m pytest tests/test_gpu_parse.py tests/test_gpu_validate.py tests/test_gpu_hostio.py -x -q > gpurun_out/r2_t50_pytest.txt 2>&1; echo "pytest rc=$?" > $O
tail -3 gpurun_out/r2_t50_pytest.txt >> $O
