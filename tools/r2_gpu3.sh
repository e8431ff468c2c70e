python -m pytest tests/test_gpu_writecount.py tests/test_gpu_concurrency.py tests/test_gpu_integration.py tests/test_gpu_cpp.py -x -q 2>&1 | tail -15 > gpurun_out/r2_t3.txt
