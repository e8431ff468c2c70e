O=gpurun_out/r2_t32.txt
timeout 600 python -m pytest tests/test_gpu_serve.py -x -q -s > gpurun_out/r2_t32_pytest.txt 2>&1; echo "pytest rc=$?" > $O
