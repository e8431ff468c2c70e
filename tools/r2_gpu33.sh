O=gpurun_out/r2_t33.txt
timeout 300 python -m pytest tests/test_gpu_serve.py -x -q -s 2>&1 | grep -v '^\s*$' | tail -30 > $O
