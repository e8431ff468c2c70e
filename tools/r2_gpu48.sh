O=gpurun_out/r2_t48.txt
timeout 1200 python -m pytest tests/test_gpu_activate.py tests/test_gpu_fullsize.py tests/test_gpu_writecount.py -q > gpurun_out/r2_t48_pytest.txt 2>&1; echo "pytest rc=$?" > $O
for i in 1 2 3 4 5 6; do
  ASNN_CHAIN_WIN=1 timeout 600 python -m pytest "tests/test_gpu_fullsize.py::test_config_full_size_bitwise" -q -k c3 2>&1 | tail -1 | sed "s/^/win=1 /" >> $O
done
