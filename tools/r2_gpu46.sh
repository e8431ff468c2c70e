O=gpurun_out/r2_t46.txt
echo > $O
for w in 1 0 1 0 1; do
  ASNN_CHAIN_WIN=$w timeout 600 python -m pytest "tests/test_gpu_fullsize.py::test_config_full_size_bitwise" -q -k c3 2>&1 | tail -1 | sed "s/^/win=$w /" >> $O
done
