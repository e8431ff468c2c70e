# sanitizer pass over the round-2 kernels (K-chain, K-serve, k_rows_tma) + the write-count test
O=gpurun_out/r2_t38.txt
timeout 900 python -m pytest tests/test_gpu_writecount.py -x -q > $O 2>&1; echo "writecount rc=$?" >> $O
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  echo "== $tool serve" >> $O
  timeout 900 $CS --tool $tool --print-limit 20 python -m pytest tests/test_gpu_serve.py -x -q 2>&1 | grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|Hazard|Error' | head -20 >> $O
done
for tool in memcheck racecheck synccheck; do
  echo "== $tool c3 (k_chain, full size)" >> $O
  timeout 1200 $CS --tool $tool --print-limit 20 python bench.py --config c3 --ncu-sweeps 1 2>&1 | grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|Hazard|Error' | head -20 >> $O
  echo "== $tool c1 (k_chain NF=4)" >> $O
  timeout 600 $CS --tool $tool --print-limit 20 python bench.py --config c1 --ncu-sweeps 3 2>&1 | grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|Hazard|Error' | head -20 >> $O
done
echo "== memcheck activate (k_chain via sweep modes)" >> $O
timeout 1200 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_activate.py -x -q 2>&1 | grep -E 'ERROR SUMMARY|passed|failed' | tail -3 >> $O
echo "== memcheck c2 tma variant" >> $O
ASNN_LEVEL_VARIANT=13 timeout 1200 $CS --tool memcheck --print-limit 20 python bench.py --config c2 --ncu-sweeps 1 2>&1 | grep -E 'ERROR SUMMARY|Error' | head -5 >> $O
