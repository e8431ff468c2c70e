# K-rows-bulk (bulk_rows.cuh, ASNN_LEVEL_VARIANT 14-16): parity suites under the
# variant, then config 2 sweep times against the default k_rows (variant 5).
O=gpurun_out/bulk/r2_bulk.txt; mkdir -p gpurun_out/bulk; : > $O
ASNN_LEVEL_VARIANT=14 timeout 900 python -m pytest tests/test_gpu_activate.py tests/test_gpu_segments.py -x -q 2>&1 | tail -3 >> $O
ASNN_LEVEL_VARIANT=14 timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "c2 or config2 or full_size_bitwise" 2>&1 | tail -3 >> $O
for v in 5 14 15 16; do
  echo "variant $v c2 $(ASNN_LEVEL_VARIANT=$v timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'])")" >> $O
done
ASNN_LEVEL_VARIANT=14 timeout 300 ncu --metrics gpu__time_duration.sum,lts__t_sectors.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_rows_bulk -c 5 --csv --log-file gpurun_out/bulk/ncu_v14.csv python bench.py --config c2 --ncu-sweeps 1 > /dev/null 2>&1
