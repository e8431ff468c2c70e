python -m pytest tests/test_gpu_activate.py -x -q -k "k_cta-window or zero_row" 2>&1 | tail -2 > gpurun_out/r2_t9.txt
python -m pytest tests/test_gpu_fullsize.py -x -q -k "c3" 2>&1 | tail -1 >> gpurun_out/r2_t9.txt
for v in "ASNN_CTA_STAGE=1" "ASNN_CTA_WIN=0"; do echo "$v" >> gpurun_out/r2_t9.txt; env $v python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'])" >> gpurun_out/r2_t9.txt 2>&1; done
echo "L2 gathers: 2 MB slab of 512-byte rows" >> gpurun_out/r2_t9.txt
./tools/gather_bw 4000 512 400000000 >> gpurun_out/r2_t9.txt 2>&1
echo "L2 gathers: 32 MB slab of 512-byte rows" >> gpurun_out/r2_t9.txt
./tools/gather_bw 64000 512 400000000 >> gpurun_out/r2_t9.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_rows -s 100 -c 1 -o gpurun_out/r2_c2_k_rows python bench.py --config c2 --ncu-sweeps 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,lts__t_sectors_op_read.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/r2_c2_launches.csv python bench.py --config c2 --ncu-sweeps 1 > /dev/null 2>&1
