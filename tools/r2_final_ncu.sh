# Round-2 closing captures: C4 launch list of the bench command (cold-cache,
# serialised -- shares, not absolutes), one full capture of a C4 k_rows level,
# and one full capture of each one-call variant on its bench network.
O=gpurun_out/fncu; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file $O/c4_launches.csv python bench.py --config c4 --ncu-sweeps 2 > $O/c4_launches.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_rows -s 60 -c 1 -o $O/c4_k_rows python bench.py --config c4 --ncu-sweeps 1 > $O/c4_full.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:k_once_cluster -c 1 -o $O/once_cluster python tools/once_one.py 100000 10 2 > $O/once_cluster.log 2>&1
ASNN_ONCE_MODE=6 timeout 300 ncu --set full --clock-control none -k regex:k_once_cluster -c 1 -o $O/once_ranges python tools/once_one.py 100000 100 2 > $O/once_ranges.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:k_once -c 1 -o $O/once_cta python tools/once_one.py 10000 10 2 > $O/once_cta.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:k_once_pipe -c 1 -o $O/once_grid python tools/once_one.py 1000000 10 2 > $O/once_grid.log 2>&1
