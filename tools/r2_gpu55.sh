ncu --set full --import-source on --clock-control none -k regex:k_rows_win -s 100 -c 1 -o gpurun_out/r2_c2_rows_win python bench.py --config c2 --ncu-sweeps 2 > gpurun_out/r2_t55.txt 2>&1
