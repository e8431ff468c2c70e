ncu --set full --import-source on --clock-control none -k regex:k_chain -s 2 -c 1 -o gpurun_out/r2_c3_chain4 python bench.py --config c3 --ncu-sweeps 4 > gpurun_out/r2_t30.txt 2>&1
