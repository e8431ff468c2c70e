ncu --set full --import-source on --clock-control none -k regex:k_chain -s 2 -c 1 -o gpurun_out/r2_c3_chainwin python bench.py --config c3 --ncu-sweeps 4 > gpurun_out/r2_t45.txt 2>&1
