# ncu full capture (source counters) of K-chain (grouped staging) on config 3
ncu --set full --import-source on --clock-control none -k regex:k_chain -s 2 -c 1 -o gpurun_out/r2_c3_chain2 python bench.py --config c3 --ncu-sweeps 4 > gpurun_out/r2_t25.txt 2>&1
