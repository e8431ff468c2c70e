ncu --set full --warp-sampling-interval 0 --import-source on --clock-control none -k regex:k_cta -s 20 -c 1 -o gpurun_out/r2_c1_kcta_s0 python bench.py --config c1 --ncu-sweeps 30 > gpurun_out/r2_t14.txt 2>&1
python tools/latency_probe.py >> gpurun_out/r2_t14.txt 2>&1
