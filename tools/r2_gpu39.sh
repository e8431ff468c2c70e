O=gpurun_out/r2_t39.txt
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool synccheck --print-limit 6 python bench.py --config c3 --ncu-sweeps 1 > $O 2>&1
