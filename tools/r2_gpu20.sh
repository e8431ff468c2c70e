O=gpurun_out/r2_t20.txt
echo "prof c3" > $O
ASNN_B200_LIB=$PWD/build/exp/libasnn_b200_prof.so timeout 300 python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline 2>&1 | grep "trace" | head -24 >> $O
