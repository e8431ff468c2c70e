# round-2 evidence run: full GPU suite, smoke, default bench (C4), per-config
# benches, ncu captures of K-chain (C3) and the C1 K-chain launch, launch lists
set -x
O=gpurun_out/r2_t37.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_t37_pytest.txt 2>&1; echo "pytest rc=$?" > $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $O 2>&1
for c in c1 c2 c3 c5; do
  timeout 600 python bench.py --config $c > gpurun_out/r2_bench_$c.json 2> gpurun_out/r2_bench_$c.err
done
timeout 600 python bench.py > gpurun_out/r2_bench_c4.json 2> gpurun_out/r2_bench_c4.err
ncu --set full --import-source on --clock-control none -k regex:k_chain -s 2 -c 1 -o gpurun_out/r2_c3_k_chain_final python bench.py --config c3 --ncu-sweeps 4 > gpurun_out/r2_t37_ncu_c3.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_c3_launches.csv python bench.py --config c3 --ncu-sweeps 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_c1_launches.csv python bench.py --config c1 --ncu-sweeps 20 > /dev/null 2>&1
