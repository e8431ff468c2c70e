# A/B of the sweep kernels between a saved baseline build (build/ab/*.so) and
# the current in-tree libasnn_b200.so, after the exhaustive sigmoid checks.
BASE=${BASE:-build/ab/libasnn_tab128.so}
timeout 600 python -m pytest tests/test_gpu_sigmoid.py -q -m gpu -x 2>&1 | tail -2
for cfg in ${CFGS:-c5 c2 c3 c4 c1}; do for lib in $BASE paper_2005_04347_b200/libasnn_b200.so; do
ASNN_B200_LIB=$PWD/$lib timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$cfg $lib\", round(d[\"ms_per_step\"],4), d[\"e2e\"][\"value\"])"
done; done
