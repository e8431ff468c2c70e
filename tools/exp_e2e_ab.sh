# e2e (host buffers) A/B: saved build vs in-tree library, configs in $CFGS.
for cfg in ${CFGS:-c2 c4 c5 c1}; do for lib in build/ab/base.so paper_2005_04347_b200/libasnn_b200.so; do
ASNN_B200_LIB=$PWD/$lib timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$cfg $lib\", round(d[\"ms_per_step\"],4), \"e2e %.4g\" % d[\"e2e\"][\"value\"])"
done; done
