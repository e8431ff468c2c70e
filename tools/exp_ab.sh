# A/B: saved baseline build (build/ab/base.so) against the in-tree library on
# the configs in $CFGS (default c3 c5 c2), 10 timed steps each, twice.
for cfg in ${CFGS:-c3 c5 c2}; do for rep in 1 2; do for lib in build/ab/base.so paper_2005_04347_b200/libasnn_b200.so; do
ASNN_B200_LIB=$PWD/$lib timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$cfg $lib\", round(d[\"ms_per_step\"],4))"
done; done; done
