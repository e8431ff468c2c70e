# Exhaustive sigmoid check + config 5/2/4 timing for each saved build under build/ab/.
for lib in build/ab/libasnn_branchfree.so build/ab/lib_TAB32.so build/ab/lib_NOINL.so build/ab/lib_BOTH.so; do
  echo "== $lib"
  ASNN_B200_LIB=$PWD/$lib timeout 300 python -m pytest tests/test_gpu_sigmoid.py -q -m gpu -x 2>&1 | tail -1
  for cfg in c5 c2 c4; do
    ASNN_B200_LIB=$PWD/$lib timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$cfg\", round(d[\"ms_per_step\"],4))"
  done
done
