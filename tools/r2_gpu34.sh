O=gpurun_out/r2_t34.txt
echo > $O
for c in c1 c3; do
timeout -s SIGABRT 200 python -X faulthandler bench.py --config $c --steps 200 --warmup 20 --no-cpu-baseline 2>>$O | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e'], d['value'])" >> $O 2>&1
done
