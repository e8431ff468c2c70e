python -m pytest tests/test_gpu_gen.py -x -q 2>&1 | tail -3 > gpurun_out/r2_t8.txt
for v in "ASNN_CTA_WIN_LOG2=16" "ASNN_CTA_WIN_LOG2=14" "ASNN_CTA_WIN_LOG2=16 ASNN_CTA_STAGE=0"; do echo "$v" >> gpurun_out/r2_t8.txt; env $v python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'])" >> gpurun_out/r2_t8.txt 2>&1; done
python - >> gpurun_out/r2_t8.txt 2>&1 <<'PY'
import time, sys
sys.path.insert(0, '.')
import paper_2005_04347_b200 as A
dev = A.Device.get(0)
for rep in range(2):
    t = time.perf_counter(); dl = A.DeviceLayout.generated_powerlaw(10_000_000, 100, 1024, 1024, 500_000_000, 2.1, 4); dev.synchronize(); t1 = time.perf_counter() - t
    print("c4 device generate + levels", round(t1, 3), "s", dl.info()["edge_count"], dev.timings()); dl.free()
t = time.perf_counter(); net = A.generate_powerlaw(10_000_000, 100, 1024, 1024, 500_000_000, 2.1, 4); print("c4 host generate", round(time.perf_counter() - t, 2), "s")
t = time.perf_counter(); dl = A.DeviceLayout.from_network(net); dev.synchronize(); print("c4 host arrays -> layout", round(time.perf_counter() - t, 2), "s")
PY
