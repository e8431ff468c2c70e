#!/bin/bash
# C4 experiment: random-gather ceiling + heavy-branch scheduling variants.
mkdir -p gpurun_out
./tools/gather_bw 10000000 256 400000000 > gpurun_out/gather_bw.txt 2>&1
./tools/gather_bw 10000000 512 400000000 >> gpurun_out/gather_bw.txt 2>&1
for P in 1 0; do for T in 256 512 1024 4096; do
  echo "prio=$P thr=$T $(ASNN_HEAVY_PRIO=$P ASNN_HEAVY_THRESHOLD=$T python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["value"])')"
done; done > gpurun_out/c4_heavy_variants.txt 2>&1
