# C4 per-rank slices (bench.py --shard-of G: rank 0's 64/G columns on one GPU)
# with an L2 persistence window over the earliest positions of A
# (ASNN_L2_PERSIST_MB): the earliest bands carry most gathers (uniform sources
# over all earlier ids), and at 8 columns their rows are 32 bytes.
O=gpurun_out/l2w/r2_l2win_shard.txt; mkdir -p gpurun_out/l2w; : > $O
python -c "import ctypes,torch; print('max persisting L2', torch.cuda.get_device_properties(0))" >> $O 2>&1
for g in 8 4; do for mb in 0 32 64 96; do
  echo "shard-of $g persist_mb $mb $(ASNN_L2_PERSIST_MB=$mb timeout 300 python bench.py --config c4 --shard-of $g --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), d['value'])")" >> $O
done; done
