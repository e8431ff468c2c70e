#!/bin/bash
# Serialized per-launch times (ncu launch list) of one C4 sweep per light-kernel variant.
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for V in 0 1 5 6; do
  ASNN_SWEEP_MODE=3 ASNN_LEVEL_VARIANT=$V ASNN_HEAVY_THRESHOLD=512 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/light_v$V.csv python bench.py --config c4 --ncu-sweeps 1 > /dev/null 2>&1
done
ASNN_HEAVY_THRESHOLD=512 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/light_stream.csv python bench.py --config c4 --ncu-sweeps 1 > /dev/null 2>&1
ls gpurun_out/light_*
