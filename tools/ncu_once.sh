mkdir -p gpurun_out/once3; rm -f gpurun_out/once3/*
for m in 1 3; do for cd in "100000 100" "100000 10" "1000 100"; do
  set -- $cd
  ASNN_ONCE_MODE=$m timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/once3/m${m}_c$1_d$2.csv python tools/once_one.py $1 $2 5 > gpurun_out/once3/m${m}_c$1_d$2.log 2>&1
done; done
for cd in "1000000 100" "1000000 10"; do set -- $cd
  for m in 2 4; do ASNN_ONCE_MODE=$m timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/once3/m${m}_c$1_d$2.csv python tools/once_one.py $1 $2 5 > gpurun_out/once3/m${m}_c$1_d$2.log 2>&1; done
done
