O=gpurun_out/r2_t53.txt
echo > $O
for i in 1 2; do
  timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2_t53_pytest_$i.txt 2>&1; echo "suite $i rc=$?" >> $O
  tail -1 gpurun_out/r2_t53_pytest_$i.txt >> $O
done
timeout 600 python tools/percall_probe.py >> $O 2>&1
