cd /root/repo
python scripts/sweep_jitter.py cfg2 > gpurun_out/jitter.txt 2>&1
for v in trace tr_noprod tr_nowait tr_both; do
  echo "== $v" >> gpurun_out/exp.txt
  LP_LIB_PATH=build/variants/$v.so timeout 300 python scripts/trace_sweep.py cfg2 2>&1 | grep -E "^0 |^1 |^2 |lead" >> gpurun_out/exp.txt
done
