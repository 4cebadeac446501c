#!/bin/bash
# Profiling pass for profiles/ (run on the GPU box via gpurun).  Each ncu run
# follows a plain run of the same command that exited 0.
cd /root/repo
set -o pipefail
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err || { echo "plain run failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/prof_launches.csv $CMD > gpurun_out/prof_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:box_sweep_kernel -c 2 --csv --page raw \
  --log-file gpurun_out/prof_sweep_full.csv $CMD > gpurun_out/prof_ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:box_ilu0_tasks -c 1 --csv --page raw \
  --log-file gpurun_out/prof_ilu_full.csv $CMD > gpurun_out/prof_ncu3.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:line_transform_kernel -c 4 --csv --page raw \
  --log-file gpurun_out/prof_mv_full.csv $CMD > gpurun_out/prof_ncu4.log 2>&1
echo done
