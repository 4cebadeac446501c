#!/bin/bash
# Round-1c profiling pass (run on the GPU box via gpurun).  Every ncu run follows
# a plain run of the same command that exited 0.
cd /root/repo
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err || { echo "plain bench failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/prof_launches.csv $CMD > gpurun_out/prof_ncu1.log 2>&1
C3="python scripts/probe_3d.py cfg4 128 --nopcg"
$C3 > gpurun_out/prof_c3_plain.txt 2>&1 || { echo "plain cfg4 probe failed"; exit 1; }
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:box_sweep3d_kernel -c 2 \
  -o gpurun_out/r01c_sweep3d_cfg4 $C3 > gpurun_out/prof_ncu2.log 2>&1
C4="python scripts/probe_3d.py cfg4 48 --nopcg"
$C4 > gpurun_out/prof_c4_plain.txt 2>&1 || { echo "plain cfg4 N=48 probe failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:box_ilu0_3d_kernel -c 1 \
  -o gpurun_out/r01c_ilu3d_n48 $C4 > gpurun_out/prof_ncu3.log 2>&1
echo done
