#!/bin/bash
# Round-1f captures (run on the GPU box via gpurun); each ncu run follows a plain run
# of the same command that exited 0.
cd /root/repo
C5="python scripts/probe_3d.py cfg5 512 --T 0 --nopcg"
$C5 > gpurun_out/r01f_c5_plain.txt 2>&1 || { echo "plain cfg5 probe failed"; exit 1; }
timeout 1500 ncu --set full --clock-control none -k regex:line_transform_kernel -c 6 \
  -o gpurun_out/r01f_mv_cfg5 $C5 > gpurun_out/r01f_ncu1.log 2>&1
C4="python scripts/probe_3d.py cfg4 48 --nopcg"
$C4 > gpurun_out/r01f_c4_plain.txt 2>&1 || { echo "plain cfg4 probe failed"; exit 1; }
timeout 1500 ncu --set full --clock-control none --replay-mode application -k regex:box_ilu0_3d_kernel -c 1 \
  -o gpurun_out/r01f_ilu3d_n48 $C4 > gpurun_out/r01f_ncu2.log 2>&1
echo done
