#!/bin/bash
# Round-1d evidence pass (run on the GPU box via gpurun).  Every ncu run follows a plain
# run of the same command that exited 0.
cd /root/repo
python bench.py > gpurun_out/r01d_bench.json 2> gpurun_out/r01d_bench.err || echo "bench failed"
python scripts/bench_3d.py --no-cpu5 > gpurun_out/r01d_bench_3d.jsonl 2> gpurun_out/r01d_bench_3d.err || echo "bench_3d failed"
C5="python scripts/probe_3d.py cfg5 512 --T 0 --nopcg"
$C5 > gpurun_out/r01d_c5_plain.txt 2>&1 || { echo "plain cfg5 probe failed"; exit 1; }
timeout 1500 ncu --set full --clock-control none -k regex:"box_sweep3d_multi_kernel|line_transform_kernel" -c 8 \
  -o gpurun_out/r01d_cfg5_t0 $C5 > gpurun_out/r01d_ncu.log 2>&1
echo done
