#!/bin/bash
# Profiling pass for profiles/ (run on the GPU box via gpurun).  Each ncu run
# follows a plain run of the same command that exited 0.  Usage: profile_round.sh <tag> [workload]
cd /root/repo
set -o pipefail
TAG=${1:-r02}
WL=${2:-cfg3}
CMD="python bench.py --workload $WL --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err || { echo "plain run failed"; exit 1; }
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/prof_launches.csv $CMD > gpurun_out/prof_ncu1.log 2>&1
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__registers_per_thread,launch__grid_size,launch__block_size,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct"
timeout 1200 ncu --set full --clock-control none -k regex:ilu2d_kernel -c 1 --csv --page raw \
  --log-file gpurun_out/prof_ilu_full.csv $CMD > gpurun_out/prof_ncu2.log 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:box_sweep_kernel -c 2 --csv --page raw \
  --log-file gpurun_out/prof_sweep_full.csv $CMD > gpurun_out/prof_ncu3.log 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:line_transform_kernel -c 4 --csv --page raw \
  --log-file gpurun_out/prof_matvec_full.csv $CMD > gpurun_out/prof_ncu4.log 2>&1
echo done
