#!/bin/bash
# Dev loop: rebuild, run GPU tests + sweep trace + sweep bench on one gpurun call.
cd /root/repo || exit 1
make -s -j8 -C paper_2004_13961_b200/csrc 2>&1 | grep -iE "error" && exit 1
scripts/build_variants.sh trace -DLP_SWEEP_TRACE || exit 1
rm -f gpurun_out/gpu_tests.log gpurun_out/trace.txt gpurun_out/sweep.json
timeout 2400 /usr/local/graft/bin/gpurun --timeout 1500 -- "timeout 900 python -m pytest tests -q -m gpu --timeout 240 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo EXIT \$? >> gpurun_out/gpu_tests.log; LP_LIB_PATH=build/variants/trace.so timeout 300 python scripts/trace_sweep.py ${TRACE_CFG:-cfg2} > gpurun_out/trace.txt 2>&1; timeout 600 python scripts/bench_sweep.py ${SWEEP_CFGS:-cfg2 cfg3} > gpurun_out/sweep.json 2>&1" 2>&1 | tail -1
grep -E "passed|failed|EXIT|^FAILED" gpurun_out/gpu_tests.log | head
head -14 gpurun_out/trace.txt; grep -A8 "line 127 t" gpurun_out/trace.txt | cut -c1-40; grep lead gpurun_out/trace.txt
cat gpurun_out/sweep.json
