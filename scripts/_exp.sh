cd /root/repo
LP_LIB_PATH=build/variants/itrace.so timeout 300 python scripts/trace_ilu.py cfg2 > gpurun_out/exp.txt 2>&1
