cd /root/repo
LP_LIB_PATH=build/variants/trace.so timeout 300 python scripts/trace_sweep.py cfg2 > gpurun_out/exp.txt 2>&1
