cd /root/repo
LP_LIB_PATH=build/variants/trace.so timeout 300 python scripts/trace_sweep.py cfg2 2>&1 | grep -E "detect|slope|second-half|group:" > gpurun_out/exp.txt
