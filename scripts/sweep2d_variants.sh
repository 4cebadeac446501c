#!/bin/bash
# 2-D sweep timing of library variants (dev tool)
for v in "$@"; do
  if [ "$v" = base ]; then L=""; else L="LP_LIB_PATH=build/variants/$v.so"; fi
  echo "== $v"; env $L timeout 600 python scripts/bench_sweep.py cfg2 cfg3 2>&1 | grep -o '"cfg": "[a-z0-9]*"\|"fwd_s": [0-9.e-]*\|"bwd_s": [0-9.e-]*\|"ilu0_s": [0-9.e-]*' | tr '\n' ' '; echo
done
