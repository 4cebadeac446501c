#!/bin/bash
# matvec timing of library variants (dev tool): mv_variants.sh v1 v2 ...
for v in "$@"; do
  if [ "$v" = base ]; then L=""; else L="LP_LIB_PATH=build/variants/$v.so"; fi
  echo "== $v"; env $L timeout 600 python scripts/bench_matvec.py cfg2 cfg3 cfg4 cfg5 2>&1 | grep -o '"cfg": "[a-z0-9]*"\|"matvec_s": [0-9.e-]*\|"frac_fp64": [0-9.]*' | tr '\n' ' '; echo
done
