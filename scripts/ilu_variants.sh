#!/bin/bash
# Time the 3-D ILU(0) of several library variants (dev tool): ilu_variants.sh "<probe args>" v1 v2 ...
ARGS=$1; shift
for v in "$@"; do
  if [ "$v" = base ]; then L=""; else L="LP_LIB_PATH=build/variants/$v.so"; fi
  echo -n "$v $ARGS: "; env $L timeout 600 python scripts/probe_3d.py $ARGS --nopcg 2>&1 | grep -o '"ilu0_s": [0-9.]*\|"sweep_pair_s": [0-9.]*' | tr '\n' ' '; echo
done
