#!/bin/bash
# Time the 3-D sweep pair of several library variants on one cfg-4-recipe size (dev tool).
N=${N:-96}
for v in "$@"; do
  if [ "$v" = base ]; then L=""; else L="LP_LIB_PATH=build/variants/$v.so"; fi
  echo -n "$v "; env $L timeout 400 python scripts/probe_3d.py cfg4 $N --nopcg 2>&1 | grep -o '"sweep_pair_s": [0-9.]*'
done
