#!/bin/bash
# ncu --set full of the first launch (after one warm iteration) of each named kernel
# of tools/profile_step.py: bash tools/ncu_kernels.sh OUTDIR kernel [kernel ...]
# (env SSR_CFG / SSR_FUSED pass through to profile_step.py)
O=$1; shift
mkdir -p $O
for K in "$@"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 \
    -o $O/full_${K//[^A-Za-z0-9_]/} python tools/profile_step.py > $O/ncu_full_${K//[^A-Za-z0-9_]/}.log 2>&1
  echo "ncu_full_${K//[^A-Za-z0-9_]/} exit $?" >> $O/status.txt
done
