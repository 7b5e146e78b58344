#!/bin/bash
# usage: tools/bin_ab.sh OUTDIR V1 V2 ...: stage-2 device times (tools/bin_bench.py) per library build, configs 2 and 4
out=gpurun_out/$1; shift; mkdir -p $out
for rep in 1 2; do for v in "$@"; do for c in 2 4; do
  echo "$v c$c $(SSR_LIB=paper_2503_13086_b200/libssr_$v.so python tools/bin_bench.py --config $c --reps 30 2>/dev/null | tail -1)" >> $out/bin.log
done; done; done
cat $out/bin.log
