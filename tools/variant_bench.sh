#!/bin/bash
# usage: tools/variant_bench.sh OUTDIR V1 V2 ...   (libssr_<V>.so built beside libssr.so)
out=gpurun_out/$1; shift; mkdir -p $out
for v in "$@"; do
  SSR_LIB=paper_2503_13086_b200/libssr_$v.so python bench.py --steps 20 --warmup 3 --batch-steps 0 --extra-steps 0 \
    --progressive-events 0 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), round(d['e2e']['value'],1), d['stage_ms'])" >> $out/variants.log
done
