#!/bin/bash
# usage: tools/variant_bench_c4.sh OUTDIR V1 V2 ...: config-2 step and config-4 batch leg per library build
out=gpurun_out/$1; shift; mkdir -p $out
for v in "$@"; do
  SSR_LIB=paper_2503_13086_b200/libssr_$v.so python bench.py --steps 20 --warmup 3 --batch-steps 2 --extra-steps 0 \
    --progressive-events 0 --no-cpu-baseline 2>>$out/err_$v.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); b=d['semi_global_batch']
print('$v', round(d['value'],1), round(d['e2e']['value'],1), d['stage_ms'], 'c4', round(b['views_per_s'],1), b['stage_ms_per_call'])" >> $out/variants.log
done
