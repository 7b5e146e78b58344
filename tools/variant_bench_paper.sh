#!/bin/bash
# usage: tools/variant_bench_paper.sh OUTDIR V1 V2 ...: the paper-objective leg (soft path) per library build
out=gpurun_out/$1; shift; mkdir -p $out
for v in "$@"; do
  SSR_LIB=paper_2503_13086_b200/libssr_$v.so python bench.py --steps 5 --warmup 3 --batch-steps 0 --extra-steps 10 \
    --progressive-events 0 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), d['paper_objective'], d['no_splat_parallel']['value'])" >> $out/variants_paper.log
done
