out=gpurun_out/s3r; mkdir -p $out
for rep in 1 2; do
for v in copy mapped; do
for late in "" 1; do
  SSR_PREFETCH_LATE=$late SSR_LIB=paper_2503_13086_b200/libssr_$v.so python bench.py --steps 30 --warmup 3 --batch-steps 0 --extra-steps 0 --progressive-events 0 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v late=$late', round(d['value'],1), round(d['e2e']['value'],1))" >> $out/e2e.log
done; done; done
cat $out/e2e.log
