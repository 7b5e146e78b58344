mkdir -p gpurun_out/$1; rm -f gpurun_out/$1/bb.log
for c in 2 3; do python tools/bin_bench.py --config $c 2>&1 | grep -v Warn >> gpurun_out/$1/bb.log; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$1/bin_launches.csv python tools/bin_bench.py --config 2 --reps 1 > /dev/null 2>&1
