#!/bin/bash
# One GPU validation pass: parity tests, smoke, bench (both arms), launch list and
# ncu captures of the blend kernels.  Run under gpurun from the repo root:
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh [tag]'
# Each step is bounded by its own timeout; outputs land in gpurun_out/<tag>/.
TAG=${1:-run}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest_gpu exit $?" >> $O/status.txt
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/status.txt
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/status.txt
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "bench_ref exit $?" >> $O/status.txt
if [ -z "$SKIP_NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches.csv python tools/profile_step.py > $O/ncu_launch.log 2>&1; echo "ncu_launch exit $?" >> $O/status.txt
for K in ${NCU_KERNELS:-k_backward_splat k_forward}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^${K}\$|ssr::${K}" -s 1 -c 1 \
    -o $O/full_$K python tools/profile_step.py > $O/ncu_full_$K.log 2>&1; echo "ncu_full_$K exit $?" >> $O/status.txt
done
fi
if [ -n "$PROGRESSIVE" ]; then
  timeout 900 python tools/progressive.py $PROGRESSIVE > $O/progressive.json 2> $O/progressive.err; echo "progressive exit $?" >> $O/status.txt
fi
cat $O/status.txt
