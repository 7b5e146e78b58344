#!/bin/bash
# Evidence pass for profiles/: bench (both arms), launch lists at configs 2 and 3,
# ncu --set full of the main kernels, progressive config-3 timing, device-timeline
# busy/idle splits (tools/gap_profile.py) at configs 2 and 3 and for a trained config-3 event.
#   gpurun --timeout 3000 -- 'bash tools/profile_round.sh TAG'
TAG=${1:-prof}
O=gpurun_out/$TAG
mkdir -p $O
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/status.txt
timeout 600 python bench.py --fused 0 --no-cpu-baseline > $O/bench_unfused.json 2> $O/bench_unfused.err; echo "bench_unfused exit $?" >> $O/status.txt
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "bench_ref exit $?" >> $O/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --progressive-events 0 > $O/ncu_bench.log 2>&1; echo "ncu_launch_bench exit $?" >> $O/status.txt
SSR_CFG=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv \
  python tools/profile_step.py > $O/ncu_c3.log 2>&1; echo "ncu_launch_c3 exit $?" >> $O/status.txt
bash tools/ncu_kernels.sh $O "k_forward$" k_backward_splat k_adam k_chain_geo k_chain_sh k_preprocess k_ssim_fwd k_ssim_bwd k_backward_fixup k_forward_fixup k_merge_big k_duplicate
SSR_FUSED=1 bash tools/ncu_kernels.sh $O/fused k_chain_geo k_chain_sh
timeout 900 python tools/progressive.py --events 4 > $O/progressive.json 2> $O/progressive.err; echo "progressive exit $?" >> $O/status.txt
SSR_CFG=2 timeout 400 python tools/gap_profile.py --view 8 > $O/gap_c2.txt 2>&1; echo "gap_c2 exit $?" >> $O/status.txt
SSR_CFG=3 timeout 400 python tools/gap_profile.py > $O/gap_c3.txt 2>&1; echo "gap_c3 exit $?" >> $O/status.txt
timeout 900 python tools/progressive.py --events 2 --gaps > $O/progressive_gaps.txt 2>&1; echo "progressive_gaps exit $?" >> $O/status.txt
cat $O/status.txt
