#!/bin/bash
# Evidence pass for profiles/: GPU tests + smoke, bench (both arms), launch lists at
# configs 2 and 3, ncu --set full of the main kernels, device-timeline busy/idle splits,
# and a functional (gloo, one GPU, never a measurement) run of the N = 2 sharded bench path.
#   gpurun --timeout 3600 -- 'bash tools/profile_round.sh TAG'
TAG=${1:-prof}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest_gpu exit $?" >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/status.txt
T0=$(date +%s); timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $? ($(( $(date +%s) - T0 )) s)" >> $O/status.txt
T0=$(date +%s); timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "bench_ref exit $? ($(( $(date +%s) - T0 )) s)" >> $O/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv \
  python tools/profile_step.py > $O/ncu_c2.log 2>&1; echo "ncu_launch_c2 exit $?" >> $O/status.txt
SSR_CFG=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv \
  python tools/profile_step.py > $O/ncu_c3.log 2>&1; echo "ncu_launch_c3 exit $?" >> $O/status.txt
bash tools/ncu_kernels.sh $O "^k_forward$" k_backward_splat k_adam k_chain_geo k_chain_sh k_preprocess k_ssim_fwd k_ssim_bwd k_backward_fixup k_forward_fixup k_merge_big k_duplicate k_radix_down
SSR_FUSED=1 bash tools/ncu_kernels.sh $O/fused k_chain_geo k_chain_sh
SSR_CFG=2 timeout 400 python tools/gap_profile.py --view 8 > $O/gap_c2.txt 2>&1; echo "gap_c2 exit $?" >> $O/status.txt
SSR_CFG=3 timeout 400 python tools/gap_profile.py > $O/gap_c3.txt 2>&1; echo "gap_c3 exit $?" >> $O/status.txt
SSR_DIST_BACKEND=gloo SSR_FORCE_DEVICE0=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 3 --warmup 3 --exchange sharded \
  --batch-views 8 --batch-steps 1 --extra-steps 0 --progressive-events 0 --no-cpu-baseline \
  > $O/mg2_sharded_functional.json 2> $O/mg2_sharded_functional.err; echo "mg2_functional exit $?" >> $O/status.txt
SSR_DIST_BACKEND=gloo SSR_FORCE_DEVICE0=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 3 --warmup 3 --exchange p2p \
  --batch-views 8 --batch-steps 1 --extra-steps 0 --progressive-events 0 --no-cpu-baseline \
  > $O/mg2_p2p_functional.json 2> $O/mg2_p2p_functional.err; echo "mg2_p2p_functional exit $?" >> $O/status.txt
SSR_CFG=4 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv \
  python tools/profile_step.py > $O/ncu_c4.log 2>&1; echo "ncu_launch_c4 exit $?" >> $O/status.txt
cat $O/status.txt
