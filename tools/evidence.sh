#!/bin/bash
# Copy one profile_round.sh pass (gpurun_out/TAG) into profiles/TAG_*: bench lines, launch
# summaries, gap profiles, functional multi-rank runs, test logs, ncu digests and
# profiles/ncu_traffic.json.   bash tools/evidence.sh TAG
T=$1; O=gpurun_out/$T; P=profiles/$T
cp $O/bench.json ${P}_bench.json; cp $O/bench_ref.json ${P}_bench_ref.json
cp $O/gap_c2.txt ${P}_gap_c2.txt; cp $O/gap_c3.txt ${P}_gap_c3.txt
cp $O/launches_c2.csv ${P}_launches_c2.csv; cp $O/launches_c4.csv ${P}_launches_c4.csv
for c in c2 c3 c4; do python tools/launch_summary.py $O/launches_$c.csv > ${P}_launch_summary_$c.txt; done
cp $O/mg2_sharded_functional.json ${P}_mg2_sharded_functional.json
cp $O/mg2_p2p_functional.json ${P}_mg2_p2p_functional.json
tail -3 $O/pytest_gpu.log > ${P}_pytest_gpu.log; cp $O/smoke.log ${P}_smoke.log
python tools/ncu_summary.py $(ls -t $O/full_*.ncu-rep | head -13) $O/fused/full_*.ncu-rep > ${P}_ncu_full_summary.json 2>/dev/null
python tools/ncu_traffic.py ${P}_ncu_full_summary.json "dram__bytes_read.sum + dram__bytes_write.sum and duration of one launch (ncu --set full, cold cache, tools/profile_step.py at config 2 with the training objective's render (no soft counts); fused = SSR_FUSED=1); gpurun_out/$T -> profiles/${T}_*" > profiles/ncu_traffic.json
