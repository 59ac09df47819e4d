#!/bin/bash
# End-of-round evidence: bench line (with CPU baseline), ncu launch list of
# the bench command, DRAM traffic per kernel class of one update, ncu --set
# full of one minibatch step's GEMMs.  Outputs in gpurun_out/.
O=gpurun_out
timeout 600 python bench.py > $O/bench_final.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 3 > $O/bench_under_ncu.log 2>&1
python tools/launch_summary.py $O/launches_bench.csv > $O/launches_bench_summary.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none \
  --clock-control none --csv --log-file $O/launches_traffic.csv python tools/profile_ppo.py bf16 > $O/pp.log 2>&1
python tools/ncu_traffic.py $O/launches_traffic.csv $O/ncu_traffic.json > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 24 -c 8 -o $O/gemm_step -f \
  python tools/profile_ppo.py bf16 > $O/ncu_full.log 2>&1
tail -1 $O/bench_final.log | cut -c1-200
