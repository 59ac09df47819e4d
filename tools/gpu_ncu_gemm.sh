#!/bin/bash
# ncu --set full of each cfg2 GEMM shape (one launch per shape) + launch list of one bf16 update
O=gpurun_out
BENCH_GEMM_ONCE=1 BENCH_DT=1 timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:tc_gemm -o $O/gemm_full -f python tools/bench_gemm.py > $O/ncu_gemm.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_bf16.csv python tools/profile_ppo.py bf16 > $O/profile_ppo_bf16.log 2>&1
python tools/launch_summary.py $O/launches_bf16.csv > $O/launch_summary_bf16.txt 2>&1
