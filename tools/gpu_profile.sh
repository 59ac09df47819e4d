#!/bin/bash
# One gpurun call: per-GEMM timings, HBM kernel microbench, ncu launch list of
# one un-graphed cfg2 update, a bench line.  Outputs land in gpurun_out/.
set -x
O=gpurun_out
BENCH_DT=1 timeout 120 python tools/bench_gemm.py > $O/gemm_bf16.json 2>&1
timeout 300 python tools/bench_kernels.py > $O/kernels.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches.csv python tools/profile_ppo.py > $O/profile_ppo.log 2>&1
python tools/launch_summary.py $O/launches.csv > $O/launch_summary.txt 2>&1
timeout 400 python bench.py --no-cpu-baseline > $O/bench2.log 2>&1
