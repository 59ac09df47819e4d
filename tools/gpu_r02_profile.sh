#!/bin/bash
# Round-2 evidence: ncu launch list of the bench command, DRAM traffic per
# kernel class of one cfg2 update, ncu --set full of one step's GEMMs and of
# the fused output stage, and one SAC cfg4 bf16 GEMM.  Outputs in gpurun_out/.
O=gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench_r02.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 3 > $O/bench_under_ncu_r02.log 2>&1
python tools/launch_summary.py $O/launches_bench_r02.csv > $O/launches_bench_r02_summary.txt
head -400 $O/launches_bench_r02.csv > $O/launches_bench_r02_head.csv; rm -f $O/launches_bench_r02.csv
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none \
  --clock-control none --csv --log-file $O/launches_traffic_r02.csv python tools/profile_ppo.py bf16 > $O/pp_r02.log 2>&1
python tools/ncu_traffic.py $O/launches_traffic_r02.csv $O/ncu_traffic_r02.json > /dev/null; rm -f $O/launches_traffic_r02.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 24 -c 8 -o $O/gemm_step_r02 -f \
  python tools/profile_ppo.py bf16 > $O/ncu_full_r02.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ppo_fused_mma -s 4 -c 1 -o $O/fused_r02 -f \
  python tools/profile_ppo.py bf16 > $O/ncu_fused_r02.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:tc_gemm -s 40 -c 4 -o $O/sac_gemm_r02 -f \
  python tools/bench_sac.py --cfg cfg4 --precision bf16 --cpu-updates 0 --steps 8 --warmup 8 > $O/ncu_sac_r02.log 2>&1
for r in gemm_step_r02 fused_r02 sac_gemm_r02; do
  ncu -i $O/$r.ncu-rep --page raw --csv > $O/$r.raw.csv 2>/dev/null
done
ls -la $O
