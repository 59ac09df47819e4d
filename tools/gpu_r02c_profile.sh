#!/bin/bash
# Round-2 third-session (r02c) evidence: full GPU suite, bench line, ncu launch list of the
# bench command, DRAM traffic per kernel class of one cfg2 update, SAC cfg3 /
# cfg4 and APPO cfg5 lines.  Outputs in gpurun_out/.
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > $O/gputest_r02c.log 2>&1; echo "pytest rc=$?" >> $O/gputest_r02c.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/smoke_r02c.log 2>&1
timeout 600 python bench.py > $O/bench_r02c.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench_r02c.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 3 > $O/bench_under_ncu_r02c.log 2>&1
python tools/launch_summary.py $O/launches_bench_r02c.csv > $O/launches_bench_r02c_summary.txt
head -400 $O/launches_bench_r02c.csv > $O/launches_bench_r02c_head.csv; rm -f $O/launches_bench_r02c.csv
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none \
  --clock-control none --csv --log-file $O/launches_traffic_r02c.csv python tools/profile_ppo.py bf16 > $O/pp_r02c.log 2>&1
python tools/ncu_traffic.py $O/launches_traffic_r02c.csv $O/ncu_traffic_r02c.json > /dev/null; rm -f $O/launches_traffic_r02c.csv
for c in cfg3 cfg4; do timeout 300 python tools/bench_sac.py --cfg $c --precision bf16 --cpu-updates 0 > $O/sac_${c}_r02c.json 2>&1; done
timeout 600 python tools/bench_appo.py --cpu-envs 0 > $O/appo_cfg5_r02c.json 2>&1
tail -2 $O/gputest_r02c.log; tail -1 $O/smoke_r02c.log; tail -1 $O/bench_r02c.log | cut -c1-300
