O=gpurun_out
timeout 600 python tools/bench_sac.py > $O/sac_cfg3.json 2>&1; tail -1 $O/sac_cfg3.json | cut -c1-600
timeout 600 python tools/bench_sac.py --no-ln > $O/sac_cfg3_noln.json 2>&1; tail -1 $O/sac_cfg3_noln.json | cut -c1-400
