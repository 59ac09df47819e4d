O=gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ppo_fused -s 2 -c 1 -o $O/fused -f python tools/profile_ppo.py bf16 > $O/ncu_fused.log 2>&1
tail -3 $O/ncu_fused.log
