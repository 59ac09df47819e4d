O=gpurun_out
UL_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > $O/mr.log 2>&1; echo "rc=$?"; grep -v "^W\|^\*" $O/mr.log | tail -3 | cut -c1-400
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > $O/mr_ref.log 2>&1; echo "ref rc=$?"; tail -1 $O/mr_ref.log | cut -c1-300
