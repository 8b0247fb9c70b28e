TSG_SHARE_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --steps 20 --warmup 3 > gpurun_out/bench4.log 2>&1
echo rc=$?
tail -c 2500 gpurun_out/bench4.log
