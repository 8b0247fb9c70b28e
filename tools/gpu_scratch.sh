timeout 900 python -m pytest tests/test_distributed.py -q -x 2>&1 | tail -3
TSG_SHARE_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/bench2.log 2>&1
echo rc=$?; python -c "
import json
d=json.loads(open('gpurun_out/bench2.log').read().strip().splitlines()[-1])
print(d['setup']['path'], d['setup']['halo_exchange'][:60], d['o1280_strong']['path'])
"
