TSG_SHARE_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 bench.py --gpus 2 --steps 20 --warmup 3 --no-o1280 > gpurun_out/bench2.log 2>&1
echo rc=$?
python -c "
import json
d=json.loads(open('gpurun_out/bench2.log').read().strip().splitlines()[-1])
print(json.dumps(d['e2e'])); print(d['e2e_all_inputs'], d['time_loop'], d['e2e_time_loop'])
"
timeout 600 python bench.py --steps 20 --warmup 3 --no-o1280 > gpurun_out/bench1.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/bench1.log').read().strip().splitlines()[-1])
print(d['e2e']['value'], d['e2e_all_inputs']['value'], d['time_loop']['value'], d['e2e_time_loop']['value'])
"
