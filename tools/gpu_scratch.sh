timeout 600 python bench.py --steps 20 --warmup 3 --no-o1280 > gpurun_out/bp.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/bp.log').read().strip().splitlines()[-1])
print(json.dumps(d['cpu_baseline']))
print(d['ms_per_step'], d['roofline']['frac'])
"
