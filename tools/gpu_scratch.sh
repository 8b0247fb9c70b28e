for d in 2 3 4 2 3; do
TSG_PIPE_DEPTH=$d timeout 600 python bench.py --steps 100 --no-o1280 --no-cpu --sustained-seconds 0 > gpurun_out/bp.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/bp.log').read().strip().splitlines()[-1])
print('depth $d', round(d['e2e']['ms_per_step'],4), round(d['e2e_all_inputs']['ms_per_step'],3))
"
done
