mkdir -p gpurun_out
for i in 1 2; do for pr in 0 1 2; do
TSG_PROMO=$pr timeout 600 python bench.py --no-o1280 --no-cpu --steps 200 > gpurun_out/bp$pr.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/bp$pr.log').read().strip().splitlines()[-1])
print('promo $pr', round(d['ms_per_step']*1e3,2), round(d['roofline']['frac'],3), 'flushed', round(d['step_flushed']['ms_per_step']*1e3,2), 'static-graph', round(d['time_loop']['ms_per_step']*1e3,2), 'e2e', round(d['e2e']['value']/1e9,2))
"
done; done
