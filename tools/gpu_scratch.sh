timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_parity.py tests/test_gpu_acceptance.py -q -x 2>&1 | tail -2
timeout 900 python tools/bench_stencils.py r2e > /dev/null 2>&1; python -c "
import json
for d in json.load(open('gpurun_out/stencils_r2e.json')):
    if d['name'].startswith('mpdata'): print(d['name'], d['patch'], round(d['us'],1), round(d['frac'],3), d.get('fused_speedup'))
"
