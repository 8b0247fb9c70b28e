for rep in 1 2; do timeout 600 python tools/bench_stencils.py ab fusion 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['name'], d['patch'], round(d['us'],1), round(d['frac'],3))
"; done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/prof_unfused_o1280.py > gpurun_out/unfused_o1280_d.csv 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
