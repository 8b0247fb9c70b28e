mkdir -p gpurun_out
run() { TSG_HINT=$1 timeout 600 python bench.py --no-o1280 --no-cpu --steps 200 > gpurun_out/bp.log 2>gpurun_out/bp.err
python -c "
import json
d=json.loads(open('gpurun_out/bp.log').read().strip().splitlines()[-1])
print('hint $1', round(d['ms_per_step']*1e3,2), round(d['roofline']['frac'],3), 'flushed', round(d['step_flushed']['ms_per_step']*1e3,2))
"; }
for h in 0 1 2 3 4 5 7 0; do run $h; done
for h in 0 1 5; do TSG_HINT=$h timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:mpdata_dyn -s 2 -c 1 --csv python tools/prof_loop.py 10 2>/dev/null | grep -o '"dram__bytes_read.sum","byte","[0-9]*"\|"gpu__time_duration.sum","ns","[0-9]*"' | tr '\n' ' ' | sed "s/^/hint $h loop10 /"; echo; done
