for rep in 1 2; do for lib in libtsg.so libtsg_a4.so; do
TSG_LIBRARY=$PWD/paper_1908_06094_b200/$lib timeout 600 python bench.py --no-cpu --cpu-seconds 0 --sustained-seconds 0 > gpurun_out/bh_$lib.json 2>gpurun_out/bh_$lib.err
python - "$lib" <<'PY'
import json,sys
d=json.loads([l for l in open(f"gpurun_out/bh_{sys.argv[1]}.json") if l.startswith('{')][-1])
o=d['o1280_strong']
print(sys.argv[1], 'loop %.2f us %.3f'%(d['ms_per_step']*1e3, d['roofline']['frac']), 'flushed %.2f'%(d['step_flushed']['ms_per_step']*1e3),
      'o1280 %.2f ms (%.3f) iso %.2f'%(o['ms_per_step'], o['roofline_frac'], o['isolated_step']['ms_per_step']))
PY
done; done
