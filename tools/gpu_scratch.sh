timeout 900 python tools/bench_stencils.py r2g > gpurun_out/stencils_r2g.log 2>&1; tail -3 gpurun_out/stencils_r2g.log
