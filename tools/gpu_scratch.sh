mkdir -p gpurun_out
timeout 900 python tools/bench_stencils.py r2c > gpurun_out/stencils_r2c.log 2>&1
tail -2 gpurun_out/stencils_r2c.log
