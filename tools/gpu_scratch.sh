mkdir -p gpurun_out
timeout 900 python tools/bench_stencils.py r2 > gpurun_out/stencils_r2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_table1_small_r2.csv python tools/prof_table1_small.py > /dev/null 2>&1
tail -3 gpurun_out/stencils_r2.log
