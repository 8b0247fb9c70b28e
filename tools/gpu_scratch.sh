bash tools/gpu_round.sh > gpurun_out/round.log 2>&1
cp gpurun_out/bench.log gpurun_out/bench_r2e.log; cp gpurun_out/bench_ref.log gpurun_out/bench_ref_r2e.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_r2e.csv python bench.py --steps 20 --warmup 5 --no-cpu --no-o1280 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mpdata_dyn -s 1 -c 1 \
    -o gpurun_out/prof_r2e -f python tools/prof_loop.py 10 > gpurun_out/ncu_r2e.log 2>&1
timeout 900 python tools/bench_stencils.py r2f > gpurun_out/stencils_r2f.log 2>&1
tail -30 gpurun_out/round.log
