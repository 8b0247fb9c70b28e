mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/gputest.log
cat gpurun_out/gputest.log
timeout 900 python tools/bench_stencils.py r2b > gpurun_out/stencils_r2b.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
tail -c 3000 gpurun_out/bench.log | python tools/bench_brief.py /dev/stdin 2>/dev/null || tail -c 1500 gpurun_out/bench.log
