timeout 900 python bench.py > gpurun_out/bench_s.log 2>&1
python tools/bench_brief.py gpurun_out/bench_s.log
timeout 900 python bench.py > gpurun_out/bench_s2.log 2>&1
python tools/bench_brief.py gpurun_out/bench_s2.log
