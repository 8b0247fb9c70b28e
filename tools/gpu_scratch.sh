CS=/usr/local/cuda/bin/compute-sanitizer
timeout 3300 $CS --tool memcheck --target-processes all --print-limit 5 python -m pytest tests -m gpu -q -x -k "not o1280 and not bench_line" > gpurun_out/memcheck_all_r2.log 2>&1
echo rc=$?
grep -v "^=========     \(#\|in \|Saved\)" gpurun_out/memcheck_all_r2.log | tail -6
