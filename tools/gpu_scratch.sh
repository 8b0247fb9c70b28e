CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool racecheck --print-limit 5 python tools/sanitize_dyn.py 64x128x32 > gpurun_out/san_rc2.log 2>&1; grep -v "^=========     \(#\|in \|Saved\)" gpurun_out/san_rc2.log | tail -5
