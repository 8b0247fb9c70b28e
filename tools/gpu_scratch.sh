for w in 2 3 4; do timeout 1500 python tools/o1280_strips_check.py 3 $w 2>&1 | tail -2; done | tee gpurun_out/o1280_strips_r2.log
