timeout 300 python tools/e2e_ab.py
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mpdata_dyn -s 1 -c 1 -o gpurun_out/prof_loop_r2d -f python tools/prof_loop.py 10 > gpurun_out/ncu_loop_r2d.log 2>&1; tail -2 gpurun_out/ncu_loop_r2d.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mpdata_dyn -s 2 -c 1 -o gpurun_out/prof_step_r2d -f python tools/prof_fused.py 0 4 > gpurun_out/ncu_step_r2d.log 2>&1; tail -2 gpurun_out/ncu_step_r2d.log
