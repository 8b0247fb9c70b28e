mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:reduce_tma -s 3 -c 1 -o gpurun_out/prof_cc -f python tools/prof_secondary.py reduce_cc > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:pack_pairs -s 3 -c 1 -o gpurun_out/prof_pack -f python tools/prof_secondary.py pack > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:reduce_indirect -s 3 -c 1 -o gpurun_out/prof_ind -f python tools/prof_secondary.py indirect > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
