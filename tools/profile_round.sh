#!/usr/bin/env bash
# Profiling recipe (run under gpurun on ONE GPU).  Produces in gpurun_out/:
#   bench_<tag>.json       a normal bench line (the driver's arguments; not under a profiler)
#   launches_<tag>.csv     every launch of a short bench run with its device time (cold, serialised)
#   prof_<tag>.ncu-rep     one --set full capture of the persistent loop kernel (10 steps, 279x256x80)
#   prof_step_<tag>.ncu-rep  one --set full capture of a single flushed step (279x256x80)
set -u
TAG=${1:-r2}
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 20 --warmup 5 --no-cpu --no-o1280 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mpdata_dyn -s 1 -c 1 \
    -o gpurun_out/prof_${TAG} -f python tools/prof_loop.py 10 > gpurun_out/ncu_${TAG}.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mpdata_dyn -s 2 -c 1 \
    -o gpurun_out/prof_step_${TAG} -f python tools/prof_fused.py 0 4 > gpurun_out/ncu_step_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_${TAG}.log
python tools/bench_brief.py gpurun_out/bench_${TAG}.json
