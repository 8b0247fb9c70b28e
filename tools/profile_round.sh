#!/usr/bin/env bash
# Profiling recipe (run under gpurun on ONE GPU).  Produces in gpurun_out/:
#   launches_<tag>.csv  every launch of a short bench run with its device time (cold, serialised)
#   prof_<tag>.ncu-rep  one --set full capture of the fused MPDATA kernel (279x256x80)
#   bench_<tag>.json    a normal bench line (not under a profiler)
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 300 python bench.py --steps 2000 --warmup 20 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 20 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mpdata_fused -s 2 -c 1 \
    -o gpurun_out/prof_${TAG} -f python tools/prof_fused.py 0 4 > gpurun_out/ncu_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_${TAG}.log
cat gpurun_out/bench_${TAG}.json | tail -1 | cut -c1-400
