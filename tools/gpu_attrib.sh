#!/usr/bin/env bash
# Attribution of the fused step's time and DRAM bytes per field (one GPU, under gpurun).
set -u
TAG=${1:-r2a}
mkdir -p gpurun_out
timeout 300 python tools/attrib_fused.py --out gpurun_out/attrib_${TAG}.json > gpurun_out/attrib_${TAG}.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_requests_srcunit_tex.sum \
    --clock-control none -k regex:mpdata_fused --csv --log-file gpurun_out/attrib_ncu_${TAG}.csv \
    python tools/prof_ops.py 0 99 94 90 91 92 93 0 > gpurun_out/attrib_ncu_${TAG}.log 2>&1
tail -n 3 gpurun_out/attrib_ncu_${TAG}.log
