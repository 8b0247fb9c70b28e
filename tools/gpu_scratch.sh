timeout 900 python -m pytest tests -m gpu -x -q -k "pack or reorder or layout or strided or stream or relabel or point_bands or acceptance" 2>&1 | tail -2
for sz in "2560 2576 137" "2560 2576 136" "1024 1024 81" "1024 1024 80" "279 256 80" "279 256 79"; do timeout 900 python tools/reorder_probe.py $sz 2 2>&1 | grep '"sn"'; done
