nvidia-smi --query-gpu=name,memory.total --format=csv,noheader
for sz in "4096 4096 137 10" "3300 3300 137 10" "2560 2576 137 10"; do timeout 900 python tools/big_patch_probe.py $sz 2>&1 | tail -1; done
